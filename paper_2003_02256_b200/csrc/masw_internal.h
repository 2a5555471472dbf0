// masw_internal.h -- declarations shared by the kernels TU and the C-ABI TU of libmasw.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace masw {

// Device workspace of one call (allocated stream-ordered, zeroed before use).
struct Workspace {
    unsigned long long queue;          // next row to scan (work-stealing counter)
    unsigned long long alg_dets;       // sum over rows of (event index + 1)
    unsigned long long eval_dets;      // determinants evaluated incl. speculation
    unsigned long long model_err;      // ~key of first bad model: key = m << 2 | class
    unsigned long long h_max_bits;     // max h over all layers/models (positive doubles)
    unsigned long long lam_min_nbits;  // ~bits(min lambda)
    unsigned int grid_err;             // bit0 lambda nonfinite, bit1 c nonfinite, bit2 lambda<=0,
                                       // bit3 c0<=0, bit4 c not increasing,
                                       // bit5 ce nonfinite, bit6 ce<=0
    unsigned int row_status;           // bit0 some idx == -1, bit1 some idx == -2
    int abort;                         // set by the scan kernel when validation failed
    int range_bad;                     // k_max * h_max > 350
    unsigned long long fallback_dets;  // sign re-evaluated with GEPP (block recursion not certified)
    unsigned long long prefix_rows;    // rows with a small-c prefix (reading S15''; smallc_rows_kernel)
    unsigned long long prefix_dets;    // determinants evaluated by smallc_prefix_kernel
};

// sizeof(LayerConst) (masw_det.cuh; static_assert in masw_kernels.cu) and MASW_MAX_LAYERS
// (include/masw.h; static_assert in masw_capi.cu)
constexpr size_t kLayerConstBytes = 48;
constexpr int kMaxLayers = 64;

// Model classes for Workspace::model_err
constexpr unsigned kModelNonfinite = 1u;
constexpr unsigned kModelBad = 2u;

struct ModelArgs {
    int64_t M;
    int N;
    const double *h, *alpha, *beta, *rho;
};

struct ScanArgs {
    ModelArgs mod;
    const double *lam;
    int64_t L;
    const double *c;
    int64_t V;
    double *ct;        // [M][L]
    int32_t *idx;      // [M][L] or nullptr
    Workspace *ws;
    unsigned grid_mask;  // Workspace::grid_err bits that invalidate the call (0x1F, 0x7F with C_e)
    int sched;           // 0 work-stealing queue, 1 static contiguous, 2 static modular
    unsigned long long *team_dets;  // per-team algorithmic det counts (nullable)
    int stable;          // MASW_STABLE: the scaled, cancellation-free element (row kernel)
    int pivoted;         // MASW_PIVOTED: every sign by the banded GEPP (no block recursion)
    // model-major scan only (set by its launcher): the last tail_models models are queued
    // as finer work items of tail_rows wavelengths, so the warps finish closer together
    int64_t tail_models;
    int tail_rows;
    // small-c prefix (reading S15''), written by smallc_prefix_kernel per output row m*L + i:
    // start = first grid index the scan evaluates (the dets below it were evaluated with the
    // stable element), or -1 when the row was finished there; carry = sgn Re det at start-1.
    // nullptr: no prefix (MASW_STABLE / MASW_DIRECT), every row starts at 0.
    const int32_t *pstart;
    const int8_t *pcarry;
    // pair scan only (set by its launcher): the last tail_pairs pair items are split into
    // seg_count velocity segments of seg_len grid points each (tail segments);
    // seg_found[2 tail_pairs]: each tail row's smallest in-segment event index (atomicMin);
    // seg_rec[2 tail_pairs][seg_count]: per-segment record for pair_tail_combine_kernel
    int64_t tail_pairs;
    int seg_count, seg_len;
    int *seg_found;
    int2 *seg_rec;
};

// grid_mask bit: the call uses the stable element, range guard k h <= 700 instead of 350
constexpr unsigned kGridStable = 0x100u;

// Launchers (masw_kernels.cu).  Each returns the cudaError_t of its launch.
cudaError_t launch_validate(const ModelArgs &m, const double *lam, int64_t L, const double *c,
                            int64_t V, const double *ce, Workspace *ws, cudaStream_t st);
// *teams_out (nullable) receives the number of teams the launch used.
cudaError_t launch_scan(const ScanArgs &a, int team_warps, cudaStream_t st, int device,
                        long long *teams_out = nullptr);
long long scan_teams(const ScanArgs &a, int team_warps, int device);
cudaError_t launch_misfit(const double *ct, const double *ce, int64_t M, int64_t L,
                          double *misfit, Workspace *ws, unsigned grid_mask, bool check_models,
                          cudaStream_t st);
cudaError_t launch_validate_ce(const double *ce, int64_t L, Workspace *ws, cudaStream_t st);
cudaError_t launch_argmin(const double *misfit, int64_t M, int64_t *best, double *best_val,
                          cudaStream_t st);
cudaError_t launch_det_grid(const ModelArgs &m, const double *lam, int64_t L, const double *c,
                            int64_t V, double *mre, double *mim, int32_t *ex, Workspace *ws,
                            cudaStream_t st, bool stable = false, bool prefix = true);
int auto_team_warps(int64_t rows, int64_t V, int device);
// Reading S15'': find and list the rows with a small-c prefix (grid points with c_j^4 < Q_r;
// list: scratch for M L row ids; lcbuf: for M (N+1) k-free LayerConst, or nullptr), evaluate their prefixes with the stable element, write pstart /
// pcarry (ScanArgs) and finish rows whose first change lies in the prefix.  Runs before any
// scan kernel of the same call on the same stream.
cudaError_t launch_smallc_prefix(const ScanArgs &a, int32_t *start, int8_t *carry, int64_t *list,
                                 void *lcbuf, cudaStream_t st, int device);
// Model-major scan (ensembles): suitable when there are many (model, wavelength-block) items
// and the per-warp caches fit two CTAs per SM; same outputs as launch_scan.
bool models_scan_suitable(const ScanArgs &a, int device, bool forced);
// pair scan (single curves of many wavelengths, two rows per warp in lockstep)
bool pairs_scan_suitable(const ScanArgs &a, int device, bool forced);
// Scratch bytes the pair scan needs for its tail segments (0: none); the caller passes that
// many bytes (device, 16-byte aligned) to launch_scan_pairs.
size_t pair_tail_scratch_bytes(const ScanArgs &a, int device);
cudaError_t launch_scan_pairs(const ScanArgs &a, void *tail_scratch, cudaStream_t st, int device,
                              long long *warps_out = nullptr);
long long scan_pairs_warps(const ScanArgs &a, int device);
cudaError_t launch_scan_models(const ScanArgs &a, cudaStream_t st, int device,
                               long long *warps_out = nullptr);
long long scan_models_warps(const ScanArgs &a, int device);

void count_launch();
long long launches();

}  // namespace masw
