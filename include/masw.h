/*
 * masw.h -- C ABI of the B200-native MASW theoretical dispersion-curve forward model
 * (Kump & Martin, "MASWAccelerated", arXiv:2003.02256; PAPER.md in the survey).
 *
 * Library: paper_2003_02256_b200/libmasw.so (sm_100a SASS, no PTX JIT).
 *
 * The forward model: for a layered model M over a half-space, for every
 * wavelength lambda_i and ascending test velocity c_j, form the Kausel-Roesset stiffness
 * matrix K(k = 2*pi/lambda_i, c_j) of order 2(N+1), take the sign of
 * Re det K, and return C_t(lambda_i) = c_n at the first sign change (Algorithm 1,
 * PAPER.md:50-71); then the misfit m = (1/l) sum |C_t - C_e| / C_e (Algorithm 2,
 * PAPER.md:80-93).  Readings of points the paper leaves open are listed in DESIGN.md
 * ("Readings S1-S22") and are restated where they affect an argument below.
 *
 * Conventions for every entry point
 *   - fp64 SI units (m, m/s, kg/m^3); indices int32; sizes int64.
 *   - Model layout is structure-of-arrays, row-major: h[M][N], alpha/beta/rho[M][N+1];
 *     index N of alpha/beta/rho is the half-space (reading S22).
 *   - The caller owns every buffer.  Array pointers are either ALL host pointers or ALL
 *     device pointers (classified with cudaPointerGetAttributes; managed memory counts as
 *     device; mixing kinds in one call returns MASW_E_ARG).
 *       host pointers:   inputs are staged to the device, results copied back; the call
 *                        returns after completion.
 *       device pointers: work is enqueued on exec->cuda_stream; the call synchronises that
 *                        stream once to read the status word back, unless MASW_ASYNC is set
 *                        (then it returns right after enqueue, skips the status readback and
 *                        the caller guarantees valid inputs; per-row outcomes stay in idx).
 *   - On any error (< 0) the output buffers are left untouched.
 *   - Thread-safe for concurrent calls on distinct streams.
 *   - Per-row outcomes are in-band: idx = j >= 1 is the index of the first sign change and
 *     C_t = c[j] (the unperturbed grid value, reading S7); idx = MASW_IDX_NO_CHANGE (-1)
 *     means no sign change on the grid (reading S8), idx = MASW_IDX_NONFINITE (-2) means a
 *     determinant before the first change was NaN/Inf (reading S9); C_t = NaN for both.
 *     The return code is the worst status: MASW_WARN_NO_SIGN_CHANGE (> 0) if any row is < 0.
 *
 * Validation (the same for every entry point that takes these arguments, in this order):
 *   MASW_E_ARG       null required pointer, L < 1, L > INT32_MAX, V < 2, V > INT32_MAX, M < 0,
 *                    N < 1 or N > MASW_MAX_LAYERS
 *   MASW_E_NONFINITE a NaN/Inf in lambda or c                                 (reading S9)
 *   MASW_E_GRID      lambda_i <= 0, c_0 <= 0, or c not strictly increasing
 *   MASW_E_NONFINITE / MASW_E_MODEL  the lowest-index model with a NaN/Inf, or violating
 *                    h > 0, rho > 0, beta > 0, alpha > beta
 *   MASW_E_RANGE     (2*pi/lambda_i) * h_e > 350 for some i, e (cosh overflow guard, S9;
 *                    700 with MASW_STABLE)
 *   then C_e (when given): NaN/Inf -> MASW_E_NONFINITE, C_e <= 0 -> MASW_E_ARG
 */
#ifndef MASW_H
#define MASW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MASW_ABI_VERSION 1
/* Largest N (finite layers) the kernels accept; the paper's models have N <= 10. */
#define MASW_MAX_LAYERS 64

enum masw_status {
    MASW_OK = 0,
    MASW_WARN_NO_SIGN_CHANGE = 1, /* outputs valid; some idx < 0                         */
    MASW_E_ARG = -1,
    MASW_E_MODEL = -2,
    MASW_E_GRID = -3,
    MASW_E_RANGE = -4,            /* 2*pi*h/lambda > 350                                 */
    MASW_E_NONFINITE = -5,
    MASW_E_CUDA = -6,             /* a CUDA runtime call failed (see masw_last_cuda_error) */
    MASW_E_NOMEM = -7
};

#define MASW_IDX_NO_CHANGE (-1)
#define MASW_IDX_NONFINITE (-2)

/* One layered model (Algorithm 1's M): N finite layers over a half-space. */
typedef struct {
    int32_t n_layers;      /* N >= 1                                                       */
    const double *h;       /* [N]   thickness, m, > 0                                      */
    const double *alpha;   /* [N+1] P-wave velocity, m/s; alpha > beta                     */
    const double *beta;    /* [N+1] S-wave velocity, m/s; > 0                               */
    const double *rho;     /* [N+1] density, kg/m^3; > 0                                   */
} masw_model;

/* M candidate models with the same N (the repeated evaluations of PAPER.md:99), SoA. */
typedef struct {
    int64_t n_models;      /* M >= 0 (M == 0 is a no-op returning MASW_OK)                 */
    int32_t n_layers;      /* N                                                            */
    const double *h;       /* [M][N]                                                        */
    const double *alpha;   /* [M][N+1]                                                      */
    const double *beta;    /* [M][N+1]                                                      */
    const double *rho;     /* [M][N+1]                                                      */
} masw_ensemble;

/* exec.flags */
#define MASW_ASYNC 0x1u       /* device pointers: no status readback, return after enqueue  */
#define MASW_TIME_SCAN 0x2u   /* record CUDA events around the scan kernels (both cosh/sinh table
                                 instances; not the small-c pre-pass): masw_last_scan_ms */
/* Row schedule of the scan (default: a work-stealing queue over rows, lambda-major).  The two
 * static schedules are the paper's partitions, here over the kernel's teams:
 * team g of G takes a contiguous block of rows, or rows g, g+G, g+2G, ... (load-balance
 * study; results are identical for every schedule). */
#define MASW_SCHED_CONTIGUOUS 0x4u
#define MASW_SCHED_MODULAR 0x8u
/* record each team's algorithmic det count (masw_last_team_dets; synchronous calls only) */
#define MASW_TEAM_STATS 0x10u
/* Kernel choice for the queue schedule (default: automatic).  Ensembles with many models use
 * the MODEL-MAJOR scan: a warp takes one model and up to 64 of its wavelengths and computes
 * the wavelength-free terms of each velocity (wave square roots, half-space element / k)
 * once for all of them; otherwise the ROW scan (teams of
 * team_warps warps per (model, lambda) row).  Results are identical.  MASW_SCHED_ROWS forces
 * the row scan; MASW_SCHED_MODELS forces the model-major scan where its per-warp cache fits
 * (N <= ~8; else the row scan runs).  With MASW_TEAM_STATS a model-major "team" is a warp. */
#define MASW_SCHED_ROWS 0x20u
#define MASW_SCHED_MODELS 0x40u
/* Calls that do not take the model-major scan (one model, or ensembles too small for it, or
 * N > ~8) run a pair scan when there are >= 4 rows per resident warp: a warp scans two
 * consecutive wavelengths of one model in lockstep, sharing the per-velocity wave roots
 * (results identical to the row scan).  MASW_SCHED_PAIRS forces it (any call with L >= 2);
 * MASW_SCHED_ROWS forces the row scan. */
#define MASW_SCHED_PAIRS 0x200u
/* Small-c prefix (reading S15'').  At very low c the direct App. A formulas
 * cancel: the relative fp64 error of det K is of the order of
 *   P(c, k) = 2^-53 max_e [16 (beta_e/c)^4 + (alpha_e beta_e / c^2)^2 / (k h_e)^4],
 * so their signs are noise where P ~ 1 (e.g. a thin stiff lid scanned from 0.5 m/s).  By
 * DEFAULT every determinant with P > 1e-3 -- a prefix of each row's ascending grid -- is
 * evaluated with the stable element below (in a pre-pass kernel shared by every scan) and
 * the rest with the direct element, so C_t is the first change of the exact signs for any
 * grid start.  MASW_DIRECT skips the prefix (the direct element everywhere: A/B only). */
#define MASW_DIRECT 0x400u
/* Numerically stable element: the layer
 * stiffness is evaluated in cancellation-free form for c -> 0 (both waves hyperbolic) and
 * with exponentially scaled hyperbolic functions, so the range guard becomes
 * (2*pi/lambda_i) * h_e <= 700 instead of 350 (MASW_E_RANGE above that).  Costs ~2.6x per
 * determinant; runs through the same scans as the default (row, model-major, pair; results
 * identical across them).  With it every determinant uses the stable element (no prefix
 * is needed).  Applies to masw_curve, masw_curves_ensemble and masw_det_grid. */
#define MASW_STABLE 0x80u
/* Scan signs by the banded GEPP for every determinant (default: the block LDL^T recursion,
 * certified per determinant, GEPP only where the certificate fails; DESIGN.md "sign by
 * block recursion").  For validation and A/B measurement; the results agree. */
#define MASW_PIVOTED 0x100u

/* Execution options; a NULL masw_exec means {device = current, stream = legacy default,
 * team_warps = 0 (auto), flags = 0}. */
typedef struct {
    int32_t device;        /* CUDA device ordinal; -1 = current device                      */
    void *cuda_stream;     /* cudaStream_t; NULL = legacy default stream                     */
    int32_t team_warps;    /* warps cooperating on one (model, lambda) row: 0 = auto, else a
                              power of two in [1, 16]; each step scans 32*team_warps
                              consecutive velocities speculatively.
                              (SURVEY.md 8(b)'s chunk_width, counted in warps: chunk width
                              = 32 * team_warps velocities.)                                */
    uint32_t flags;        /* MASW_* flags above                                             */
} masw_exec;

/* Theoretical dispersion curve of one model (Algorithm 1).
 *   lambda[L]  wavelengths W, m, any order (reading S17)
 *   c[V]       test velocities V, m/s, strictly increasing, c[0] > 0 (reading S20)
 *   ct_out[L]  C_t(lambda_i) = c[idx_i] or NaN                         (required)
 *   idx_out[L] first-sign-change index, or MASW_IDX_* (nullable)
 * Returns MASW_OK, MASW_WARN_NO_SIGN_CHANGE or an error code. */
int masw_curve(const masw_model *model, const double *lambda, int64_t L, const double *c,
               int64_t V, double *ct_out, int32_t *idx_out, const masw_exec *exec);

/* Misfit of one curve (Algorithm 2): m = (1/L) sum_i |ct_i - ce_i| / ce_i.
 * +inf if any ct_i is NaN/Inf (reading S8).  Errors: L < 1 or null -> MASW_E_ARG;
 * ce NaN/Inf -> MASW_E_NONFINITE; ce <= 0 -> MASW_E_ARG.  misfit_out: one double.
 * exec (nullable; an addition to SURVEY.md 8(b)'s signature): device and stream for
 * device-pointer calls, as for the other entry points. */
int masw_misfit(const double *ct, const double *ce, int64_t L, double *misfit_out,
                const masw_exec *exec);

/* Misfits of M curves against one C_e: ct[M][L] -> misfit_out[M] (same rules as above). */
int masw_misfit_batch(const double *ct, const double *ce, int64_t M, int64_t L,
                      double *misfit_out, const masw_exec *exec);

/* C_t, idx and misfit of M models against one experimental curve (the optimisation /
 * uncertainty loop of PAPER.md:31, :99).  ce[L] nullable -> no misfit; ct_out[M][L]
 * required; idx_out[M][L] and misfit_out[M] nullable (misfit_out requires ce). */
int masw_curves_ensemble(const masw_ensemble *ens, const double *lambda, int64_t L,
                         const double *c, int64_t V, const double *ce, double *ct_out,
                         int32_t *idx_out, double *misfit_out, const masw_exec *exec);

/* Index of the smallest misfit, ties -> lowest index, NaN treated as +inf.
 * best_out: one int64 (-1 when M == 0); best_misfit_out: one double (nullable). */
int masw_argmin(const double *misfit, int64_t M, int64_t *best_out, double *best_misfit_out,
                const masw_exec *exec);

/* Debug / parity: every det K(lambda_i, c_j) on the full grid, no early exit (the (lambda, c)
 * "grid" of PAPER.md:109).  det = (mant_re + i*mant_im) * 2^exp2 with
 * max(|mant_re|, |mant_im|) in [0.5, 1) (0 for an exactly zero det).  Outputs [L][V]. */
int masw_det_grid(const masw_model *model, const double *lambda, int64_t L, const double *c,
                  int64_t V, double *mant_re, double *mant_im, int32_t *exp2,
                  const masw_exec *exec);

/* Human-readable name of a status code (static storage). */
const char *masw_strerror(int code);

/* MASW_ABI_VERSION of the loaded library. */
int masw_version(void);

/* Last CUDA error string seen by the calling thread (static storage; "" if none). */
const char *masw_last_cuda_error(void);

/* Number of kernels this library has launched in this process (all threads). */
int64_t masw_kernel_launches(void);

/* Device time in ms of the calling thread's last scan kernel launched with MASW_TIME_SCAN
 * (CUDA events recorded around the launch on the launching stream; for a MASW_ASYNC call the
 * first query waits for the end event); -1 if none. */
double masw_last_scan_ms(void);

/* Device times in ms of the calling thread's most recent MASW_TIME_SCAN scan launches (up to
 * the last 64), oldest first, into ms_out[0..n); waits for their end events.  Returns the
 * number written (<= n) or MASW_E_ARG. */
int masw_recent_scan_ms(double *ms_out, int32_t n);

/* Per-team algorithmic det counts (sum of idx+1 over the rows each team scanned) of the
 * calling thread's last synchronous call made with MASW_TEAM_STATS, into out[0..n).  Returns
 * the number of teams of that launch (which may exceed n), or -1 if none was recorded. */
int64_t masw_last_team_dets(int64_t *out, int64_t n);

/* Algorithmic work of the calling thread's last curve/ensemble call: the early-exit
 * determinant count sum_rows (idx+1) of SPEC.md:246 (rows with idx < 0 count V for -1 and
 * are not counted for -2), and the determinants actually evaluated including speculation.
 * Only filled for synchronous calls (not MASW_ASYNC); -1 otherwise. */
int masw_last_work(int64_t *algorithmic_dets, int64_t *evaluated_dets);

/* Small-c prefix (reading S15'', MASW_DIRECT) of the calling thread's last synchronous
 * curve/ensemble call: rows with a prefix, and determinants evaluated with the stable element
 * there.  Returns 0, or -1 if none was recorded (MASW_ASYNC, MASW_STABLE, MASW_DIRECT). */
int masw_last_prefix(int64_t *rows, int64_t *dets);

/* Of the determinants the calling thread's last synchronous scan evaluated, how many had
 * their sign re-evaluated by the banded GEPP because the block recursion's multipliers were
 * not certified; -1 if there was no such call. */
int64_t masw_last_fallbacks(void);

#ifdef __cplusplus
}
#endif
#endif /* MASW_H */
