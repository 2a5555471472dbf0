// masw_capi.cu -- the extern "C" boundary of libmasw.so (include/masw.h).
//
// Host responsibilities only: argument checks that need no data, pointer classification,
// staging of host buffers, stream-ordered workspace, kernel launches (masw_kernels.cu) and
// the status readback.  Every step of the forward model runs in the kernels; there is no
// CPU compute path.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/masw.h"
#include "masw_det.cuh"
#include "masw_internal.h"

using namespace masw;
static_assert(kMaxLayers == MASW_MAX_LAYERS, "masw_internal.h kMaxLayers");

namespace {

thread_local char t_cuda_err[256] = "";
thread_local Workspace *t_pinned_ws = nullptr;   // pinned host copy target for the status read
// Scan-kernel timing events of the calling thread (MASW_TIME_SCAN): a ring of the last
// kScanRing launches, resolved lazily so MASW_ASYNC calls can be timed without host waits.
constexpr int kScanRing = 64;
thread_local cudaEvent_t t_scan_ev[kScanRing][2] = {};
thread_local int t_scan_dev[kScanRing] = {};   // device + 1 the slot's events were created on
thread_local long long t_scan_count = 0;   // TIME_SCAN launches recorded by this thread
thread_local long long t_last_alg = -1, t_last_eval = -1, t_last_fb = -1;
thread_local long long t_last_prefix_rows = -1, t_last_prefix_dets = -1;
thread_local std::vector<long long> t_team_dets;
thread_local long long t_team_count = -1;

struct Fail {
    int code;
};

int cuda_fail(cudaError_t e, const char *what)
{
    snprintf(t_cuda_err, sizeof(t_cuda_err), "%s: %s", what, cudaGetErrorString(e));
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? MASW_E_NOMEM : MASW_E_CUDA;
}

#define CK(call)                                         \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) throw Fail{cuda_fail(_e, #call)}; \
    } while (0)

// 0 = null, 1 = host, 2 = device (or managed); device ordinal in *dev for device pointers.
int classify(const void *p, int *dev)
{
    if (!p) return 0;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        *dev = a.device;
        return 2;
    }
    return 1;
}

// All non-null pointers must share a kind.  Returns 1 (host), 2 (device) or -1 (mixed).
int common_kind(std::initializer_list<const void *> ps, int *dev)
{
    int kind = 0;
    for (const void *p : ps) {
        int d = -1;
        const int k = classify(p, &d);
        if (k == 0) continue;
        if (kind == 0) {
            kind = k;
            if (k == 2) *dev = d;
        } else if (k != kind) {
            return -1;
        }
    }
    return kind == 0 ? 1 : kind;
}

struct Exec {
    int device;
    cudaStream_t stream;
    int team;
    uint32_t flags;
};

Exec resolve(const masw_exec *ex)
{
    Exec r{-1, nullptr, 0, 0u};
    if (ex) {
        r.device = ex->device;
        r.stream = static_cast<cudaStream_t>(ex->cuda_stream);
        r.team = ex->team_warps;
        r.flags = ex->flags;
    }
    return r;
}

// The stream-ordered allocator's default pool releases memory back to the OS at every
// synchronisation (release threshold 0), so the host path's staging buffers (~70 MB for C5)
// were unmapped and re-mapped on every call; measured on the GPU box as 2-350 ms per call.
// Keep freed memory in the pool (once per device).
std::atomic<unsigned long long> g_pool_configured{0};

void configure_pool(int dev)
{
    if (dev < 0 || dev >= 64) return;
    const unsigned long long bit = 1ull << dev;
    if (g_pool_configured.load(std::memory_order_acquire) & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    g_pool_configured.fetch_or(bit, std::memory_order_acq_rel);
}

// Restores the caller's current device on scope exit.
struct DeviceScope {
    int prev = -1;
    bool changed = false;
    void set(int dev)
    {
        CK(cudaGetDevice(&prev));
        if (dev >= 0 && dev != prev) {
            CK(cudaSetDevice(dev));
            changed = true;
        }
        configure_pool(dev >= 0 ? dev : prev);
    }
    ~DeviceScope()
    {
        if (changed) cudaSetDevice(prev);
    }
};

// Stream-ordered device buffers freed on scope exit (after the final synchronisation).
struct Arena {
    cudaStream_t st;
    void *ptrs[32];
    int n = 0;
    explicit Arena(cudaStream_t s) : st(s) {}
    template <class T>
    T *alloc(size_t count)
    {
        void *p = nullptr;
        CK(cudaMallocAsync(&p, count * sizeof(T) + 16, st));
        ptrs[n++] = p;
        return static_cast<T *>(p);
    }
    template <class T>
    T *stage_in(const T *host, size_t count)
    {
        if (!host) return nullptr;
        T *d = alloc<T>(count);
        CK(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
        return d;
    }
    ~Arena()
    {
        for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], st);
    }
};

// Waits for everything enqueued on `st` (spin-wait: a blocking-sync event was measured to
// wake up 10-700 ms late on the GPU box; callers that must not wait use MASW_ASYNC).
void wait_stream(cudaStream_t st)
{
    CK(cudaStreamSynchronize(st));
}

// Reads the device workspace into pinned host memory (pageable copies can stall) and
// waits for the stream.
Workspace read_status(const Workspace *ws, cudaStream_t st)
{
    if (!t_pinned_ws) CK(cudaMallocHost(&t_pinned_ws, sizeof(Workspace)));
    CK(cudaMemcpyAsync(t_pinned_ws, ws, sizeof(Workspace), cudaMemcpyDeviceToHost, st));
    wait_stream(st);
    return *t_pinned_ws;
}

// Error precedence of include/masw.h from the workspace filled by validate_kernel.
int decode(const Workspace &w, bool with_ce, bool with_models, bool stable = false)
{
    if (w.grid_err & 3u) return MASW_E_NONFINITE;
    if (w.grid_err & 28u) return MASW_E_GRID;
    if (with_models) {
        if (w.model_err) {
            const unsigned long long key = ~w.model_err;
            return ((key & 3ull) == kModelNonfinite) ? MASW_E_NONFINITE : MASW_E_MODEL;
        }
        double lam_min, h_max;
        const unsigned long long lb = ~w.lam_min_nbits;
        memcpy(&lam_min, &lb, 8);
        memcpy(&h_max, &w.h_max_bits, 8);
        const double kmax = kTwoPi / lam_min;
        if (kmax * h_max > (stable ? kMaxKHStable : kMaxKH)) return MASW_E_RANGE;
    }
    if (with_ce) {
        if (w.grid_err & 32u) return MASW_E_NONFINITE;
        if (w.grid_err & 64u) return MASW_E_ARG;
    }
    return w.row_status ? MASW_WARN_NO_SIGN_CHANGE : MASW_OK;
}

// ------------------------------------------------------------------ curves / ensemble core
int run_curves(const ModelArgs &mod_in, const double *lam, int64_t L, const double *c,
               int64_t V, const double *ce, double *ct_out, int32_t *idx_out,
               double *misfit_out, const masw_exec *exp)
{
    if (!mod_in.h || !mod_in.alpha || !mod_in.beta || !mod_in.rho || !lam || !c || !ct_out)
        return MASW_E_ARG;
    if (L < 1 || L > INT32_MAX || V < 2 || V > INT32_MAX || mod_in.M < 0 || mod_in.N < 1 ||
        mod_in.N > MASW_MAX_LAYERS)
        return MASW_E_ARG;
    if (misfit_out && !ce) return MASW_E_ARG;
    if (mod_in.M == 0) return MASW_OK;
    t_last_alg = t_last_eval = t_last_fb = -1;
    t_last_prefix_rows = t_last_prefix_dets = -1;
    const Exec ex = resolve(exp);
    if (ex.team != 0 && (ex.team < 1 || ex.team > 16 || (ex.team & (ex.team - 1))))
        return MASW_E_ARG;
    int pdev = -1;
    const int kind = common_kind({mod_in.h, mod_in.alpha, mod_in.beta, mod_in.rho, lam, c, ce,
                                  ct_out, idx_out, misfit_out},
                                 &pdev);
    if (kind < 0) return MASW_E_ARG;
    const bool host = (kind == 1);
    try {
        DeviceScope scope;
        scope.set(ex.device >= 0 ? ex.device : (host ? -1 : pdev));
        int dev = 0;
        CK(cudaGetDevice(&dev));
        const cudaStream_t st = ex.stream;
        Arena arena(st);
        const int64_t M = mod_in.M, N = mod_in.N, R = M * L;

        ModelArgs mod = mod_in;
        const double *dlam = lam, *dc = c, *dce = ce;
        double *dct = ct_out, *dmis = misfit_out;
        int32_t *didx = idx_out;
        if (host) {
            mod.h = arena.stage_in(mod_in.h, M * N);
            mod.alpha = arena.stage_in(mod_in.alpha, M * (N + 1));
            mod.beta = arena.stage_in(mod_in.beta, M * (N + 1));
            mod.rho = arena.stage_in(mod_in.rho, M * (N + 1));
            dlam = arena.stage_in(lam, L);
            dc = arena.stage_in(c, V);
            dce = arena.stage_in(ce, L);
            dct = arena.alloc<double>(R);
            didx = idx_out ? arena.alloc<int32_t>(R) : nullptr;
            dmis = misfit_out ? arena.alloc<double>(M) : nullptr;
        }
        Workspace *ws = arena.alloc<Workspace>(1);
        CK(cudaMemsetAsync(ws, 0, sizeof(Workspace), st));
        CK(launch_validate(mod, dlam, L, dc, V, dce, ws, st));

        const int team = ex.team ? ex.team : auto_team_warps(R, V, dev);
        const int sched = (ex.flags & MASW_SCHED_CONTIGUOUS) ? 1 : ((ex.flags & MASW_SCHED_MODULAR) ? 2 : 0);
        const bool stable = (ex.flags & MASW_STABLE) != 0;
        ScanArgs sa{mod, dlam, L, dc, V, dct, didx, ws,
                    (dce ? 0x7Fu : 0x1Fu) | (stable ? kGridStable : 0u), sched, nullptr, stable,
                    (ex.flags & MASW_PIVOTED) != 0};
        // model-major scan for ensembles (auto unless a team size, a static schedule or
        // MASW_SCHED_ROWS is requested; MASW_SCHED_MODELS forces it where it fits)
        const bool models = !(ex.flags & MASW_SCHED_ROWS) && sched == 0 &&
                            (((ex.flags & MASW_SCHED_MODELS) && models_scan_suitable(sa, dev, true)) ||
                             (ex.team == 0 && models_scan_suitable(sa, dev, false)));
        // pair scan for single curves of many wavelengths (auto unless a team size, a static
        // schedule or MASW_SCHED_ROWS is requested; MASW_SCHED_PAIRS forces it for M == 1)
        const bool pairs = !models && !(ex.flags & MASW_SCHED_ROWS) &&
                           (((ex.flags & MASW_SCHED_PAIRS) && pairs_scan_suitable(sa, dev, true)) ||
                            (ex.team == 0 && pairs_scan_suitable(sa, dev, false)));
        const bool stats = (ex.flags & MASW_TEAM_STATS) != 0 && !(ex.flags & MASW_ASYNC);
        long long nteams = 0;
        if (stats) {
            nteams = models ? scan_models_warps(sa, dev)
                            : (pairs ? scan_pairs_warps(sa, dev) : scan_teams(sa, team, dev));
            if (nteams <= 0) return MASW_E_CUDA;
            sa.team_dets = arena.alloc<unsigned long long>((size_t)nteams);
            CK(cudaMemsetAsync(sa.team_dets, 0, nteams * sizeof(unsigned long long), st));
        }
        const bool timed = (ex.flags & MASW_TIME_SCAN) != 0;
        cudaEvent_t *slot = t_scan_ev[t_scan_count % kScanRing];
        if (timed) {
            // an event records only on a stream of its own device: (re)create the slot's pair
            // on this call's device when the thread last used the slot on another one
            int &sdev = t_scan_dev[t_scan_count % kScanRing];
            if (sdev != dev + 1) {
                for (int q = 0; q < 2; ++q)
                    if (slot[q]) {
                        cudaEventDestroy(slot[q]);
                        slot[q] = nullptr;
                    }
                CK(cudaEventCreate(&slot[0]));
                CK(cudaEventCreate(&slot[1]));
                sdev = dev + 1;
            }
        }
        // reading S15'': the rows' small-c prefixes with the stable element, before the scan
        if (!stable && !(ex.flags & MASW_DIRECT)) {
            int32_t *pst = arena.alloc<int32_t>((size_t)R);
            int8_t *pca = arena.alloc<int8_t>((size_t)R);
            // per-model constants for the prefix pass (bounded: formed per element beyond)
            const size_t lcb_bytes = (size_t)M * (size_t)(N + 1) * kLayerConstBytes;
            void *lcb = (lcb_bytes <= (256u << 20)) ? arena.alloc<double2>(lcb_bytes / 16) : nullptr;
            int64_t *plist = arena.alloc<int64_t>((size_t)R);
            CK(launch_smallc_prefix(sa, pst, pca, plist, lcb, st, dev));
            sa.pstart = pst;
            sa.pcarry = pca;
        }
        if (timed) CK(cudaEventRecord(slot[0], st));   // the scan kernels only
        if (models) {
            CK(launch_scan_models(sa, st, dev));
        } else if (pairs) {
            const size_t tb = pair_tail_scratch_bytes(sa, dev);
            void *tail = tb ? (void *)arena.alloc<double2>((tb + 15) / 16) : nullptr;
            CK(launch_scan_pairs(sa, tail, st, dev));
        } else {
            CK(launch_scan(sa, team, st, dev));
        }
        if (timed) {
            CK(cudaEventRecord(slot[1], st));
            ++t_scan_count;
        }
        if (dmis) CK(launch_misfit(dct, dce, M, L, dmis, ws, 0x7Fu | (stable ? kGridStable : 0u), true, st));

        if (!host && (ex.flags & MASW_ASYNC)) return MASW_OK;
        const Workspace w = read_status(ws, st);
        const int code = decode(w, dce != nullptr, true, stable);
        if (code < 0) return code;
        t_last_alg = (long long)w.alg_dets;
        t_last_eval = (long long)w.eval_dets;
        t_last_fb = (long long)w.fallback_dets;
        if (sa.pstart) {
            t_last_prefix_rows = (long long)w.prefix_rows;
            t_last_prefix_dets = (long long)w.prefix_dets;
        }
        if (stats) {
            t_team_dets.assign((size_t)nteams, 0);
            CK(cudaMemcpy(t_team_dets.data(), sa.team_dets, nteams * sizeof(long long),
                          cudaMemcpyDeviceToHost));
            t_team_count = nteams;
        }
        if (host) {
            CK(cudaMemcpyAsync(ct_out, dct, R * sizeof(double), cudaMemcpyDeviceToHost, st));
            if (idx_out)
                CK(cudaMemcpyAsync(idx_out, didx, R * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            if (misfit_out)
                CK(cudaMemcpyAsync(misfit_out, dmis, M * sizeof(double), cudaMemcpyDeviceToHost, st));
            wait_stream(st);
        }
        return code;
    } catch (const Fail &f) {
        return f.code;
    }
}

int run_misfit(const double *ct, const double *ce, int64_t M, int64_t L, double *out,
               const masw_exec *exp)
{
    if (!ct || !ce || !out || L < 1 || M < 0) return MASW_E_ARG;
    if (M == 0) return MASW_OK;
    const Exec ex = resolve(exp);
    int pdev = -1;
    const int kind = common_kind({ct, ce, out}, &pdev);
    if (kind < 0) return MASW_E_ARG;
    const bool host = (kind == 1);
    try {
        DeviceScope scope;
        scope.set(ex.device >= 0 ? ex.device : (host ? -1 : pdev));
        const cudaStream_t st = ex.stream;
        Arena arena(st);
        const double *dct = ct, *dce = ce;
        double *dout = out;
        if (host) {
            dct = arena.stage_in(ct, M * L);
            dce = arena.stage_in(ce, L);
            dout = arena.alloc<double>(M);
        }
        Workspace *ws = arena.alloc<Workspace>(1);
        CK(cudaMemsetAsync(ws, 0, sizeof(Workspace), st));
        CK(launch_validate_ce(dce, L, ws, st));
        CK(launch_misfit(dct, dce, M, L, dout, ws, 0x60u, false, st));
        if (!host && (ex.flags & MASW_ASYNC)) return MASW_OK;
        const Workspace w = read_status(ws, st);
        const int code = decode(w, true, false);
        if (code < 0) return code;
        if (host) {
            CK(cudaMemcpyAsync(out, dout, M * sizeof(double), cudaMemcpyDeviceToHost, st));
            wait_stream(st);
        }
        return MASW_OK;
    } catch (const Fail &f) {
        return f.code;
    }
}

// NVTX range around each C-ABI call (header-only NVTX v3; a no-op unless a tool attaches).
struct Range {
    explicit Range(const char *name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

}  // namespace

// ====================================================================== extern "C"
extern "C" {

int masw_curve(const masw_model *model, const double *lambda, int64_t L, const double *c,
               int64_t V, double *ct_out, int32_t *idx_out, const masw_exec *exec)
{
    Range nvtx_range("masw_curve");
    if (!model) return MASW_E_ARG;
    ModelArgs m{1, model->n_layers, model->h, model->alpha, model->beta, model->rho};
    return run_curves(m, lambda, L, c, V, nullptr, ct_out, idx_out, nullptr, exec);
}

int masw_curves_ensemble(const masw_ensemble *ens, const double *lambda, int64_t L,
                         const double *c, int64_t V, const double *ce, double *ct_out,
                         int32_t *idx_out, double *misfit_out, const masw_exec *exec)
{
    Range nvtx_range("masw_curves_ensemble");
    if (!ens) return MASW_E_ARG;
    ModelArgs m{ens->n_models, ens->n_layers, ens->h, ens->alpha, ens->beta, ens->rho};
    return run_curves(m, lambda, L, c, V, ce, ct_out, idx_out, misfit_out, exec);
}

int masw_misfit(const double *ct, const double *ce, int64_t L, double *misfit_out,
                const masw_exec *exec)
{
    Range nvtx_range("masw_misfit");
    return run_misfit(ct, ce, 1, L, misfit_out, exec);
}

int masw_misfit_batch(const double *ct, const double *ce, int64_t M, int64_t L,
                      double *misfit_out, const masw_exec *exec)
{
    Range nvtx_range("masw_misfit_batch");
    return run_misfit(ct, ce, M, L, misfit_out, exec);
}

int masw_argmin(const double *misfit, int64_t M, int64_t *best_out, double *best_misfit_out,
                const masw_exec *exp)
{
    Range nvtx_range("masw_argmin");
    if (!misfit || !best_out || M < 0) return MASW_E_ARG;
    if (M == 0) {
        int d = -1;
        if (classify(best_out, &d) == 2) {
            const long long neg = -1;
            if (cudaMemcpy(best_out, &neg, 8, cudaMemcpyHostToDevice) != cudaSuccess)
                return cuda_fail(cudaGetLastError(), "cudaMemcpy");
        } else {
            *best_out = -1;
        }
        return MASW_OK;
    }
    const Exec ex = resolve(exp);
    int pdev = -1;
    const int kind = common_kind({misfit, best_out, best_misfit_out}, &pdev);
    if (kind < 0) return MASW_E_ARG;
    const bool host = (kind == 1);
    try {
        DeviceScope scope;
        scope.set(ex.device >= 0 ? ex.device : (host ? -1 : pdev));
        const cudaStream_t st = ex.stream;
        Arena arena(st);
        const double *dm = misfit;
        int64_t *db = best_out;
        double *dv = best_misfit_out;
        if (host) {
            dm = arena.stage_in(misfit, M);
            db = arena.alloc<int64_t>(1);
            dv = arena.alloc<double>(1);
        }
        CK(launch_argmin(dm, M, db, dv, st));
        if (host) {
            CK(cudaMemcpyAsync(best_out, db, 8, cudaMemcpyDeviceToHost, st));
            if (best_misfit_out)
                CK(cudaMemcpyAsync(best_misfit_out, dv, 8, cudaMemcpyDeviceToHost, st));
            wait_stream(st);
        } else if (!(ex.flags & MASW_ASYNC)) {
            wait_stream(st);
        }
        return MASW_OK;
    } catch (const Fail &f) {
        return f.code;
    }
}

int masw_det_grid(const masw_model *model, const double *lambda, int64_t L, const double *c,
                  int64_t V, double *mant_re, double *mant_im, int32_t *exp2,
                  const masw_exec *exp)
{
    Range nvtx_range("masw_det_grid");
    if (!model || !model->h || !model->alpha || !model->beta || !model->rho || !lambda || !c ||
        !mant_re || !mant_im || !exp2)
        return MASW_E_ARG;
    if (L < 1 || V < 2 || V > INT32_MAX || model->n_layers < 1 ||
        model->n_layers > MASW_MAX_LAYERS || L > 65535)
        return MASW_E_ARG;
    const Exec ex = resolve(exp);
    int pdev = -1;
    const int kind = common_kind({model->h, model->alpha, model->beta, model->rho, lambda, c,
                                  mant_re, mant_im, exp2},
                                 &pdev);
    if (kind < 0) return MASW_E_ARG;
    const bool host = (kind == 1);
    try {
        DeviceScope scope;
        scope.set(ex.device >= 0 ? ex.device : (host ? -1 : pdev));
        const cudaStream_t st = ex.stream;
        Arena arena(st);
        const int64_t N = model->n_layers, G = L * V;
        ModelArgs mod{1, model->n_layers, model->h, model->alpha, model->beta, model->rho};
        const double *dlam = lambda, *dc = c;
        double *dre = mant_re, *dim = mant_im;
        int32_t *dex = exp2;
        if (host) {
            mod.h = arena.stage_in(model->h, N);
            mod.alpha = arena.stage_in(model->alpha, N + 1);
            mod.beta = arena.stage_in(model->beta, N + 1);
            mod.rho = arena.stage_in(model->rho, N + 1);
            dlam = arena.stage_in(lambda, L);
            dc = arena.stage_in(c, V);
            dre = arena.alloc<double>(G);
            dim = arena.alloc<double>(G);
            dex = arena.alloc<int32_t>(G);
        }
        Workspace *ws = arena.alloc<Workspace>(1);
        CK(cudaMemsetAsync(ws, 0, sizeof(Workspace), st));
        CK(launch_validate(mod, dlam, L, dc, V, nullptr, ws, st));
        const bool stable = (ex.flags & MASW_STABLE) != 0;
        CK(launch_det_grid(mod, dlam, L, dc, V, dre, dim, dex, ws, st, stable,
                           (ex.flags & MASW_DIRECT) == 0));
        if (!host && (ex.flags & MASW_ASYNC)) return MASW_OK;
        const Workspace w = read_status(ws, st);
        const int code = decode(w, false, true, stable);
        if (code < 0) return code;
        if (host) {
            CK(cudaMemcpyAsync(mant_re, dre, G * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(mant_im, dim, G * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(exp2, dex, G * 4, cudaMemcpyDeviceToHost, st));
            wait_stream(st);
        }
        return MASW_OK;
    } catch (const Fail &f) {
        return f.code;
    }
}

const char *masw_strerror(int code)
{
    switch (code) {
        case MASW_OK: return "MASW_OK";
        case MASW_WARN_NO_SIGN_CHANGE: return "MASW_WARN_NO_SIGN_CHANGE: some wavelength has no sign change (idx < 0)";
        case MASW_E_ARG: return "MASW_E_ARG: invalid argument";
        case MASW_E_MODEL: return "MASW_E_MODEL: model violates h>0, rho>0, beta>0, alpha>beta";
        case MASW_E_GRID: return "MASW_E_GRID: lambda <= 0, c0 <= 0 or c not strictly increasing";
        case MASW_E_RANGE: return "MASW_E_RANGE: 2*pi*h/lambda > 350 (700 with MASW_STABLE)";
        case MASW_E_NONFINITE: return "MASW_E_NONFINITE: NaN/Inf input";
        case MASW_E_CUDA: return "MASW_E_CUDA: CUDA runtime error";
        case MASW_E_NOMEM: return "MASW_E_NOMEM: device allocation failed";
        default: return "unknown masw status";
    }
}

int masw_version(void) { return MASW_ABI_VERSION; }

const char *masw_last_cuda_error(void) { return t_cuda_err; }

int64_t masw_kernel_launches(void) { return (int64_t)launches(); }

int masw_recent_scan_ms(double *ms_out, int32_t n)
{
    if (!ms_out || n < 0) return MASW_E_ARG;
    long long avail = t_scan_count < kScanRing ? t_scan_count : kScanRing;
    if (n > avail) n = (int32_t)avail;
    for (int32_t i = 0; i < n; ++i) {
        const long long k = t_scan_count - n + i;   // oldest first
        cudaEvent_t *slot = t_scan_ev[k % kScanRing];
        float ms = -1.0f;
        if (cudaEventSynchronize(slot[1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms, slot[0], slot[1]) != cudaSuccess) {
            cudaGetLastError();
            ms = -1.0f;
        }
        ms_out[i] = ms;
    }
    return n;
}

double masw_last_scan_ms(void)
{
    double ms = -1.0;
    return masw_recent_scan_ms(&ms, 1) == 1 ? ms : -1.0;
}

int64_t masw_last_team_dets(int64_t *out, int64_t n)
{
    if (t_team_count < 0) return -1;
    if (out)
        for (int64_t i = 0; i < n && i < t_team_count; ++i) out[i] = t_team_dets[(size_t)i];
    return t_team_count;
}

int64_t masw_last_fallbacks(void) { return t_last_fb; }

int masw_last_prefix(int64_t *rows, int64_t *dets)
{
    if (rows) *rows = t_last_prefix_rows;
    if (dets) *dets = t_last_prefix_dets;
    return (t_last_prefix_rows < 0) ? -1 : 0;
}

int masw_last_work(int64_t *algorithmic_dets, int64_t *evaluated_dets)
{
    if (algorithmic_dets) *algorithmic_dets = t_last_alg;
    if (evaluated_dets) *evaluated_dets = t_last_eval;
    return (t_last_alg < 0) ? -1 : 0;
}

}  // extern "C"
