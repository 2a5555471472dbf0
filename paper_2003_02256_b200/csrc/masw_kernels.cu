// masw_kernels.cu -- sm_100a kernels of libmasw.so.
//
//   validate_kernel   argument checks of include/masw.h on device-resident inputs
//   scan_kernel<TEAM> the hot path: persistent work-stealing kernel; a team of TEAM warps
//                     takes one (model, lambda) row at a time and scans c upward in chunks
//                     of 32*TEAM velocities; each lane assembles + eliminates one det in
//                     registers (masw_det.cuh), signs are compared across lanes with
//                     shuffles, the first change is found with a warp ballot (+ a shared-
//                     memory min across the team's warps), and the team exits the row at
//                     the first chunk that contains a change (Algorithm 1).
//   misfit_kernel     Algorithm 2, one warp per model, fixed-order
//                     butterfly sum (deterministic, independent of sharding).
//   argmin_kernel     lowest misfit, ties -> lowest index.
//   det_grid_kernel   debug/parity: every (lambda, c) det with mantissa/exponent.
//
// What differs from the paper's GPU design and why is in DESIGN.md:
// no stiffness matrices in global memory, no separate assemble / eliminate / search / reduce
// kernels, early exit instead of evaluating the whole grid, a work queue for
// the load imbalance the paper repartitions for.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "masw_det.cuh"
#include "masw_internal.h"

namespace masw {

namespace {
std::atomic<long long> g_launches{0};
constexpr unsigned FULL = 0xffffffffu;
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launches() { return g_launches.load(std::memory_order_relaxed); }

// ------------------------------------------------------------------ validation

__device__ __forceinline__ bool ws_range_bad(const Workspace *ws, bool stable)
{
    // max_i,e fl(fl(2pi/lambda_i) * h_e) = fl(fl(2pi/lambda_min) * h_max): both roundings are
    // monotone, so this is exactly the per-pair guard of include/masw.h (350, or 700 for the
    // scaled elements of MASW_STABLE).
    const double lam_min = __longlong_as_double((long long)~ws->lam_min_nbits);
    const double h_max = __longlong_as_double((long long)ws->h_max_bits);
    const double kmax = kTwoPi / lam_min;
    return kmax * h_max > (stable ? kMaxKHStable : kMaxKH);
}

// max over the call's rows and layers of k h_e (validated: <= 350)
__device__ __forceinline__ double ws_kh_max(const Workspace *ws)
{
    const double lam_min = __longlong_as_double((long long)~ws->lam_min_nbits);
    const double h_max = __longlong_as_double((long long)ws->h_max_bits);
    return (kTwoPi / lam_min) * h_max;
}
// -> rows of the cosh/sinh table the call can reach
template <class TabT = unsigned>
__device__ __forceinline__ int ws_exp_rows(const Workspace *ws)
{
    return exp_rows_needed<TabT>(ws_kh_max(ws));
}
// the call's direct elements take the fine cosh/sinh table (FineTab, masw_det.cuh)
__device__ __forceinline__ bool ws_fine(const Workspace *ws)
{
    return ws_kh_max(ws) <= kFineKhMax;
}

// grid_mask selects which grid_err bits make the call invalid.
__device__ __forceinline__ bool ws_invalid(const Workspace *ws, unsigned grid_mask,
                                           bool check_models)
{
    if (ws->grid_err & grid_mask) return true;
    if (check_models) {
        if (ws->model_err != 0ull) return true;
        if (ws_range_bad(ws, (grid_mask & kGridStable) != 0)) return true;
    }
    return false;
}

__global__ void validate_kernel(ModelArgs m, const double *__restrict__ lam, int64_t L,
                                const double *__restrict__ c, int64_t V,
                                const double *__restrict__ ce, Workspace *ws)
{
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned gerr = 0;
    double lmin = INFINITY, hmax = 0.0;
    if (lam) {
        for (int64_t i = tid; i < L; i += stride) {
            const double x = lam[i];
            if (!isfinite(x)) gerr |= 1u;
            else if (!(x > 0.0)) gerr |= 4u;
            else lmin = fmin(lmin, x);
        }
    }
    if (c) {
        for (int64_t j = tid; j < V; j += stride) {
            const double x = c[j];
            if (!isfinite(x)) {
                gerr |= 2u;
            } else {
                if (j == 0 && !(x > 0.0)) gerr |= 8u;
                if (j > 0 && !(x > c[j - 1])) gerr |= 16u;
            }
        }
    }
    if (ce) {
        for (int64_t i = tid; i < L; i += stride) {
            const double x = ce[i];
            if (!isfinite(x)) gerr |= 32u;
            else if (!(x > 0.0)) gerr |= 64u;
        }
    }
    const int N = m.N;
    for (int64_t k = tid; k < m.M; k += stride) {
        bool nonfinite = false, bad = false;
        for (int e = 0; e < N; ++e) {
            const double h = m.h[k * N + e];
            nonfinite |= !isfinite(h);
            bad |= !(h > 0.0);
            if (isfinite(h)) hmax = fmax(hmax, h);
        }
        for (int e = 0; e <= N; ++e) {
            const double a = m.alpha[k * (N + 1) + e], b = m.beta[k * (N + 1) + e],
                         r = m.rho[k * (N + 1) + e];
            nonfinite |= !isfinite(a) || !isfinite(b) || !isfinite(r);
            bad |= !(r > 0.0) || !(b > 0.0) || !(a > b);
        }
        const unsigned cls = nonfinite ? kModelNonfinite : (bad ? kModelBad : 0u);
        if (cls) atomicMax(&ws->model_err, ~(((unsigned long long)k << 2) | cls));
    }
    if (gerr) atomicOr(&ws->grid_err, gerr);
    if (lmin < INFINITY)
        atomicMax(&ws->lam_min_nbits, ~(unsigned long long)__double_as_longlong(lmin));
    if (hmax > 0.0) atomicMax(&ws->h_max_bits, (unsigned long long)__double_as_longlong(hmax));
}

cudaError_t launch_validate(const ModelArgs &m, const double *lam, int64_t L, const double *c,
                            int64_t V, const double *ce, Workspace *ws, cudaStream_t st)
{
    int64_t n = m.M;
    if (L > n) n = L;
    if (V > n) n = V;
    int blocks = (int)((n + 255) / 256);
    if (blocks < 1) blocks = 1;
    if (blocks > 1184) blocks = 1184;
    validate_kernel<<<blocks, 256, 0, st>>>(m, lam, L, c, V, ce, ws);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_validate_ce(const double *ce, int64_t L, Workspace *ws, cudaStream_t st)
{
    ModelArgs none{0, 1, nullptr, nullptr, nullptr, nullptr};
    return launch_validate(none, nullptr, L, nullptr, 0, ce, ws, st);
}

// ------------------------------------------------------------------ small-c prefix (S15'')
__device__ __forceinline__ unsigned long long warp_sum_u64_pre(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Reading S15'': at very low c the direct App. A element cancels; the relative
// rounding error of an fp64 det K is of the order of
//   P(c, k) = u max_e [16 (beta_e/c)^4 + (alpha_e beta_e / c^2)^2 / (k h_e)^4].
// Every det with P > tau -- i.e. c_j^4 < Q_r = (u/tau) max_e [16 beta_e^4 + (alpha_e beta_e)^2
// / (k h_e)^4], a PREFIX of each row's ascending grid -- is evaluated with the cancellation-
// free stable element (f3) by this kernel, before the scan; the scans evaluate the rest with
// the direct element.  The rule depends only on (model, lambda, c_j), so every scan gives the
// same result.  C5 (tau = 1e-3): ~1/3 of the rows have a prefix of 1-6 grid points (2.2e6 of
// 1.03e9 dets), so the prefix dets are PACKED 32 to a warp pass (each warp takes 32 rows,
// lays their prefix dets out contiguously and evaluates them in ceil(T / 32) passes) -- the
// row-wise alternative (one row's 1-6 dets per warp pass) would idle 26-31 lanes.
constexpr double kSmallCTau = 1e-3;
constexpr double kSmallCScale = 0x1p-53 / kSmallCTau;

// Q_r = s max_e (a_e + b_e / k^4) with a_e = 16 beta_e^4, b_e = (alpha_e beta_e / h_e^2)^2,
// s = u / tau (e < N: the finite layers).  a_e, b_e depend on the model only; every user
// (smallc_rows_kernel, det_grid_kernel) forms them and Q with these same operations, so the
// prefix rule is bitwise the same everywhere.
__device__ __forceinline__ void smallc_ab(double al, double be, double h, double &a, double &b)
{
    const double b2 = be * be;
    a = (16.0 * b2) * b2;
    const double t = (al * be) / (h * h);
    b = t * t;
}

__device__ __forceinline__ double smallc_ik4(double k)
{
    const double kk = k * k;
    return 1.0 / (kk * kk);
}

// Q_r of model m at wavenumber k (global-memory model arrays; det_grid_kernel)
__device__ __forceinline__ double smallc_q(const ModelArgs &mod, int64_t m, double k)
{
    const int N = mod.N;
    const double ik4 = smallc_ik4(k);
    double worst = 0.0;
    for (int e = 0; e < N; ++e) {
        double a, b;
        smallc_ab(mod.alpha[m * (N + 1) + e], mod.beta[m * (N + 1) + e], mod.h[m * N + e], a, b);
        worst = fmax(worst, fma(b, ik4, a));
    }
    return kSmallCScale * worst;
}

// LayerConst of layer e of model m at wavenumber k, formed exactly as the row scan forms it
// (K / k constants: rho, rho beta^2; only k h carries the wavelength).
__device__ __forceinline__ LayerConst row_layer_const(const ModelArgs &mod, int64_t m, int e,
                                                      double k)
{
    const int N = mod.N;
    const double al = mod.alpha[m * (N + 1) + e];
    const double be = mod.beta[m * (N + 1) + e];
    const double rh = mod.rho[m * (N + 1) + e];
    LayerConst x;
    x.kh = (e < N) ? k * mod.h[m * N + e] : 0.0;
    x.ia2 = 1.0 / (al * al);
    x.ib2 = 1.0 / (be * be);
    x.krho = rh;
    x.b2 = 2.0 * (be * be);
    x.aux = (e < N) ? rh / mod.rho[m * (N + 1) + e + 1] : (rh * (be * be)) / mod.rho[m * (N + 1) + N - 1];
    return x;
}

// sgn Re det K (2: non-finite) of model m at (k, c') with the stable element: the certified
// block recursion, the banded GEPP where it is not certified (or always, MASW_PIVOTED) --
// what the row scan computes under MASW_STABLE.  lcm: the model's k-free LayerConst[N + 1]
// (kh field = h; smallc_rows_kernel's cache, bitwise what row_layer_const forms), or nullptr
// (formed from the model arrays per element).
static __device__ __noinline__ int prefix_det_sign(ModelArgs mod, int64_t m, double k, double c,
                                                   unsigned tab, bool pivoted,
                                                   const LayerConst *lcm)
{
    const int N = mod.N;
    const double c2 = c * c;
    auto lc = [&](int e) {
        if (lcm) {
            LayerConst x = load_lc(lcm + e);
            x.kh = (e < N) ? k * x.kh : 0.0;
            return x;
        }
        return row_layer_const(mod, m, e, k);
    };
    if (!pivoted) {
        const double ic2 = rcp_fast(c2);
        const SignOut so = det_sign_block_u<1>(
            N, [&](int e) { return layer_elemu_stable(lc(e), c2, ic2, tab); },
            [&] {
                const LayerConst H = lc(N);
                return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), H.aux * ic2);
            });
        if (so.ok) return so.sign;
    }
    const DetOut d = det_core<false, 0, 1>(
        N, [&](int e) { return layer_elem_stable(lc(e), c2, tab); },
        [&] {
            const LayerConst H = lc(N);
            return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), lc_mu(H));
        });
    return d.bad ? 2 : d.sign;
}

// the S4-perturbed velocity of model m (layer velocities read from global memory)
__device__ __forceinline__ double perturb_model(const ModelArgs &mod, int64_t m, double c)
{
    const int N = mod.N;
    for (;;) {
        bool near = false;
        for (int e = 0; e <= N; ++e)
            near |= (fabs(c - mod.alpha[m * (N + 1) + e]) < kPerturbTol) |
                    (fabs(c - mod.beta[m * (N + 1) + e]) < kPerturbTol);
        if (!near) return c;
        c = c * kPerturbFactor;
    }
}

constexpr int kPrefixBlock = 256;

// Pass 1: a CTA takes a tile of 256 PER consecutive output rows q = m L + i, a thread PER of
// them (strided by 256, so every store is coalesced and each thread has PER independent
// chains in flight; PER = 8 for large calls, 1 when that leaves the GPU short of CTAs -- a
// single 10k-wavelength curve ran in 5 CTAs of 8-row threads, 30 us under ncu).  The per-layer terms a_e, b_e of Q_r (smallc_ab: one IEEE
// division each) are formed once per (model, layer) of the tile in shared memory when they
// fit (C5: ~52 models per tile), else per row.  n = #{j : c_j^4 < Q_r} (reading S15'') -- a
// short linear probe, then bisection -- goes to pstart[q] (pass 2 replaces it) with
// pcarry[q] = 0; ws->prefix_rows counts the rows with n > 0 (one reduction per CTA).  The CTA
// also writes the k-free LayerConst[N + 1] of each model whose first row it holds to `lcbuf`
// (if given) for pass 2.  (No validation check: on an invalid call the values are garbage
// but every access stays in bounds, and pass 2 and the scans return without using them.)
constexpr int kPrefixPerThread = 8;   // PER of large calls
constexpr int kPrefixAbMax = 1024;   // (a_e, b_e) pairs staged per CTA (16 KB)

template <int PER>
__global__ void __launch_bounds__(kPrefixBlock) smallc_rows_kernel(ScanArgs a, int32_t *pstart,
                                                                   int8_t *pcarry, int64_t *list,
                                                                   LayerConst *lcbuf)
{
    __shared__ double2 s_ab[kPrefixAbMax];
    constexpr int kPrefixTile = kPrefixBlock * PER;
    __shared__ double s_ik4[kPrefixTile];
    __shared__ unsigned s_off[PER][kPrefixBlock / 32];
    __shared__ unsigned long long s_base;
    const int N = a.mod.N;
    const int64_t M = a.mod.M, L = a.L, V = a.V, R = M * L;
    const double *__restrict__ cg = a.c;
    const int64_t q0 = (int64_t)blockIdx.x * kPrefixTile;
    // the tile's models m_lo .. m_hi (q - m_lo L < kPrefixTile + L < 2^32: 32-bit divisions)
    const int64_t m_lo = q0 / L;
    const unsigned span = (unsigned)(min(q0 + kPrefixTile, R) - 1 - m_lo * L);
    const unsigned nmod = span / (unsigned)L + 1u;
    const bool staged = nmod * (unsigned)N <= (unsigned)kPrefixAbMax;
    // 1/k^4 of the tile's wavelengths i_lo .. i_lo + ni - 1 (one model: a contiguous range;
    // several: all L of them when L fits), else per row
    const unsigned i_lo = (nmod == 1u) ? (unsigned)(q0 - m_lo * L) : 0u;
    const unsigned ni = (nmod == 1u) ? span - i_lo + 1u : (L <= kPrefixTile ? (unsigned)L : 0u);
    for (unsigned t = threadIdx.x; t < ni; t += kPrefixBlock)
        s_ik4[t] = smallc_ik4(kTwoPi / a.lam[i_lo + t]);      // reading S2
    if (staged) {
        for (unsigned t = threadIdx.x; t < nmod * (unsigned)N; t += kPrefixBlock) {
            const unsigned tm = t / (unsigned)N;
            const int e = (int)(t - tm * (unsigned)N);
            const int64_t mm = m_lo + tm;
            double x, y;
            smallc_ab(a.mod.alpha[mm * (N + 1) + e], a.mod.beta[mm * (N + 1) + e],
                      a.mod.h[mm * N + e], x, y);
            s_ab[t] = make_double2(x, y);
        }
    }
    if (lcbuf) {   // models whose first row lies in this tile
        for (unsigned t = threadIdx.x; t < nmod * (unsigned)(N + 1); t += kPrefixBlock) {
            const unsigned tm = t / (unsigned)(N + 1);
            const int e = (int)(t - tm * (unsigned)(N + 1));
            const int64_t mm = m_lo + tm;
            if (mm * L < q0) continue;
            LayerConst x = row_layer_const(a.mod, mm, e, 1.0);
            x.kh = (e < N) ? a.mod.h[mm * N + e] : 0.0;     // k-free: pass 2 forms k h
            lcbuf[mm * (N + 1) + e] = x;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned mk[PER];   // per slab u: the warp's rows with n > 0
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int64_t q = q0 + u * kPrefixBlock + threadIdx.x;
        int n = 0;
        if (q < R) {
            const unsigned rq = (unsigned)(q - m_lo * L);
            const unsigned dm = rq / (unsigned)L;
            const int64_t m = m_lo + dm;
            const unsigned i = rq - dm * (unsigned)L;
            const double ik4 = ni ? s_ik4[i - i_lo] : smallc_ik4(kTwoPi / a.lam[i]);   // reading S2
            double worst = 0.0;
            if (staged) {
                const double2 *ab = s_ab + dm * (unsigned)N;
                for (int e = 0; e < N; ++e) worst = fmax(worst, fma(ab[e].y, ik4, ab[e].x));
            } else {
                for (int e = 0; e < N; ++e) {
                    double x, y;
                    smallc_ab(a.mod.alpha[m * (N + 1) + e], a.mod.beta[m * (N + 1) + e],
                              a.mod.h[m * N + e], x, y);
                    worst = fmax(worst, fma(y, ik4, x));
                }
            }
            const double Q = kSmallCScale * worst;
            auto below = [&](int64_t j) {
                const double c2 = cg[j] * cg[j];
                return c2 * c2 < Q;
            };
            if (below(0)) {                                       // first j with c_j^4 >= Q
                int64_t lo = 1;
                while (lo < V && lo < 8 && below(lo)) ++lo;      // prefixes are short (C5: 1-6)
                if (lo == 8 && lo < V && below(lo)) {
                    int64_t hi = V;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (below(mid)) lo = mid + 1; else hi = mid;
                    }
                }
                n = (int)lo;
            }
            pstart[q] = n;
            pcarry[q] = 0;
        }
        mk[u] = __ballot_sync(FULL, n > 0);
        if (lane == 0) s_off[u][warp] = __popc(mk[u]);
    }
    // the tile's rows with n > 0 go to `list` in row order (u-major, then warp, then lane):
    // one exclusive scan over the (u, warp) counts and one global atomic per CTA
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int u = 0; u < PER; ++u)
            for (int w = 0; w < kPrefixBlock / 32; ++w) {
                const unsigned t = s_off[u][w];
                s_off[u][w] = tot;
                tot += t;
            }
        s_base = tot ? atomicAdd(&a.ws->prefix_rows, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u)
        if ((mk[u] >> lane) & 1u)
            list[s_base + s_off[u][warp] + __popc(mk[u] & ((1u << lane) - 1u))] =
                q0 + u * kPrefixBlock + threadIdx.x;
}

// Pass 2: the listed rows' prefix determinants with the stable element.  The prefixes are
// short (C5: 1-6 grid points), so they are PACKED 32 to a warp pass: each warp takes 32 listed
// rows, lays their prefix dets out contiguously and evaluates them in ceil(T / 32) passes
// (C5: ~52 dets per 32 rows, 2 passes at ~80 % of the lanes) -- one row's 1-6 dets per warp
// pass would idle 26-31 lanes.  Writes pstart (first index the scan evaluates, or -1 when the
// row's first change lies in the prefix / the whole grid is prefix) and pcarry (the sign at
// pstart - 1), and the outputs of the rows finished here.
__global__ void __launch_bounds__(kPrefixBlock, 2) smallc_prefix_kernel(ScanArgs a, int32_t *pstart,
                                                                        int8_t *pcarry,
                                                                        const int64_t *list,
                                                                        const LayerConst *lcbuf)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_abort;
    Workspace *ws = a.ws;
    if (threadIdx.x == 0) s_abort = ws_invalid(ws, a.grid_mask, true) || ws->prefix_rows == 0ull;
    __syncthreads();
    if (s_abort) return;
    const int64_t nlist = (int64_t)ws->prefix_rows;
    exp_scale_fill(smem, ws_exp_rows(ws));
    __syncthreads();
    const unsigned ta = opaque(smem_addr(smem));

    const int lane = threadIdx.x & 31;
    const int64_t L = a.L, V = a.V;
    const double *__restrict__ cg = a.c;
    const int64_t nwarps = (int64_t)gridDim.x * (kPrefixBlock / 32);
    struct {
        unsigned long long alg, eval;
        unsigned status;
    } acc{0ull, 0ull, 0u};
    for (int64_t b = (int64_t)blockIdx.x * (kPrefixBlock / 32) + (threadIdx.x >> 5); b * 32 < nlist;
         b += nwarps) {
        const bool valid = b * 32 + lane < nlist;
        const int64_t q = valid ? list[b * 32 + lane] : 0;
        const int64_t n = valid ? (int64_t)pstart[q] : 0;
        int64_t m, i;
        if (q < 0x80000000ll && L < 0x80000000ll) {   // 32-bit division where it fits
            const unsigned mq = (unsigned)q / (unsigned)L;
            m = mq;
            i = (int64_t)((unsigned)q - mq * (unsigned)L);
        } else {
            m = q / L;
            i = q - m * L;
        }
        const double k = kTwoPi / a.lam[i];                       // reading S2
        // pack the rows' prefix dets: row o's dets are tasks excl_o .. excl_o + n_o - 1
        int64_t excl = n;
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(FULL, excl, o);
            if (lane >= o) excl += t;
        }
        const int64_t T = __shfl_sync(FULL, excl, 31);
        excl -= n;
        bool done = false, fbad = false;
        int64_t fj = -1;
        int prev = 0;   // sign of the previous task (across passes)
        for (int64_t t0 = 0; t0 < T; t0 += 32) {
            const int64_t t = t0 + lane;
            const bool act = t < T;
            int o = 0;   // owner: the last lane with excl <= t (it has n > 0 when t < T)
        #pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int64_t e = __shfl_sync(FULL, excl, o + step);
                if (e <= t) o += step;
            }
            const int64_t jj = t - __shfl_sync(FULL, excl, o);
            const int64_t mo = __shfl_sync(FULL, m, o);
            const int64_t qo = __shfl_sync(FULL, q, o);
            const double ko = __shfl_sync(FULL, k, o);
            const int64_t no = __shfl_sync(FULL, n, o);
            int s = 0;
            bool bad = false;
            if (act) {
                const double cp = perturb_model(a.mod, mo, cg[jj]);
                const int r = prefix_det_sign(a.mod, mo, ko, cp, ta, a.pivoted != 0,
                                              lcbuf ? lcbuf + mo * (a.mod.N + 1) : nullptr);
                bad = (r == 2);
                s = bad ? 0 : r;
                if (jj == no - 1) pcarry[qo] = (int8_t)s;   // the scan's carried sign
            }
            int sp = __shfl_up_sync(FULL, s, 1);
            if (lane == 0) sp = prev;
            prev = __shfl_sync(FULL, s, 31);
            const bool ev = act && jj > 0 && (bad || s != sp);
            for (unsigned mk = __ballot_sync(FULL, ev); mk; mk &= mk - 1) {
                const int src = __ffs(mk) - 1;     // task order = (row, j) order
                const int ob = __shfl_sync(FULL, o, src);
                const int64_t jb = __shfl_sync(FULL, jj, src);
                const bool bb = __shfl_sync(FULL, (int)bad, src) != 0;
                if (lane == ob && !done) {
                    done = true;
                    fj = jb;
                    fbad = bb;
                }
            }
        }
        acc.eval += (lane == 0) ? (unsigned long long)T : 0ull;
        if (valid) {
            if (done) {                       // first change inside the prefix (Algorithm 1)
                pstart[q] = -1;
                if (fbad) {
                    a.ct[q] = __longlong_as_double(0x7ff8000000000000ll);
                    if (a.idx) a.idx[q] = -2;
                    acc.status |= 2u;
                } else {
                    a.ct[q] = cg[fj];
                    if (a.idx) a.idx[q] = (int32_t)fj;
                }
                acc.alg += (unsigned long long)(fj + 1);
            } else if (n >= V) {              // the whole grid was the prefix: no change
                pstart[q] = -1;
                a.ct[q] = __longlong_as_double(0x7ff8000000000000ll);
                if (a.idx) a.idx[q] = -1;
                acc.status |= 1u;
                acc.alg += (unsigned long long)V;
            }                                 // else: the scan starts at n (carry written above)
        }
    }
    const unsigned long long my_alg = warp_sum_u64_pre(acc.alg);
    const unsigned long long my_eval = warp_sum_u64_pre(acc.eval);
    const unsigned my_status = __reduce_or_sync(FULL, acc.status);
    if (lane == 0) {
        if (my_alg) atomicAdd(&ws->alg_dets, my_alg);
        if (my_eval) {
            atomicAdd(&ws->eval_dets, my_eval);
            atomicAdd(&ws->prefix_dets, my_eval);
        }
        if (my_status) atomicOr(&ws->row_status, my_status);
    }
}

// ------------------------------------------------------------------ scan

template <int TEAM, int BLOCK>
__device__ __forceinline__ void team_sync(int team)
{
    if constexpr (TEAM == 1) {
        __syncwarp();
    } else if constexpr (TEAM * 32 == BLOCK) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TEAM * 32) : "memory");
    }
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Shared memory: per team a control block then the row's LayerConst[N+1] and the
// 2(N+1) layer velocities used by the perturbation rule.
struct TeamCtrl {
    long long row;
    int first[2][32];
    int last[2][32];
};

__host__ __device__ constexpr unsigned round16(unsigned x) { return (x + 15u) & ~15u; }

__host__ __device__ inline unsigned team_model_bytes(int N)
{
    return round16((unsigned)(N + 1) * (unsigned)sizeof(LayerConst) +
                   2u * (unsigned)(N + 1) * (unsigned)sizeof(double));
}

// Resident CTAs per SM requested from ptxas for 256-thread CTAs: 2 (<= 128 registers; the
// kernel needs 122 without spills).  Measured on B200 with the current kernel: equal to the
// 3-CTA / 80-register build on C5 and ~5% faster on C3/C4 (the 3-CTA build spills ~100 B;
// it was the better choice before the elementary functions were trimmed).
// -DMASW_SCAN_MINB=k overrides it (0 = unconstrained).
#ifndef MASW_SCAN_MINB
#define MASW_SCAN_MINB 2
#endif
template <int BLOCK>
constexpr int scan_min_blocks()
{
    return BLOCK == 256 ? MASW_SCAN_MINB : 1;
}

// Sign of det K by the banded GEPP for one lane whose block-recursion sign was not certified
// (det_sign_block); out of line so the hot loop's code stays small.  Returns -1/0/+1, or 2
// for a non-finite determinant.
#ifndef MASW_BLOCK_SIGN
#define MASW_BLOCK_SIGN 1
#endif
template <bool STABLE, class TabT>
static __device__ __noinline__ int row_det_gepp(const LayerConst *lc, const double *vel,
                                                TabT ta, int N, double c)
{
    const DetOut d = det_K<false, 0, STABLE>(lc, vel, ta, N, c, false);
    return d.bad ? 2 : d.sign;
}

template <int TEAM, int BLOCK, bool STABLE, class TabT>
__device__ __forceinline__ void scan_kernel_body(ScanArgs a)
{
    constexpr int TEAMS = BLOCK / (32 * TEAM);
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_abort;

    const int N = a.mod.N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int team = warp / TEAM, wt = warp % TEAM, tl = wt * 32 + lane;

    // dynamic shared memory: [cosh/sinh scale table | team controls | per-team row constants]
    unsigned char *tab = smem;
    TeamCtrl *ctrl = reinterpret_cast<TeamCtrl *>(smem + kExpTabBytes) + team;
    const unsigned moff = kExpTabBytes + round16((unsigned)sizeof(TeamCtrl) * TEAMS) +
                          (unsigned)team * team_model_bytes(N);
    LayerConst *lc = reinterpret_cast<LayerConst *>(smem + moff);
    double *vel = reinterpret_cast<double *>(smem + moff + (unsigned)(N + 1) * sizeof(LayerConst));

    Workspace *ws = a.ws;
    if (threadIdx.x == 0) {
        const bool bad = ws_invalid(ws, a.grid_mask, true);
        s_abort = bad;
        if (bad && blockIdx.x == 0) ws->abort = 1;
    }
    __syncthreads();
    if (s_abort) return;
    exp_scale_fill<TabT>(tab, ws_exp_rows<TabT>(ws));
    __syncthreads();
    const TabT ta = TabTraits<TabT>::make(opaque(smem_addr(tab)));
    // rows with a small-c prefix (reading S15''; smallc_prefix_kernel ran before this kernel)
    const bool prefix = a.pstart != nullptr && ws->prefix_rows != 0ull;

    const int64_t M = a.mod.M, L = a.L, V = a.V;
    const int64_t rows = M * L;
    const double *__restrict__ cg = a.c;
    unsigned long long my_alg = 0, my_eval = 0, team_alg = 0, my_fb = 0;
    unsigned my_status = 0;
    int buf = 0;
    // static schedules (the paper's partitions): team g of G takes a
    // contiguous block of rows, or rows g, g+G, g+2G, ...
    const long long G = (long long)gridDim.x * TEAMS;
    const long long g = (long long)blockIdx.x * TEAMS + team;
    const long long cbase = rows / G, cextra = rows % G;
    const long long clo = g * cbase + (g < cextra ? g : cextra);
    const long long chi = clo + cbase + (g < cextra ? 1 : 0);
    long long kth = 0;

    for (;;) {
        // ---- next row: work-stealing queue (default; rows i-major so long wavelengths go
        //      first when lambda is given in the usual decreasing order) or a
        //      static schedule
        long long row;
        if (a.sched == 1) {
            row = clo + kth;
            if (row >= chi) row = rows;
            ++kth;
        } else if (a.sched == 2) {
            row = g + kth * G;
            ++kth;
        } else if constexpr (TEAM == 1) {
            if (lane == 0) row = (long long)atomicAdd(&ws->queue, 1ull);
            row = __shfl_sync(FULL, row, 0);
        } else {
            if (tl == 0) ctrl->row = (long long)atomicAdd(&ws->queue, 1ull);
            team_sync<TEAM, BLOCK>(team);
            row = ctrl->row;
        }
        if (row >= rows) break;
        const int64_t i = row / M, m = row - i * M;

        // ---- per-row constants into shared memory (reading S2: k = 2 pi / lambda)
        const double k = kTwoPi / a.lam[i];
        for (int e = tl; e <= N; e += 32 * TEAM) {
            const double al = a.mod.alpha[m * (N + 1) + e];
            const double be = a.mod.beta[m * (N + 1) + e];
            const double rh = a.mod.rho[m * (N + 1) + e];
            LayerConst x;
            // K / k (every entry of K is k times a function of k h and c, so det K =
            // k^(2(N+1)) det(K/k): same sign).  The scans use these k-free constants; only
            // k h carries the wavelength (det_grid_kernel, which returns values, keeps k).
            x.kh = (e < N) ? k * a.mod.h[m * N + e] : 0.0;
            x.ia2 = 1.0 / (al * al);
            x.ib2 = 1.0 / (be * be);
            x.krho = rh;
            x.b2 = 2.0 * (be * be);
            // f-free sign recursion (BlockSignU): rho_e / rho_(e+1); half-space: mu' factor
            x.aux = (e < N) ? rh / a.mod.rho[m * (N + 1) + e + 1]
                            : (rh * (be * be)) / a.mod.rho[m * (N + 1) + N - 1];
            lc[e] = x;
            vel[2 * e] = al;
            vel[2 * e + 1] = be;
        }
        team_sync<TEAM, BLOCK>(team);

        // ---- the row's small-c prefix (reading S15''): grid points below jstart were
        //      evaluated with the stable element by smallc_prefix_kernel (sign pcs at
        //      jstart - 1); jstart = -1: the row was finished there
        int64_t jstart = 0;
        int pcs = 0;
        if (prefix) {
            const int st = a.pstart[m * L + i];
            if (st < 0) continue;
            jstart = st;
            pcs = a.pcarry[m * L + i];
        }

        // ---- ascending scan in chunks of 32*TEAM velocities
        int carry = pcs;
        bool found = false;
        for (int64_t base = (jstart / (32 * TEAM)) * (32 * TEAM); base < V; base += 32 * TEAM) {
            const int64_t j = base + tl;
            // Reading S4 without a per-lane loop over all 2(N+1) layer velocities: the grid is
            // strictly increasing, so only velocities inside this warp's range [c_lo, c_hi]
            // (+-1e-3) can be within 1e-4 of a lane's c.  The warp ballots them (usually none,
            // rarely one or two); a lane tests just those, and only a lane that IS within 1e-4
            // of one runs the full S4 loop (exact: its perturbed c' may approach any velocity).
            const int nv = 2 * (N + 1);
            double c = 0.0;
            if (j < V) c = cg[j];
            {
                const int64_t w0 = base + wt * 32;
                const double clo = cg[min(w0, V - 1)] - 1e-3;
                const double chi = cg[min(w0 + 31, V - 1)] + 1e-3;
                bool lane_near = false;
                for (int e0 = 0; e0 < nv; e0 += 32) {
                    bool in = false;
                    if (e0 + lane < nv) {
                        const double v = vel[e0 + lane];
                        in = (v > clo) && (v < chi);
                    }
                    for (unsigned b = __ballot_sync(FULL, in); b; b &= b - 1)
                        lane_near |= fabs(c - vel[e0 + __ffs(b) - 1]) < kPerturbTol;
                }
                if (lane_near) c = perturb_velocity(vel, nv, c);
            }
            int s = 0;
            bool bad = false;
            if (j < jstart) {
                s = pcs;   // evaluated by the small-c prefix (no change there)
            } else if (j < V) {
#if MASW_BLOCK_SIGN
                const double c2 = c * c;
                SignOut so;
                so.ok = false;
                if (!a.pivoted) {
                    if constexpr (STABLE) {
                        const double ic2 = rcp_fast(c2);
                        so = det_sign_block_u<MASW_LAYER_UNROLL>(
                            N, [&](int e) { return layer_elemu_stable(load_lc(lc + e), c2, ic2, ta); },
                            [&] {
                                const LayerConst H = load_lc(lc + N);
                                return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), H.aux * ic2);
                            });
                    } else {
                        const double ic2 = rcp_fast(c2);
                        so = det_sign_block_u<MASW_LAYER_UNROLL>(
                            N, [&](int e) { return layer_elem_u(load_lc(lc + e), c2, ic2, ta); },
                            [&] {
                                const LayerConst H = load_lc(lc + N);
                                return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), H.aux * ic2);
                            });
                    }
                }
                if (so.ok) {
                    s = so.sign;
                } else {
                    const int r = row_det_gepp<STABLE>(lc, vel, ta, N, c);
                    bad = (r == 2);
                    s = bad ? 0 : r;
                    my_fb += a.pivoted ? 0 : 1;
                }
#else
                const DetOut d = det_K<false, 0, STABLE>(lc, vel, ta, N, c, false);
                s = d.sign;
                bad = d.bad;
#endif
                ++my_eval;
            }
            int sprev = __shfl_up_sync(FULL, s, 1);
            int64_t first = -1;
            if constexpr (TEAM == 1) {
                if (lane == 0) sprev = carry;
                const bool ev = (j < V) && (bad || (j > 0 && s != sprev));
                const unsigned mask = __ballot_sync(FULL, ev);
                if (mask) first = base + (__ffs(mask) - 1);
                carry = __shfl_sync(FULL, s, 31);
            } else {
                if (lane == 31) ctrl->last[buf][wt] = s;
                team_sync<TEAM, BLOCK>(team);
                if (lane == 0) sprev = (wt == 0) ? carry : ctrl->last[buf][wt - 1];
                const bool ev = (j < V) && (bad || (j > 0 && s != sprev));
                const unsigned mask = __ballot_sync(FULL, ev);
                if (lane == 0) ctrl->first[buf][wt] = mask ? wt * 32 + (__ffs(mask) - 1) : INT_MAX;
                team_sync<TEAM, BLOCK>(team);
                int f = INT_MAX;
#pragma unroll
                for (int w = 0; w < TEAM; ++w) f = min(f, ctrl->first[buf][w]);
                if (f != INT_MAX) first = base + f;
                carry = ctrl->last[buf][TEAM - 1];
                buf ^= 1;
            }
            if (first >= 0) {
                if (j == first) {
                    const int64_t o = m * L + i;
                    if (bad) {
                        a.ct[o] = __longlong_as_double(0x7ff8000000000000ll);
                        if (a.idx) a.idx[o] = -2;
                        my_status |= 2u;
                    } else {
                        a.ct[o] = cg[j];
                        if (a.idx) a.idx[o] = (int32_t)j;
                    }
                    my_alg += (unsigned long long)(j + 1);
                }
                team_alg += (unsigned long long)(first + 1);
                found = true;
                break;
            }
        }
        if (!found) {
            team_alg += (unsigned long long)V;
            if (tl == 0) {
                const int64_t o = m * L + i;
                a.ct[o] = __longlong_as_double(0x7ff8000000000000ll);
                if (a.idx) a.idx[o] = -1;
                my_status |= 1u;
                my_alg += (unsigned long long)V;
            }
        }
    }
    if (a.team_dets && tl == 0) a.team_dets[g] = team_alg;

    // ---- per-warp aggregation of the work counters (one atomic per warp)
    my_alg = warp_sum_u64(my_alg);
    my_eval = warp_sum_u64(my_eval);
    my_fb = warp_sum_u64(my_fb);
    my_status = __reduce_or_sync(FULL, my_status);
    if (lane == 0) {
        if (my_alg) atomicAdd(&ws->alg_dets, my_alg);
        if (my_eval) atomicAdd(&ws->eval_dets, my_eval);
        if (my_fb) atomicAdd(&ws->fallback_dets, my_fb);
        if (my_status) atomicOr(&ws->row_status, my_status);
    }
}

// The direct element's cosh/sinh table (FineTab where the call allows it, ws_fine) is a
// kernel template parameter: the launcher enqueues both instances and the one that does not
// match the call returns at once (the table choice needs the validation pass, which runs on
// the device; one kernel holding both bodies behind a run-time branch was measured slower:
// C5 38.89 ms vs 37.85 ms for the fine body alone).
template <class TabT>
__device__ __forceinline__ bool tab_mismatch(const Workspace *ws)
{
    return ws_fine(ws) != std::is_same<TabT, FineTab>::value;
}

template <int TEAM, int BLOCK, bool STABLE, class TabT>
__global__ void __launch_bounds__(BLOCK, scan_min_blocks<BLOCK>()) scan_kernel(ScanArgs a)
{
    if (!STABLE && tab_mismatch<TabT>(a.ws)) return;
    scan_kernel_body<TEAM, BLOCK, STABLE, TabT>(a);
}

// ------------------------------------------------------------------ model-major scan
// For ensembles (many models): a warp takes a WORK ITEM = one model and up to kModelRows of
// its wavelengths, and scans the velocity chunks in ascending order for all of the item's
// rows that have not found their first sign change yet.  Per chunk each lane computes the
// wavelength-free terms of its velocity once (the P/S square roots of every layer and the
// half-space element / k, see wave_root and halfspace in masw_det.cuh) into warp-private
// shared memory, and reuses them for every active row -- each row's determinant then needs
// only its k h_e-dependent part.  Results are those of scan_kernel (same algorithm per row,
// K^ = K / k has the sign of K).
// Two wavelengths per lane with fully interleaved (branch-free) sign evaluations, 16 warps
// per SM at 128 registers (76 B of spills): measured on C5 45.7 ms vs 46.9 ms at 12 warps
// (164 registers, no spills) and 46.9 ms for one wavelength per lane; the node loop is best
// not unrolled (58.5 ms unrolled twice).
#ifndef MASW_MODELS_PAIR
#define MASW_MODELS_PAIR 1
#endif
#ifndef MASW_MODELS_UNROLL
#define MASW_MODELS_UNROLL 1
#endif
constexpr int kModelRows = 40;   // wavelengths per work item (C5: 40, one item per model)
#ifndef MASW_TAIL_ROWS
#define MASW_TAIL_ROWS 8
#endif
#ifndef MASW_TAIL_ITEMS
#define MASW_TAIL_ITEMS 2
#endif
constexpr int kTailRows = MASW_TAIL_ROWS;            // wavelengths per tail piece
constexpr int64_t kTailItemsPerWarp = MASW_TAIL_ITEMS;
// ONE CTA per SM: one copy of the 89 KB cosh/sinh table serves all of its warps; as many
// warps as the per-warp caches leave room for, up to kModelsBlock / 32 (16 for N <= 6).
#ifndef MASW_MODELS_BLOCK
#define MASW_MODELS_BLOCK 512
#endif
constexpr int kModelsBlock = MASW_MODELS_BLOCK;
constexpr int kModelsMinWarps = 12;

// Per-warp shared memory of the model-major scan: the model's k-free constants, k per row,
// the first grid index per row (small-c prefix, reading S15''),
// the carried sign per row, then the lanes' caches of 2N + 2 16-byte slots each, slot-major
// (slot q of lane l at 512 q + 16 l: a warp's 128-bit loads of one slot are contiguous and
// conflict-free): the roots (x_a, 1/|x_a|), (x_b, 1/|x_b|) of every layer (slots 2e, 2e + 1)
// and the half-space's k-free factors (r, s), (gw, t') (HsRoot; t' = t, +0 or -0 encodes the
// case, see hs_from_cache).  (32 N + 32 bytes per lane: with 16 warps at N = 6 this leaves
// room for the fine cosh/sinh table.)
__host__ __device__ inline unsigned lane_cache_stride(int N) { return 32u * (unsigned)N + 32u; }
constexpr unsigned kSlot = 512u;   // bytes between consecutive slots of one lane
__host__ __device__ inline unsigned models_cache_off(int N)
{
    return round16((unsigned)(N + 1) * (unsigned)sizeof(LayerConst) +     // model constants
                   (unsigned)kModelRows * (unsigned)sizeof(double) +       // k per row
                   (unsigned)kModelRows * (unsigned)sizeof(int32_t) +      // first index per row
                   (unsigned)kModelRows);                                  // carried sign per row (s8)
}
__host__ __device__ inline unsigned warp_model_bytes(int N)
{
    return models_cache_off(N) + 32u * lane_cache_stride(N);              // + the lanes' caches
}

// GEPP sign for one lane of the model-major kernel (see row_det_gepp); the same element
// and half-space evaluation as the kernel's hot path.
// LayerConst of a k-free model with k h formed for one wavelength (the row scan's kh field)
__device__ __forceinline__ LayerConst with_kh(LayerConst M, double kh)
{
    M.kh = kh;
    return M;
}

template <bool STABLE, class TabT>
static __device__ __noinline__ int models_det_gepp(unsigned ma, unsigned ca, unsigned ha,
                                                   TabT ta, double k,
                                                   double c2, int N)
{
    const DetOut d = det_core<false, 0, 1>(
        N,
        [&](int e) {
            const unsigned o = 2u * kSlot * (unsigned)e;
            const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
            if constexpr (STABLE) return layer_elem_stable(with_kh(M, k * M.kh), c2, ta);
            else return layer_elem_root(M, k, lds_v2(ca + o), lds_v2(ca + o + kSlot), c2, ta);
        },
        [&] {
            const LayerConst H = load_lc_at(ha);   // as the row scan's GEPP forms it
            return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), lc_mu(H));
        });
    return d.bad ? 2 : d.sign;
}

template <bool STABLE, class TabT>
__device__ __forceinline__ void scan_models_body(ScanArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_abort;

    const int N = a.mod.N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *tab = smem;
    unsigned char *wb = smem + kExpTabBytes + (unsigned)warp * warp_model_bytes(N);
    LayerConst *mc = reinterpret_cast<LayerConst *>(wb);
    double *kr = reinterpret_cast<double *>(wb + (unsigned)(N + 1) * sizeof(LayerConst));
    int32_t *jst = reinterpret_cast<int32_t *>(kr + kModelRows);             // per row: first index
    signed char *carry = reinterpret_cast<signed char *>(jst + kModelRows);  // per row: last sign
    unsigned char *cl = wb + models_cache_off(N) + 16u * (unsigned)lane;   // slot 0 of this lane

    Workspace *ws = a.ws;
    if (threadIdx.x == 0) {
        const bool bad = ws_invalid(ws, a.grid_mask, true);
        s_abort = bad;
        if (bad && blockIdx.x == 0) ws->abort = 1;
    }
    __syncthreads();
    if (s_abort) return;
    exp_scale_fill<TabT>(tab, ws_exp_rows<TabT>(ws));
    __syncthreads();
    const TabT ta = TabTraits<TabT>::make(opaque(smem_addr(tab)));
    const bool prefix = a.pstart != nullptr && ws->prefix_rows != 0ull;   // reading S15''

    const int64_t M = a.mod.M, L = a.L;
    const int V = (int)a.V;                 // < 2^31 (idx is int32; checked by the C ABI)
    const int64_t groups = (L + kModelRows - 1) / kModelRows;
    const int64_t Mt = a.tail_models, Mh = M - Mt;       // finer items for the last Mt models
    const int tr = a.tail_rows > 0 ? a.tail_rows : kModelRows;
    const int64_t groups_t = (L + tr - 1) / tr;
    const int64_t items_h = Mh * groups;
    const int64_t items = items_h + Mt * groups_t;
    const double *__restrict__ cg = a.c;
    const int nv = 2 * (N + 1);
    unsigned long long my_alg = 0, my_eval = 0, team_alg = 0, my_fb = 0;
    unsigned my_status = 0;

    for (;;) {
        long long item;
        if (lane == 0) item = (long long)atomicAdd(&ws->queue, 1ull);
        item = __shfl_sync(FULL, item, 0);
        if (item >= items) break;
        int64_t m, i0;
        int nr;
        if (item < items_h) {
            m = item / groups;
            i0 = (item - m * groups) * kModelRows;
            nr = (int)min((int64_t)kModelRows, L - i0);
        } else {
            const int64_t it = item - items_h, q = it / groups_t;
            m = Mh + q;
            i0 = (it - q * groups_t) * tr;
            nr = (int)min((int64_t)tr, L - i0);
        }

        // model constants without the wavenumber: h, 1/alpha^2, 1/beta^2, rho, beta^2
        for (int e = lane; e <= N; e += 32) {
            const double al = a.mod.alpha[m * (N + 1) + e];
            const double be = a.mod.beta[m * (N + 1) + e];
            const double rh = a.mod.rho[m * (N + 1) + e];
            LayerConst x;
            x.kh = (e < N) ? a.mod.h[m * N + e] : 0.0;
            x.ia2 = 1.0 / (al * al);
            x.ib2 = 1.0 / (be * be);
            x.krho = rh;               // K / k: rho and rho beta^2 (see scan_kernel)
            x.b2 = 2.0 * (be * be);
            x.aux = (e < N) ? rh / a.mod.rho[m * (N + 1) + e + 1]
                            : (rh * (be * be)) / a.mod.rho[m * (N + 1) + N - 1];
            mc[e] = x;
        }
        // the model's layer velocities (reading S4) are read from global memory (L1) per chunk
        const double *__restrict__ mal = a.mod.alpha + m * (N + 1);
        const double *__restrict__ mbe = a.mod.beta + m * (N + 1);
        // rows of the item in two 32-bit halves: pending = not yet found.  Small-c prefix
        // (reading S15''): row r's scan starts at jst[r] with carried sign carry[r]; rows the
        // prefix kernel finished are not pending.  smax / smin: largest / smallest start.
        unsigned pend0 = (nr >= 32) ? ~0u : ((1u << nr) - 1u);
        unsigned pend1 = (nr > 32) ? ((1u << (nr - 32)) - 1u) : 0u;
        int smax = 0, smin = 0;
        {
            int hi = 0, lo = INT_MAX;
            unsigned done0 = 0, done1 = 0;
            for (int r = lane; r < nr; r += 32) {
                kr[r] = kTwoPi / a.lam[i0 + r];   // reading S2
                int st = 0, cs = 0;
                if (prefix) {
                    st = a.pstart[m * L + i0 + r];
                    cs = a.pcarry[m * L + i0 + r];
                }
                jst[r] = st;
                carry[r] = (signed char)cs;
                if (st >= 0) {
                    hi = max(hi, st);
                    lo = min(lo, st);
                }
                const unsigned fin = __ballot_sync(__activemask(), st < 0);
                if (r < 32) done0 = fin; else done1 = fin;
            }
            pend0 &= ~__shfl_sync(FULL, done0, 0);
            pend1 &= ~__shfl_sync(FULL, done1, 0);
            smax = __reduce_max_sync(FULL, hi);
            smin = __reduce_min_sync(FULL, lo);
        }
        __syncwarp();
        const unsigned ma = opaque(smem_addr(mc));
        const unsigned ha = ma + (unsigned)N * (unsigned)sizeof(LayerConst);
        const unsigned ka = opaque(smem_addr(kr));
        const unsigned sa = opaque(smem_addr(jst));
        const unsigned ya = opaque(smem_addr(carry));

        unsigned ev32 = 0, fb32 = 0;
        const int base0 = (pend0 | pend1) ? (smin / 32) * 32 : 0;
        for (int base = base0; base < V && (pend0 | pend1); base += 32) {
            const int j = base + lane;
            const bool valid = j < V;
            double c = cg[valid ? j : V - 1];
            {   // reading S4, as in scan_kernel (velocity i = 2e + w: alpha_e, beta_e)
                const double clo = __shfl_sync(FULL, c, 0) - 1e-3;
                const double chi = __shfl_sync(FULL, c, 31) + 1e-3;
                bool lane_near = false;
                for (int e0 = 0; e0 < nv; e0 += 32) {
                    const int i = e0 + lane;
                    const double v = (i < nv) ? ((i & 1) ? mbe : mal)[i >> 1] : 0.0;
                    const bool in = (i < nv) && (v > clo) && (v < chi);
                    for (unsigned b = __ballot_sync(FULL, in); b; b &= b - 1)
                        lane_near |= fabs(c - __shfl_sync(FULL, v, __ffs(b) - 1)) < kPerturbTol;
                }
                if (lane_near) c = perturb_velocity_ab(mal, mbe, N + 1, c);
            }
            const double c2 = c * c;
            const double ic2 = rcp_fast(c2);
            // wavelength-free terms of this lane's velocity (lane-private slots: no sync)
            {
                double2 *rt = reinterpret_cast<double2 *>(cl);   // slot q at rt[32 q]
                for (int e = 0; e < N; ++e) {
                    const LayerConst Lc = mc[e];
                    rt[64 * e] = wave_root(fma(-c2, Lc.ia2, 1.0));
                    rt[64 * e + 32] = wave_root(fma(-c2, Lc.ib2, 1.0));
                }
                // the half-space's k-free factors; hs_from_cache forms the element per pair
                const LayerConst Hl = mc[N];
                const HsRoot R = halfspace_root(Hl.ia2, Hl.ib2, c2);
                rt[64 * N] = make_double2(R.r, R.s);
                rt[64 * N + 32] = make_double2(R.gw, R.kase == 1 ? R.t : (R.kase == 0 ? 0.0 : -0.0));
            }
            const unsigned ca = opaque(smem_addr(cl));
            const unsigned hca = ca + 2u * kSlot * (unsigned)N;
            // chunks below some row's small-c prefix end (reading S15''): only the rows whose
            // scan starts before the chunk's end take part; lanes below a row's start take the
            // prefix's sign
            const bool slow = base < smax;
            unsigned act0 = ~0u, act1 = ~0u;
            if (slow) {
                const bool a0 = lane < nr && lds_s32(sa + 4u * (unsigned)lane) < base + 32;
                const bool a1 = lane + 32 < nr && lds_s32(sa + 4u * (unsigned)(lane + 32)) < base + 32;
                act0 = __ballot_sync(FULL, a0);
                act1 = __ballot_sync(FULL, a1);
            }
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                unsigned pend = half ? (pend1 & act1) : (pend0 & act0);
                unsigned found = 0;
                // first-sign-change bookkeeping of row r for this chunk (lane signs s, bad)
                auto settle = [&](int r, int s, bool bad) {
                    if (slow && j < lds_s32(sa + 4u * (unsigned)r)) {
                        s = lds_s8(ya + (unsigned)r);
                        bad = false;
                    }
                    int sprev = __shfl_up_sync(FULL, s, 1);
                    if (lane == 0) sprev = lds_s8(ya + (unsigned)r);
                    const bool ev = valid && (bad || (j > 0 && s != sprev));
                    const unsigned mask = __ballot_sync(FULL, ev);
                    if (mask) {
                        const int first = base + (__ffs(mask) - 1);
                        if (j == first) {
                            const int64_t o = m * L + i0 + r;
                            if (bad) {
                                a.ct[o] = __longlong_as_double(0x7ff8000000000000ll);
                                if (a.idx) a.idx[o] = -2;
                                my_status |= 2u;
                            } else {
                                a.ct[o] = cg[j];
                                if (a.idx) a.idx[o] = (int32_t)j;
                            }
                            my_alg += (unsigned long long)(j + 1);
                        }
                        team_alg += (unsigned long long)(first + 1);
                        found |= 1u << (r - half * 32);
                    } else if (lane == 31) {
                        sts_s8(ya + (unsigned)r, s);   // carried to the next chunk
                    }
                };
                // K_hs / (rho_(N-1) c^2), k-free: from the cached HsRoot (the case from t':
                // t > 0 in case 1, +0 in case 0, -0 in case 2), formed as the row scan forms it
                auto hs_scaled = [&] {
                    const double2 p = lds_v2(hca), q = lds_v2(hca + kSlot);
                    HsRoot R;
                    R.r = p.x;
                    R.s = p.y;
                    R.gw = q.x;
                    R.t = q.y;
                    const int th = __double2hiint(q.y);
                    R.kase = th > 0 ? 1 : (th < 0 ? 2 : 0);
                    return halfspace_k(R, lds_f64(ha + 40u) * ic2);   // mu' = aux_N / c^2
                };
#if !MASW_BLOCK_SIGN
                auto hs_gepp = [&] {     // K_hs / k, as the row scan's GEPP forms it
                    const LayerConst H = load_lc_at(ha);
                    return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), lc_mu(H));
                };
#endif
                while (pend) {
                    const int r = half * 32 + __ffs(pend) - 1;
                    pend &= pend - 1;
                    const double k = lds_f64(ka + 8u * (unsigned)r);
#if MASW_MODELS_PAIR
                    if (pend && !a.pivoted) {   // two rows: fully interleaved sign evaluations
                        const int r2 = half * 32 + __ffs(pend) - 1;
                        pend &= pend - 1;
                        const double k2 = lds_f64(ka + 8u * (unsigned)r2);
                        int s1 = 0, s2 = 0;
                        bool bad1 = false, bad2 = false;
                        if (valid) {
                            SignOut o1, o2;
                            det_sign_block_u_pair<MASW_MODELS_UNROLL>(
                                N,
                                [&](int e, ElemU &E1, ElemU &E2) {
                                    const unsigned o = 2u * kSlot * (unsigned)e;
                                    const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
                                    if constexpr (STABLE) {
                                        E1 = layer_elemu_stable(with_kh(M, k * M.kh), c2, ic2, ta);
                                        E2 = layer_elemu_stable(with_kh(M, k2 * M.kh), c2, ic2, ta);
                                    } else {
                                        layer_elem_root2_u(M, k, k2, lds_v2(ca + o),
                                                           lds_v2(ca + o + kSlot), c2, ic2, ta, E1,
                                                           E2);
                                    }
                                },
                                [&](HalfSpace &H1, HalfSpace &H2) {
                                    H1 = hs_scaled();
                                    H2 = H1;
                                },
                                o1, o2);
                            if (o1.ok) {
                                s1 = o1.sign;
                            } else {
                                const int rr = models_det_gepp<STABLE>(ma, ca, ha, ta, k, c2, N);
                                bad1 = (rr == 2);
                                s1 = bad1 ? 0 : rr;
                                ++fb32;
                            }
                            if (o2.ok) {
                                s2 = o2.sign;
                            } else {
                                const int rr = models_det_gepp<STABLE>(ma, ca, ha, ta, k2, c2, N);
                                bad2 = (rr == 2);
                                s2 = bad2 ? 0 : rr;
                                ++fb32;
                            }
                            ev32 += 2;
                        }
                        settle(r, s1, bad1);
                        settle(r2, s2, bad2);
                        continue;
                    }
#endif
                    int s = 0;
                    bool bad = false;
                    if (valid) {
#if MASW_BLOCK_SIGN
                        SignOut so;
                        so.ok = false;
                        if (!a.pivoted)
                            so = det_sign_block_u<MASW_MODELS_UNROLL>(
                                N,
                                [&](int e) {
                                    const unsigned o = 2u * kSlot * (unsigned)e;
                                    const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
                                    if constexpr (STABLE)
                                        return layer_elemu_stable(with_kh(M, k * M.kh), c2, ic2, ta);
                                    else
                                        return layer_elem_root_u(M, k, lds_v2(ca + o),
                                                                 lds_v2(ca + o + kSlot), c2, ic2, ta);
                                },
                                hs_scaled);
                        if (so.ok) {
                            s = so.sign;
                        } else {
                            const int r = models_det_gepp<STABLE>(ma, ca, ha, ta, k, c2, N);
                            bad = (r == 2);
                            s = bad ? 0 : r;
                            fb32 += a.pivoted ? 0u : 1u;
                        }
#else
                        const DetOut d = det_core<false, 0, MASW_MODELS_UNROLL>(
                            N,
                            [&](int e) {
                                const unsigned o = 2u * kSlot * (unsigned)e;
                                return layer_elem_root(load_lc_at(ma + 48u * (unsigned)e), k,
                                                       lds_v2(ca + o), lds_v2(ca + o + kSlot), c2, ta);
                            },
                            hs_gepp);
                        s = d.sign;
                        bad = d.bad;
#endif
                        ++ev32;
                    }
                    settle(r, s, bad);
                }
                if (half) pend1 &= ~found; else pend0 &= ~found;
            }
            __syncwarp();   // the next chunk rewrites this lane's roots; carries are visible
        }
        my_eval += ev32;
        my_fb += fb32;
        for (int half = 0; half < 2; ++half) {
            for (unsigned pend = half ? pend1 : pend0; pend; pend &= pend - 1) {
                const int r = half * 32 + __ffs(pend) - 1;
                team_alg += (unsigned long long)V;
                if (lane == 0) {
                    const int64_t o = m * L + i0 + r;
                    a.ct[o] = __longlong_as_double(0x7ff8000000000000ll);
                    if (a.idx) a.idx[o] = -1;
                    my_status |= 1u;
                    my_alg += (unsigned long long)V;
                }
            }
        }
        __syncwarp();   // the next item rewrites this warp's constants
    }
    if (a.team_dets && lane == 0) {
#ifdef MASW_TAIL_PROBE   // measurement build (scripts/tail_probe.py): warp finish times
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.team_dets[(long long)blockIdx.x * (blockDim.x / 32) + warp] = t;
#else
        a.team_dets[(long long)blockIdx.x * (blockDim.x / 32) + warp] = team_alg;
#endif
    }

    my_alg = warp_sum_u64(my_alg);
    my_eval = warp_sum_u64(my_eval);
    my_fb = warp_sum_u64(my_fb);
    my_status = __reduce_or_sync(FULL, my_status);
    if (lane == 0) {
        if (my_alg) atomicAdd(&ws->alg_dets, my_alg);
        if (my_eval) atomicAdd(&ws->eval_dets, my_eval);
        if (my_fb) atomicAdd(&ws->fallback_dets, my_fb);
        if (my_status) atomicOr(&ws->row_status, my_status);
    }
}

template <bool STABLE, class TabT>
__global__ void __launch_bounds__(kModelsBlock, 1) scan_models_kernel(ScanArgs a)
{
    if (!STABLE && tab_mismatch<TabT>(a.ws)) return;
    scan_models_body<STABLE, TabT>(a);
}

// ------------------------------------------------------------------ pair scan (one long curve)
// Single curves with many wavelengths (C3, C4): a warp pops TWO consecutive rows of the one
// model and scans them in lockstep -- each lane evaluates both rows at its velocity with the
// model-major kernel's interleaved pair evaluation (det_sign_block_u_pair), so the
// wavelength-free terms (the 2N wave roots, the half-space factor, 1/c^2) are computed once
// per lane, chunk and PAIR instead of once per determinant.  Adjacent rows of a sorted curve
// stop at nearby indices (identical rows for C3), so the lockstep costs little; once one row
// has found its change the other continues alone.  Each determinant uses the row scan's
// operations in the row scan's order: bitwise-identical results (tests).
constexpr int kPairBlock = 512;   // one CTA (one table copy) of 16 warps per SM, 128 registers

// per warp: the current model's k-free constants and layer velocities (S4)
__host__ __device__ inline unsigned pair_warp_bytes(int N)
{
    return round16((unsigned)(N + 1) * (unsigned)sizeof(LayerConst) +
                   2u * (unsigned)(N + 1) * (unsigned)sizeof(double));
}
__host__ __device__ inline unsigned pair_smem_bytes(int N)
{
    return (unsigned)kExpTabBytes + (unsigned)(kPairBlock / 32) * pair_warp_bytes(N);
}

// GEPP sign for one lane of the pair scan (roots formed on the fly, as the row scan forms them)
template <bool STABLE, class TabT>
static __device__ __noinline__ int pair_det_gepp(unsigned ma, unsigned ha, TabT ta,
                                                 double k, double c2, int N)
{
    const DetOut d = det_core<false, 0, 1>(
        N,
        [&](int e) {
            const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
            if constexpr (STABLE) return layer_elem_stable(with_kh(M, k * M.kh), c2, ta);
            else return layer_elem_root(M, k, wave_root(fma(-c2, M.ia2, 1.0)),
                                        wave_root(fma(-c2, M.ib2, 1.0)), c2, ta);
        },
        [&] {
            const LayerConst H = load_lc_at(ha);
            return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), lc_mu(H));
        });
    return d.bad ? 2 : d.sign;
}

template <bool STABLE, class TabT>
__device__ __forceinline__ void scan_pair_body(ScanArgs a)
{
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_abort;

    const int N = a.mod.N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *tab = smem;
    unsigned char *wb = smem + kExpTabBytes + (unsigned)warp * pair_warp_bytes(N);
    LayerConst *mc = reinterpret_cast<LayerConst *>(wb);
    double *vel = reinterpret_cast<double *>(wb + (unsigned)(N + 1) * sizeof(LayerConst));

    Workspace *ws = a.ws;
    if (threadIdx.x == 0) {
        const bool bad = ws_invalid(ws, a.grid_mask, true);
        s_abort = bad;
        if (bad && blockIdx.x == 0) ws->abort = 1;
    }
    __syncthreads();
    if (s_abort) return;
    exp_scale_fill<TabT>(tab, ws_exp_rows<TabT>(ws));
    __syncthreads();
    const TabT ta = TabTraits<TabT>::make(opaque(smem_addr(tab)));

    const bool prefix = a.pstart != nullptr && ws->prefix_rows != 0ull;   // reading S15''
    const int64_t M = a.mod.M, L = a.L;
    const int64_t pairs_per_model = (L + 1) / 2;
    // work items: the first Ph pair items whole, then the last Pt pair items as velocity
    // segments, segment-major (all first segments, then all second segments, ...), so idle
    // warps share the rows still running at the end instead of waiting on them
    const int64_t P = M * pairs_per_model, Pt = a.tail_pairs, Ph = P - Pt;
    const int S = a.seg_count, SEGV = a.seg_len;
    const int64_t items = Ph + Pt * (int64_t)S;
    const int V = (int)a.V;
    const double *__restrict__ cg = a.c;
    const int nv = 2 * (N + 1);
    unsigned long long my_alg = 0, my_eval = 0, team_alg = 0, my_fb = 0;
    unsigned my_status = 0;
    int64_t cur_m = -1;

    for (;;) {
        // work item = (wavelength pair ip, model m), pair-major: the long wavelengths of
        // every model first, as the row scan's lambda-major order
        long long item;
        if (lane == 0) item = (long long)atomicAdd(&ws->queue, 1ull);
        item = __shfl_sync(FULL, item, 0);
        if (item >= items) break;
        int64_t pi = item, tp = -1;
        int seg = -1, seg_lo = 0;
        if (item >= Ph) {   // tail segment seg of tail pair tp
            const int64_t t = item - Ph;
            seg = (int)(t / Pt);
            tp = t - (int64_t)seg * Pt;
            pi = Ph + tp;
            seg_lo = seg * SEGV;
        }
        // the item's scan, instantiated for whole pairs and for tail segments (SEG): the
        // whole-pair loop carries none of the segment bookkeeping
        auto item_body = [&](auto segc) {
            constexpr bool SEG = decltype(segc)::value;
            const int seg_hi = (!SEG) ? V : min(V, seg_lo + SEGV);
            const int64_t ip = pi / M, m = pi - ip * M;
            const int64_t i0 = 2 * ip;
            const bool two = i0 + 1 < L;
            if (m != cur_m) {   // this model's k-free constants (as the model-major scan fills them)
                __syncwarp();
                for (int e = lane; e <= N; e += 32) {
                    const double al = a.mod.alpha[m * (N + 1) + e], be = a.mod.beta[m * (N + 1) + e];
                    const double rh = a.mod.rho[m * (N + 1) + e];
                    LayerConst x;
                    x.kh = (e < N) ? a.mod.h[m * N + e] : 0.0;
                    x.ia2 = 1.0 / (al * al);
                    x.ib2 = 1.0 / (be * be);
                    x.krho = rh;
                    x.b2 = 2.0 * (be * be);
                    x.aux = (e < N) ? rh / a.mod.rho[m * (N + 1) + e + 1]
                                    : (rh * (be * be)) / a.mod.rho[m * (N + 1) + N - 1];
                    mc[e] = x;
                    vel[2 * e] = al;
                    vel[2 * e + 1] = be;
                }
                __syncwarp();
                cur_m = m;
            }
            const unsigned ma = opaque(smem_addr(mc));
            const unsigned ha = ma + (unsigned)N * (unsigned)sizeof(LayerConst);
            const long long r0 = m * L + i0;                        // output row of wavelength i0
            const double k0 = kTwoPi / a.lam[i0];                   // reading S2
            const double k1 = two ? kTwoPi / a.lam[i0 + 1] : k0;
            // small-c prefixes (reading S15''): row q starts at js_q with carried sign pc_q, or
            // was finished by smallc_prefix_kernel (js_q = -1)
            int js0 = 0, js1 = 0, pc0 = 0, pc1 = 0;
            if (prefix) {
                js0 = a.pstart[r0];
                pc0 = a.pcarry[r0];
                if (two) {
                    js1 = a.pstart[r0 + 1];
                    pc1 = a.pcarry[r0 + 1];
                }
            }
            int carry0 = pc0, carry1 = pc1;
            bool pend0 = js0 >= 0, pend1 = two && js1 >= 0;
            if (SEG) {   // rows with an event in an earlier segment need no more segments
                if (pend0 && *(volatile int *)&a.seg_found[2 * tp] < seg_lo) pend0 = false;
                if (pend1 && *(volatile int *)&a.seg_found[2 * tp + 1] < seg_lo) pend1 = false;
            }
            const bool rec0 = SEG && pend0, rec1 = SEG && pend1;   // write a record
            int fs0 = 0, fs1 = 0;            // segment: sign at seg_lo
            int ev0 = -1, ev1 = -1;          // segment: in-segment event index
            bool eb0 = false, eb1 = false;   // segment: the event is a non-finite det
            const int jlo = (SEG) ? seg_lo
                          : ((pend0 && pend1) ? min(js0, js1) : (pend0 ? js0 : (pend1 ? js1 : 0)));
            const int jfirst = (SEG) ? seg_lo : 0;   // no predecessor to compare with
            for (int base = (jlo / 32) * 32; base < seg_hi && (pend0 || pend1); base += 32) {
                const int j = base + lane;
                const bool valid = j < seg_hi;
                double c = cg[valid ? j : V - 1];
                {   // reading S4, as in scan_kernel
                    const double clo = __shfl_sync(FULL, c, 0) - 1e-3;
                    const double chi = __shfl_sync(FULL, c, 31) + 1e-3;
                    bool lane_near = false;
                    for (int e0 = 0; e0 < nv; e0 += 32) {
                        bool in = false;
                        if (e0 + lane < nv) {
                            const double v = vel[e0 + lane];
                            in = (v > clo) && (v < chi);
                        }
                        for (unsigned b = __ballot_sync(FULL, in); b; b &= b - 1)
                            lane_near |= fabs(c - vel[e0 + __ffs(b) - 1]) < kPerturbTol;
                    }
                    if (lane_near) c = perturb_velocity(vel, nv, c);
                }
                const double c2 = c * c;
                const double ic2 = rcp_fast(c2);
                int s0 = 0, s1 = 0;
                bool bad0 = false, bad1 = false;
                if (valid) {
                    const LayerConst Hl = load_lc_at(ha);
                    const HalfSpace H = halfspace_k(halfspace_root(Hl.ia2, Hl.ib2, c2), Hl.aux * ic2);
                    if (pend0 && pend1) {
                        SignOut o0, o1;
                        det_sign_block_u_pair<MASW_MODELS_UNROLL>(
                            N,
                            [&](int e, ElemU &E0, ElemU &E1) {
                                const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
                                if constexpr (STABLE) {
                                    E0 = layer_elemu_stable(with_kh(M, k0 * M.kh), c2, ic2, ta);
                                    E1 = layer_elemu_stable(with_kh(M, k1 * M.kh), c2, ic2, ta);
                                } else {
                                    layer_elem_root2_u(M, k0, k1, wave_root(fma(-c2, M.ia2, 1.0)),
                                                       wave_root(fma(-c2, M.ib2, 1.0)), c2, ic2, ta,
                                                       E0, E1);
                                }
                            },
                            [&](HalfSpace &H0, HalfSpace &H1) {
                                H0 = H;
                                H1 = H;
                            },
                            o0, o1);
                        if (o0.ok) {
                            s0 = o0.sign;
                        } else {
                            const int rr = pair_det_gepp<STABLE>(ma, ha, ta, k0, c2, N);
                            bad0 = (rr == 2);
                            s0 = bad0 ? 0 : rr;
                            ++my_fb;
                        }
                        if (o1.ok) {
                            s1 = o1.sign;
                        } else {
                            const int rr = pair_det_gepp<STABLE>(ma, ha, ta, k1, c2, N);
                            bad1 = (rr == 2);
                            s1 = bad1 ? 0 : rr;
                            ++my_fb;
                        }
                        my_eval += 2;
                    } else {
                        const double k = pend0 ? k0 : k1;
                        const SignOut o = det_sign_block_u<MASW_MODELS_UNROLL>(
                            N,
                            [&](int e) {
                                const LayerConst M = load_lc_at(ma + 48u * (unsigned)e);
                                if constexpr (STABLE)
                                    return layer_elemu_stable(with_kh(M, k * M.kh), c2, ic2, ta);
                                else
                                    return layer_elem_root_u(M, k, wave_root(fma(-c2, M.ia2, 1.0)),
                                                             wave_root(fma(-c2, M.ib2, 1.0)), c2, ic2,
                                                             ta);
                            },
                            [&] { return H; });
                        int s = 0;
                        bool bad = false;
                        if (o.ok) {
                            s = o.sign;
                        } else {
                            const int rr = pair_det_gepp<STABLE>(ma, ha, ta, k, c2, N);
                            bad = (rr == 2);
                            s = bad ? 0 : rr;
                            ++my_fb;
                        }
                        if (pend0) { s0 = s; bad0 = bad; } else { s1 = s; bad1 = bad; }
                        ++my_eval;
                    }
                }
                if (j < js0) {   // evaluated by the small-c prefix
                    s0 = pc0;
                    bad0 = false;
                }
                if (j < js1) {
                    s1 = pc1;
                    bad1 = false;
                }
                // first-sign-change bookkeeping of one row for this chunk (as scan_kernel, TEAM 1);
                // a tail segment records its first sign / event instead of writing the row
                auto settle = [&](long long r, int s, bool bad, int &carry, bool &pend, int &fs,
                                  int &evj, bool &evb, int tq) {
                    int sprev = __shfl_up_sync(FULL, s, 1);
                    if (lane == 0) sprev = carry;
                    if (SEG && base == seg_lo) fs = __shfl_sync(FULL, s, 0);
                    const bool ev = valid && (bad || (j > jfirst && s != sprev));
                    const unsigned mask = __ballot_sync(FULL, ev);
                    if (mask) {
                        const int first = base + (__ffs(mask) - 1);
                        if (SEG) {
                            evj = first;
                            evb = __shfl_sync(FULL, (int)bad, __ffs(mask) - 1) != 0;
                            if (lane == 0) atomicMin(&a.seg_found[tq], first);
                            team_alg += (unsigned long long)(first + 1 - seg_lo);
                        } else if (j == first) {
                            if (bad) {
                                a.ct[r] = __longlong_as_double(0x7ff8000000000000ll);
                                if (a.idx) a.idx[r] = -2;
                                my_status |= 2u;
                            } else {
                                a.ct[r] = cg[j];
                                if (a.idx) a.idx[r] = (int32_t)j;
                            }
                            my_alg += (unsigned long long)(j + 1);
                        }
                        if (!SEG) team_alg += (unsigned long long)(first + 1);
                        pend = false;
                    }
                    // the last valid lane's sign (the segment's last sign after its last chunk)
                    carry = __shfl_sync(FULL, s, min(31, seg_hi - 1 - base));
                };
                if (pend0) settle(r0, s0, bad0, carry0, pend0, fs0, ev0, eb0, (int)(2 * tp));
                if (pend1) settle(r0 + 1, s1, bad1, carry1, pend1, fs1, ev1, eb1, (int)(2 * tp + 1));
            }
            if (SEG) {   // the segment's records: event index, first / last sign, flags
                if (lane == 0) {
                    if (rec0)
                        a.seg_rec[(2 * tp) * S + seg] =
                            make_int2(ev0, (fs0 + 1) | ((carry0 + 1) << 2) | ((int)eb0 << 4) | 32);
                    if (rec1)
                        a.seg_rec[(2 * tp + 1) * S + seg] =
                            make_int2(ev1, (fs1 + 1) | ((carry1 + 1) << 2) | ((int)eb1 << 4) | 32);
                }
                team_alg += pend0 ? (unsigned long long)(seg_hi - seg_lo) : 0ull;   // no event
                team_alg += pend1 ? (unsigned long long)(seg_hi - seg_lo) : 0ull;
                return;
            }
            for (int q = 0; q < 2; ++q) {
                const bool p = q ? pend1 : pend0;
                if (!p) continue;   // (the q loop: the other row may still need its write)
                team_alg += (unsigned long long)V;
                if (lane == 0) {
                    const long long r = r0 + q;
                    a.ct[r] = __longlong_as_double(0x7ff8000000000000ll);
                    if (a.idx) a.idx[r] = -1;
                    my_status |= 1u;
                    my_alg += (unsigned long long)V;
                }
            }
        };
        if (seg >= 0)
            item_body(std::true_type{});
        else
            item_body(std::false_type{});
    }
    if (a.team_dets && lane == 0)
        a.team_dets[(long long)blockIdx.x * (blockDim.x / 32) + warp] = team_alg;

    my_alg = warp_sum_u64(my_alg);
    my_eval = warp_sum_u64(my_eval);
    my_fb = warp_sum_u64(my_fb);
    my_status = __reduce_or_sync(FULL, my_status);
    if (lane == 0) {
        if (my_alg) atomicAdd(&ws->alg_dets, my_alg);
        if (my_eval) atomicAdd(&ws->eval_dets, my_eval);
        if (my_fb) atomicAdd(&ws->fallback_dets, my_fb);
        if (my_status) atomicOr(&ws->row_status, my_status);
    }
}

template <bool STABLE, class TabT>
__global__ void __launch_bounds__(kPairBlock, 1) scan_pair_kernel(ScanArgs a)
{
    if (!STABLE && tab_mismatch<TabT>(a.ws)) return;
    scan_pair_body<STABLE, TabT>(a);
}

// Per-device launch facts, cached: SM count and resident CTAs per SM per (kernel, smem).
namespace {
std::mutex g_cache_mu;
std::unordered_map<long long, int> g_occ_cache;
int g_sms[64] = {0};

int sm_count(int device)
{
    if (device >= 0 && device < 64 && g_sms[device] > 0) return g_sms[device];
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (device >= 0 && device < 64) g_sms[device] = sms;
    return sms;
}
// Opt-in dynamic shared memory: raised ONCE per (device, kernel) to the device maximum, so a
// later launch never runs with a limit left lower by an earlier, smaller launch (the limit
// does not enter the occupancy computation, which takes the launch's own size).
std::unordered_map<long long, bool> g_smem_set;

template <class K>
cudaError_t ensure_smem_optin(K kern, int device, int kid)
{
    const long long key = ((long long)device << 8) | kid;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        if (g_smem_set.count(key)) return cudaSuccess;
    }
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(g_cache_mu);
    g_smem_set[key] = true;
    return cudaSuccess;
}

size_t smem_optin_limit(int device)
{
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return (size_t)optin;
}
}  // namespace

cudaError_t launch_smallc_prefix(const ScanArgs &a, int32_t *start, int8_t *carry, int64_t *list,
                                 void *lcbuf, cudaStream_t st, int device)
{
    const int64_t rows = a.mod.M * a.L;
    constexpr int64_t kBig = (int64_t)kPrefixBlock * kPrefixPerThread;
    if (rows >= 2ll * sm_count(device) * kBig) {
        smallc_rows_kernel<kPrefixPerThread><<<(unsigned)((rows + kBig - 1) / kBig), kPrefixBlock, 0, st>>>(
            a, start, carry, list, static_cast<LayerConst *>(lcbuf));
    } else {
        smallc_rows_kernel<1><<<(unsigned)((rows + kPrefixBlock - 1) / kPrefixBlock), kPrefixBlock, 0, st>>>(
            a, start, carry, list, static_cast<LayerConst *>(lcbuf));
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t smem = kExpTabBytes;
    e = ensure_smem_optin(smallc_prefix_kernel, device, 7);
    if (e != cudaSuccess) return e;
    // at most all rows are listed (32 per warp); the kernel reads the actual count
    int64_t blocks = 2ll * sm_count(device);
    const int64_t need = (rows + kPrefixBlock - 1) / kPrefixBlock;
    if (need < blocks) blocks = need;
    if (blocks < 1) blocks = 1;
    smallc_prefix_kernel<<<(unsigned)blocks, kPrefixBlock, smem, st>>>(
        a, start, carry, list, static_cast<const LayerConst *>(lcbuf));
    count_launch();
    return cudaGetLastError();
}

int auto_team_warps(int64_t rows, int64_t V, int device)
{
    // Minimise tail idle (~ resident_warps / (2 TEAM rows)) + speculation waste
    // (~ 16 TEAM / dets_per_row) with dets_per_row ~ V/2:  TEAM* = sqrt(Wres d / (32 R)).
    const int sms = sm_count(device);
    const double wres = sms * 16.0;   // resident warps: 2 CTAs x 8 warps per SM (launch bounds)
    // with >= 4 rows per resident warp the tail is short anyway and one-warp teams waste the
    // least speculation (measured: C4 2.35 ms at TEAM = 1 vs 2.45 ms at 2; C3 equal)
    if ((double)rows >= 4.0 * wres) return 1;
    const double d = (double)V / 2.0;
    // halved: measured team optima on C3/C4 (1-2) sit below the bare tail/waste model (4),
    // which ignores the per-chunk team barriers
    const double t = 0.5 * sqrt(wres * d / (32.0 * (double)(rows > 0 ? rows : 1)));
    int team = 1;
    while (team * 2 <= t && team < 16) team *= 2;
    return team;
}

template <int TEAM, int BLOCK, bool STABLE>
static cudaError_t launch_scan_t(const ScanArgs &a, cudaStream_t st, int device,
                                 long long *teams_out, bool dry = false)
{
    constexpr int TEAMS = BLOCK / (32 * TEAM);
    const size_t smem = kExpTabBytes + round16((unsigned)sizeof(TeamCtrl) * TEAMS) +
                        (size_t)TEAMS * team_model_bytes(a.mod.N);
    auto kern = scan_kernel<TEAM, BLOCK, STABLE, unsigned>;
    auto kfine = scan_kernel<TEAM, BLOCK, false, FineTab>;   // (see tab_mismatch)
    const int sms = sm_count(device);
    const long long key = ((long long)device << 48) | ((long long)STABLE << 40) |
                          ((long long)TEAM << 32) | (long long)smem;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        auto it = g_occ_cache.find(key);
        if (it != g_occ_cache.end()) per_sm = it->second;
    }
    {
        cudaError_t e = ensure_smem_optin(kern, device, 16 + TEAM + (STABLE ? 32 : 0));
        if (e == cudaSuccess && !STABLE) e = ensure_smem_optin(kfine, device, 64 + TEAM);
        if (e != cudaSuccess) return e;
    }
    if (per_sm == 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem);
        if (e != cudaSuccess) return e;
        if (per_sm < 1) per_sm = 1;
        std::lock_guard<std::mutex> g(g_cache_mu);
        g_occ_cache[key] = per_sm;
    }
    const int64_t rows = a.mod.M * a.L;
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (rows + TEAMS - 1) / TEAMS;
    if (need < blocks) blocks = need;
    if (blocks < 1) blocks = 1;
    if (teams_out) *teams_out = blocks * TEAMS;
    if (dry) return cudaSuccess;
    kern<<<(unsigned)blocks, BLOCK, smem, st>>>(a);
    count_launch();
    if (!STABLE) {
        kfine<<<(unsigned)blocks, BLOCK, smem, st>>>(a);
        count_launch();
    }
    return cudaGetLastError();
}

// One run-time-N kernel per team size.  Measured and rejected on B200 (C5, 94 ms baseline):
//  * TEAM = 1 compiled per N in 1..12 with the determinant fully unrolled: 119 ms (the N=6
//    kernel grew to 9.4k instructions; instruction-cache bound);
//  * a row-pair kernel sharing the (model, c) terms of two wavelengths per lane: 132 ms
//    (register-bound: 128 registers with spills, or 230 registers at 8 warps/SM).
static cudaError_t dispatch_scan(const ScanArgs &a, int team_warps, cudaStream_t st, int device,
                                 long long *teams_out, bool dry)
{
    if (a.stable) {
        switch (team_warps) {
            case 1: return launch_scan_t<1, 256, true>(a, st, device, teams_out, dry);
            case 2: return launch_scan_t<2, 256, true>(a, st, device, teams_out, dry);
            case 4: return launch_scan_t<4, 256, true>(a, st, device, teams_out, dry);
            case 8: return launch_scan_t<8, 256, true>(a, st, device, teams_out, dry);
            case 16: return launch_scan_t<16, 512, true>(a, st, device, teams_out, dry);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (team_warps) {
        case 1: return launch_scan_t<1, 256, false>(a, st, device, teams_out, dry);
        case 2: return launch_scan_t<2, 256, false>(a, st, device, teams_out, dry);
        case 4: return launch_scan_t<4, 256, false>(a, st, device, teams_out, dry);
        case 8: return launch_scan_t<8, 256, false>(a, st, device, teams_out, dry);
        case 16: return launch_scan_t<16, 512, false>(a, st, device, teams_out, dry);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_scan(const ScanArgs &a, int team_warps, cudaStream_t st, int device,
                        long long *teams_out)
{
    return dispatch_scan(a, team_warps, st, device, teams_out, false);
}

long long scan_teams(const ScanArgs &a, int team_warps, int device)
{
    long long t = 0;
    if (dispatch_scan(a, team_warps, nullptr, device, &t, true) != cudaSuccess) return -1;
    return t;
}

// Model-major launch: one work item per (model, block of kModelRows wavelengths); one CTA per
// SM with as many warps as fit beside the table (up to kModelsBlock / 32, at least
// kModelsMinWarps; 0 = the caches do not fit).
static int models_warps(int N, int device)
{
    const size_t static_smem = 16;
    const size_t optin = smem_optin_limit(device);
    if (optin < kExpTabBytes + static_smem) return 0;
    const size_t w = (optin - kExpTabBytes - static_smem) / (size_t)warp_model_bytes(N);
    const int warps = (int)std::min<size_t>(w, (size_t)(kModelsBlock / 32));
    return warps >= kModelsMinWarps ? warps : 0;
}

static cudaError_t launch_models(const ScanArgs &a, cudaStream_t st, int device,
                                 long long *warps_out, bool dry, int *per_sm_out = nullptr)
{
    const int wpc = models_warps(a.mod.N, device);
    const size_t smem = kExpTabBytes + (size_t)wpc * (size_t)warp_model_bytes(a.mod.N);
    auto kern = a.stable ? scan_models_kernel<true, unsigned> : scan_models_kernel<false, unsigned>;
    auto kfine = scan_models_kernel<false, FineTab>;   // (see tab_mismatch)
    const int sms = sm_count(device);
    const long long key = ((long long)device << 48) | (1ll << 47) | (a.stable ? (1ll << 46) : 0ll) |
                          ((long long)wpc << 32) |
                          (long long)smem;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        auto it = g_occ_cache.find(key);
        if (it != g_occ_cache.end()) per_sm = it->second;
    }
    if (per_sm == 0) {
        // a cache that does not fit is "0 CTAs per SM", not an error (and must not leave a
        // pending runtime error for the next launch's cudaGetLastError)
        if (wpc == 0) {
            per_sm = -1;
        } else {
            if (ensure_smem_optin(kern, device, a.stable ? 5 : 1) != cudaSuccess ||
                (!a.stable && ensure_smem_optin(kfine, device, 8) != cudaSuccess)) {
                cudaGetLastError();
                per_sm = -1;
            } else if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpc,
                                                                     smem) != cudaSuccess) {
                cudaGetLastError();
                per_sm = -1;
            }
            if (per_sm == 0) per_sm = -1;
        }
        std::lock_guard<std::mutex> g(g_cache_mu);
        g_occ_cache[key] = per_sm;
    }
    if (per_sm < 0) per_sm = 0;
    if (per_sm_out) *per_sm_out = per_sm;
    if (per_sm == 0) return cudaErrorInvalidConfiguration;
    const int64_t items = a.mod.M * ((a.L + kModelRows - 1) / kModelRows);
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (items + wpc - 1) / wpc;
    if (need < blocks) blocks = need;
    if (blocks < 1) blocks = 1;
    if (warps_out) *warps_out = blocks * wpc;
    if (dry) return cudaSuccess;
    // Tail: a work item (one model's wavelengths) takes a warp ~1 ms on C5, so the warps
    // finished up to one item apart (measured: 0.55 ms average idle, 1.4 % of the scan).  The
    // last kTailItemsPerWarp items per warp are queued as kTailRows-wavelength pieces.
    ScanArgs b = a;
    b.tail_models = 0;
    b.tail_rows = 0;
    if (a.L > kTailRows) {
        b.tail_models = std::min<int64_t>(a.mod.M, kTailItemsPerWarp * blocks * wpc);
        b.tail_rows = kTailRows;
    }
    kern<<<(unsigned)blocks, 32 * wpc, smem, st>>>(b);
    count_launch();
    if (!a.stable) {
        kfine<<<(unsigned)blocks, 32 * wpc, smem, st>>>(b);
        count_launch();
    }
    return cudaGetLastError();
}

bool models_scan_suitable(const ScanArgs &a, int device, bool forced)
{
    // unless forced: enough work items to fill the GPU several times over and several
    // wavelengths per model to share the cache; and one CTA per SM of >= kModelsMinWarps
    // warps with the table and the per-warp caches must fit (16 warps for N <= 6, 14 for
    // N = 7, 12 for N = 8)
    const int64_t items = a.mod.M * ((a.L + kModelRows - 1) / kModelRows);
    const int sms = sm_count(device);
    if (a.sched != 0) return false;
    // (>= 2 items per resident warp: measured crossover with the pair scan at ~2.1 on C5-like
    // ensembles, scripts/ens_small.py)
    if (!forced && (items < 2ll * sms * 16 || a.L < 8)) return false;
    int per_sm = 0;
    long long w = 0;
    if (launch_models(a, nullptr, device, &w, true, &per_sm) != cudaSuccess) return false;
    return per_sm >= 1;
}

// Pair scan launcher: single curves (M == 1) of many wavelengths.  *warps_out: warps launched.
// Combine the tail segments of each tail row (Algorithm 1 over the segment records in
// velocity order), one warp per row, 32 segments per step: segment sg holds the row's first
// event iff it is the first segment with an event -- a non-finite det at its first point, a
// first sign different from the previous segment's last sign, or an in-segment event (the
// segments before the first event were all written: a segment is skipped only after an
// earlier one found an event).  Writes C_t / idx and the work counters of the tail rows.
constexpr int kCombineBlock = 256;
__global__ void __launch_bounds__(kCombineBlock) pair_tail_combine_kernel(ScanArgs a)
{
    Workspace *ws = a.ws;
    if (ws_invalid(ws, a.grid_mask, true)) return;
    const int64_t M = a.mod.M, L = a.L, V = a.V;
    const int64_t P = M * ((L + 1) / 2), Pt = a.tail_pairs, Ph = P - Pt;
    const int S = a.seg_count, SEGV = a.seg_len;
    const double *__restrict__ cg = a.c;
    const int lane = threadIdx.x & 31;
    const int64_t tq = ((int64_t)blockIdx.x * kCombineBlock + threadIdx.x) >> 5;   // warp: row
    unsigned long long alg = 0;
    unsigned status = 0;
    if (tq < 2 * Pt) {
        const int64_t pi = Ph + tq / 2;
        const int64_t ip = pi / M, m = pi - ip * M;
        const int64_t i = 2 * ip + (tq & 1);
        const int64_t r = m * L + i;
        const bool live = i < L && !(a.pstart && a.pstart[r] < 0);   // else: none / prefix row
        if (live) {
            int evj = -1;
            bool evb = false;
            int prev_ls = 0;   // the last sign of the segment before this step's first one
            for (int s0 = 0; s0 < S && s0 * SEGV < V; s0 += 32) {
                const int sg = s0 + lane;
                const int lo = sg * SEGV;
                const bool in = sg < S && lo < V;
                const int2 rec = in ? a.seg_rec[tq * S + sg] : make_int2(-1, 0);
                const int fs = (rec.y & 3) - 1, ls = ((rec.y >> 2) & 3) - 1;
                int pls = __shfl_up_sync(FULL, ls, 1);
                if (lane == 0) pls = prev_ls;
                // this segment's event, in the precedence of Algorithm 1 over its points: a
                // non-finite det at the first point, a change across the boundary, an
                // in-segment event (rec.x: -1 or in [lo, lo + SEGV))
                const bool rb = (rec.y >> 4) & 1;
                int cj = -1;
                bool cb = false;
                if (in) {
                    if (rec.x == lo) {
                        cj = lo;
                        cb = rb;
                    } else if (sg > 0 && fs != pls) {
                        cj = lo;
                    } else if (rec.x > lo) {
                        cj = rec.x;
                        cb = rb;
                    }
                }
                const unsigned mk = __ballot_sync(FULL, cj >= 0);
                if (mk) {
                    const int src = __ffs(mk) - 1;
                    evj = __shfl_sync(FULL, cj, src);
                    evb = __shfl_sync(FULL, (int)cb, src) != 0;
                    break;
                }
                prev_ls = __shfl_sync(FULL, ls, 31);
            }
            if (lane == 0) {
                if (evj >= 0) {
                    if (evb) {
                        a.ct[r] = __longlong_as_double(0x7ff8000000000000ll);
                        if (a.idx) a.idx[r] = -2;
                        status |= 2u;
                    } else {
                        a.ct[r] = cg[evj];
                        if (a.idx) a.idx[r] = evj;
                    }
                    alg = (unsigned long long)(evj + 1);
                } else {
                    a.ct[r] = __longlong_as_double(0x7ff8000000000000ll);
                    if (a.idx) a.idx[r] = -1;
                    status |= 1u;
                    alg = (unsigned long long)V;
                }
            }
        }
    }
    alg = warp_sum_u64(alg);
    status = __reduce_or_sync(FULL, status);
    if (lane == 0) {
        if (alg) atomicAdd(&ws->alg_dets, alg);
        if (status) atomicOr(&ws->row_status, status);
    }
}

// Tail segments of the pair scan: the pair items of the last (partial) round -- all of them
// when there are fewer pairs than warps -- are split into velocity segments (a multiple of 32
// grid points each), about 8 per warp in total.
struct PairTail {
    int64_t pairs;
    int count, len;
};

static PairTail pair_tail_plan(const ScanArgs &a, int64_t warps)
{
    PairTail t{0, 0, 0};
    const int64_t P = a.mod.M * ((a.L + 1) / 2);
    if (warps < 2 || a.V < 64) return t;
    // tail = the pairs of the last, partial round (P mod warps; all pairs when P <= warps),
    // in about 8 segments per warp.  Measured on C3 (profiles/r2/pair_tail_sweep.txt, same box): no
    // tail 6.14 ms; partial round 5.23 ms (4 segments per warp: 5.29, 16: 5.21); half a round
    // of warps: 5.38-5.94; a full round: 5.44-6.44 (more speculative segments past the
    // change).  C4 (lengths sorted longest first): 1.75 -> 1.71-1.74 ms either way.
    constexpr double kPerWarp = 8.0;
    int64_t Pt = P % warps;
    if (P <= warps) Pt = P;
    if (Pt < 1) return t;
    const int64_t chunks = (a.V + 31) / 32;
    int64_t S = (int64_t)((kPerWarp * (double)warps + (double)Pt - 1) / (double)Pt);
    S = std::max<int64_t>(1, std::min<int64_t>(S, chunks));
    if (S < 2) return t;   // no split: whole pairs
    const int64_t len = ((chunks + S - 1) / S) * 32;
    t.pairs = Pt;
    t.len = (int)len;
    t.count = (int)((a.V + len - 1) / len);
    return t;
}

static cudaError_t launch_pairs(const ScanArgs &a, cudaStream_t st, int device,
                                long long *warps_out, bool dry, void *scratch = nullptr,
                                size_t *scratch_bytes = nullptr)
{
    const size_t smem = pair_smem_bytes(a.mod.N);
    auto kern = a.stable ? scan_pair_kernel<true, unsigned> : scan_pair_kernel<false, unsigned>;
    auto kfine = scan_pair_kernel<false, FineTab>;   // (see tab_mismatch)
    const int sms = sm_count(device);
    const long long key = ((long long)device << 48) | (2ll << 44) | (a.stable ? (1ll << 43) : 0ll) |
                          (long long)smem;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        auto it = g_occ_cache.find(key);
        if (it != g_occ_cache.end()) per_sm = it->second;
    }
    if (per_sm == 0) {
        if (ensure_smem_optin(kern, device, a.stable ? 6 : 4) != cudaSuccess ||
            (!a.stable && ensure_smem_optin(kfine, device, 9) != cudaSuccess) ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPairBlock, smem) !=
                cudaSuccess) {
            cudaGetLastError();
            per_sm = -1;
        }
        if (per_sm == 0) per_sm = -1;
        std::lock_guard<std::mutex> g(g_cache_mu);
        g_occ_cache[key] = per_sm;
    }
    if (per_sm < 0) return cudaErrorInvalidConfiguration;
    const int wpc = kPairBlock / 32;
    const int64_t full = (int64_t)sms * per_sm;
    const PairTail tail = pair_tail_plan(a, full * wpc);
    const int64_t P = a.mod.M * ((a.L + 1) / 2);
    const int64_t items = P - tail.pairs + tail.pairs * tail.count;
    int64_t blocks = full;
    const int64_t need = (items + wpc - 1) / wpc;
    if (need < blocks) blocks = need;
    if (blocks < 1) blocks = 1;
    if (warps_out) *warps_out = blocks * wpc;
    const size_t found_bytes = (size_t)(2 * tail.pairs) * sizeof(int);
    const size_t rec_off = (found_bytes + 15) & ~(size_t)15;
    const size_t need_bytes = tail.pairs ? rec_off + (size_t)(2 * tail.pairs) * tail.count * sizeof(int2)
                                         : 0;
    if (scratch_bytes) *scratch_bytes = need_bytes;
    if (dry) return cudaSuccess;
    ScanArgs b = a;
    b.tail_pairs = 0;
    b.seg_count = 0;
    b.seg_len = 0;
    b.seg_found = nullptr;
    b.seg_rec = nullptr;
    if (tail.pairs && scratch) {
        b.tail_pairs = tail.pairs;
        b.seg_count = tail.count;
        b.seg_len = tail.len;
        b.seg_found = static_cast<int *>(scratch);
        b.seg_rec = reinterpret_cast<int2 *>(static_cast<unsigned char *>(scratch) + rec_off);
        cudaError_t e = cudaMemsetAsync(b.seg_found, 0x7f, found_bytes, st);   // "no event yet"
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)blocks, kPairBlock, smem, st>>>(b);
    count_launch();
    if (!a.stable) {
        kfine<<<(unsigned)blocks, kPairBlock, smem, st>>>(b);
        count_launch();
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !b.tail_pairs) return e;
    pair_tail_combine_kernel<<<(unsigned)((2 * b.tail_pairs * 32 + kCombineBlock - 1) / kCombineBlock),
                               kCombineBlock, 0, st>>>(b);
    count_launch();
    return cudaGetLastError();
}

bool pairs_scan_suitable(const ScanArgs &a, int device, bool forced)
{
    // the queue schedule; unless forced: at least 4 rows per resident warp (the row scan's
    // TEAM = 1 regime; shorter curves want teams for latency)
    if (a.sched != 0 || a.pivoted || a.L < 2) return false;
    if (!forced && a.mod.M * a.L < 4ll * sm_count(device) * (kPairBlock / 32)) return false;
    long long w = 0;
    return launch_pairs(a, nullptr, device, &w, true) == cudaSuccess;
}

size_t pair_tail_scratch_bytes(const ScanArgs &a, int device)
{
    size_t bytes = 0;
    long long w = 0;
    if (launch_pairs(a, nullptr, device, &w, true, nullptr, &bytes) != cudaSuccess) return 0;
    return bytes;
}

cudaError_t launch_scan_pairs(const ScanArgs &a, void *tail_scratch, cudaStream_t st, int device,
                              long long *warps_out)
{
    return launch_pairs(a, st, device, warps_out, false, tail_scratch);
}

long long scan_pairs_warps(const ScanArgs &a, int device)
{
    long long w = 0;
    if (launch_pairs(a, nullptr, device, &w, true) != cudaSuccess) return -1;
    return w;
}

cudaError_t launch_scan_models(const ScanArgs &a, cudaStream_t st, int device,
                               long long *warps_out)
{
    return launch_models(a, st, device, warps_out, false);
}

long long scan_models_warps(const ScanArgs &a, int device)
{
    long long w = 0;
    if (launch_models(a, nullptr, device, &w, true) != cudaSuccess) return -1;
    return w;
}

// ------------------------------------------------------------------ misfit (Algorithm 2)

__global__ void __launch_bounds__(256) misfit_kernel(const double *__restrict__ ct,
                                                     const double *__restrict__ ce, int64_t M,
                                                     int64_t L, double *__restrict__ out,
                                                     const Workspace *ws, unsigned grid_mask,
                                                     bool check_models)
{
    if (ws_invalid(ws, grid_mask, check_models)) return;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= M) return;
    const double *row = ct + wid * L;
    double s = 0.0;
    bool inf = false;
    for (int64_t i = lane; i < L; i += 32) {
        const double x = row[i];
        if (!isfinite(x)) inf = true;
        else s += fabs(x - ce[i]) / ce[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    inf = __any_sync(FULL, inf);
    if (lane == 0) out[wid] = inf ? INFINITY : s / (double)L;
}

cudaError_t launch_misfit(const double *ct, const double *ce, int64_t M, int64_t L,
                          double *misfit, Workspace *ws, unsigned grid_mask, bool check_models,
                          cudaStream_t st)
{
    const int64_t blocks = (M * 32 + 255) / 256;
    misfit_kernel<<<(unsigned)blocks, 256, 0, st>>>(ct, ce, M, L, misfit, ws, grid_mask,
                                                    check_models);
    count_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------ argmin

__global__ void __launch_bounds__(1024) argmin_kernel(const double *__restrict__ v, int64_t M,
                                                      int64_t *best, double *best_val)
{
    __shared__ double sv[32];
    __shared__ long long si[32];
    double bv = INFINITY;
    long long bi = -1;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
        double x = v[i];
        if (isnan(x)) x = INFINITY;
        if (bi < 0 || x < bv) {   // ascending i per thread: strict < keeps the lowest index
            bv = x;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const long long oi = __shfl_xor_sync(FULL, bi, o);
        if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) {
            bv = ov;
            bi = oi;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        bv = lane < nw ? sv[lane] : INFINITY;
        bi = lane < nw ? si[lane] : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv, o);
            const long long oi = __shfl_xor_sync(FULL, bi, o);
            if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            *best = bi;
            if (best_val) *best_val = bv;
        }
    }
}

cudaError_t launch_argmin(const double *misfit, int64_t M, int64_t *best, double *best_val,
                          cudaStream_t st)
{
    argmin_kernel<<<1, 1024, 0, st>>>(misfit, M, best, best_val);
    count_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------ det grid (debug)

template <bool STABLE>
__global__ void __launch_bounds__(256) det_grid_kernel(ModelArgs mod, const double *lam,
                                                       int64_t L, const double *c, int64_t V,
                                                       double *mre, double *mim, int32_t *ex,
                                                       const Workspace *ws, bool prefix)
{
    extern __shared__ __align__(16) unsigned char smem[];
    if (ws_invalid(ws, 0x1Fu | (STABLE ? kGridStable : 0u), true)) return;
    unsigned char *tab = smem;
    exp_scale_fill(tab, ws_exp_rows(ws));
    const int N = mod.N;
    LayerConst *lc = reinterpret_cast<LayerConst *>(smem + kExpTabBytes);
    double *vel = reinterpret_cast<double *>(smem + kExpTabBytes + (size_t)(N + 1) * sizeof(LayerConst));
    const int64_t i = blockIdx.y;
    const double k = kTwoPi / lam[i];
    for (int e = threadIdx.x; e <= N; e += blockDim.x) {
        const double al = mod.alpha[e], be = mod.beta[e], rh = mod.rho[e];
        LayerConst x;
        x.kh = (e < N) ? k * mod.h[e] : 0.0;
        x.ia2 = 1.0 / (al * al);
        x.ib2 = 1.0 / (be * be);
        x.krho = k * rh;
        x.b2 = 2.0 * (be * be);      // mu = (k rho) beta^2 (lc_mu), as layer_elem_root forms it
        x.aux = 0.0;
        lc[e] = x;
        vel[2 * e] = al;
        vel[2 * e + 1] = be;
    }
    __syncthreads();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    // the scans' small-c rule (reading S15''): the stable element where c_j^4 < Q
    const double cj2 = c[j] * c[j];
    const DetOut d = (STABLE || (prefix && cj2 * cj2 < smallc_q(mod, 0, k)))
                         ? det_K<true, 0, true>(lc, vel, smem_addr(tab), N, c[j])
                         : det_K<true, 0, false>(lc, vel, smem_addr(tab), N, c[j]);
    const int64_t o = i * V + j;
    mre[o] = d.mre;
    mim[o] = d.mim;
    ex[o] = d.e2;
}

cudaError_t launch_det_grid(const ModelArgs &m, const double *lam, int64_t L, const double *c,
                            int64_t V, double *mre, double *mim, int32_t *ex, Workspace *ws,
                            cudaStream_t st, bool stable, bool prefix)
{
    const size_t smem = kExpTabBytes + team_model_bytes(m.N);
    int dev = 0;
    cudaGetDevice(&dev);   // the C-ABI's DeviceScope has made the call's device current
    auto kern = stable ? det_grid_kernel<true> : det_grid_kernel<false>;
    cudaError_t e = ensure_smem_optin(kern, dev, stable ? 3 : 2);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((V + 255) / 256), (unsigned)L);
    kern<<<grid, 256, smem, st>>>(m, lam, L, c, V, mre, mim, ex, ws, prefix);
    count_launch();
    return cudaGetLastError();
}

}  // namespace masw
