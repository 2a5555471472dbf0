// masw_det.cuh -- per-(lambda, c) stiffness determinant, assembled and eliminated in
// registers (sm_100a).  Product code; shares nothing with oracle/.
//
// What it computes (readings S1-S16 in DESIGN.md):
//   K(k, c) of order 2(N+1) is the sum of N Kausel-Roesset 4x4 layer elements overlapping
//   in 2x2 blocks plus the 2x2 half-space element, i.e. a symmetric 2x2 BLOCK-TRIDIAGONAL
//   matrix (the paper's "heptadiagonal" band, reading S10):
//       A_i = bottom(layer i-1) + top(layer i) (+ K_hs at i = N),  B_i = coupling of layer i.
//   det K is computed by banded Gaussian elimination with partial pivoting streamed node by
//   node (a 4-row window, reading S10/S11), O(N) per determinant.
//   Unpivoted 2x2-block elimination (det K = prod det S_i) was the first design; it loses
//   up to ~1e-7 relative next to a layer's clamped-layer pole (D -> 0), where the element
//   entries grow like 1/D and cancel; partial pivoting keeps the oracle's ~1e-11 accuracy.
//
// Arithmetic design (B200):
//   * Every layer entry is an even function of r and s, hence exactly REAL for real (k, c)
//     (reading S3/S5): each wave contributes the real triple (C, x*S, S/x) =
//        (cosh th, x sinh th, sinh th / x),  x = sqrt(1 - c^2/v^2),   th = k h x   (x real)
//        (cos th, -xi sin th, sin th / xi),  xi = sqrt(c^2/v^2 - 1),  th = k h xi  (x = i xi)
//     so every pivot is real fp64; only the last node's columns (with the half-space) are
//     complex, and only when c > beta_N.
//   * Nothing is stored: K never exists in memory (the paper kept 3136 B per matrix in
//     global memory).  The elimination window is 2 leftover rows x 4 columns
//     in registers; parameters come from shared memory (broadcast).
//   * The sign of Re det K is the product of the pivot signs, the permutation parity and
//     sgn Re det(last 2x2), so the scan never multiplies determinants and cannot overflow
//     (reading S14).
#pragma once

#include <cstdint>

#include "masw_exp_table.h"

#ifndef MASW_LAYER_UNROLL
#define MASW_LAYER_UNROLL 1
#endif

namespace masw {

constexpr double kTwoPi = 6.283185307179586;   // reading S2 / O1
constexpr double kMaxKH = 350.0;               // reading S9 range guard
constexpr double kPerturbTol = 1e-4;           // reading S4
constexpr double kPerturbFactor = 1.0 - 1e-4;  // reading S4

// Per-row constants of one finite layer e (index N holds the half-space's ia2, ib2, krho,
// b2).  48 bytes, 16-byte aligned: read from shared memory as three 128-bit loads.
struct __align__(16) LayerConst {
    double kh;    // k * h_e
    double ia2;   // 1 / alpha_e^2
    double ib2;   // 1 / beta_e^2
    double krho;  // k * rho_e
    double b2;    // 2 beta_e^2  (mu = k rho_e beta_e^2 = krho * (b2 / 2), exactly: lc_mu)
    double aux;   // scans only (else 0): e < N: rho_e / rho_(e+1); e = N: rho_N beta_N^2 / rho_(N-1)
};
static_assert(sizeof(LayerConst) == 48, "LayerConst layout");

// mu = (k) rho beta^2, bitwise equal to krho * (beta * beta): b2 / 2 = beta^2 exactly
__device__ __forceinline__ double lc_mu(const LayerConst &L) { return L.krho * (0.5 * L.b2); }

__device__ __forceinline__ LayerConst load_lc(const LayerConst *p)
{
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = q[0], b = q[1], c = q[2];
    LayerConst L;
    L.kh = a.x;
    L.ia2 = a.y;
    L.ib2 = b.x;
    L.krho = b.y;
    L.b2 = c.x;
    L.aux = c.y;
    return L;
}

// -------------------------------------------------------------- fp64 elementary functions
// Written for this kernel's argument ranges (all inputs finite and normal; see each function)
// so that none of them needs the special-case branches of the general libm routines, and
// with polynomial coefficients in the constant bank (DFMA takes them as c[][] operands; the
// libm versions spend two UMOV issue slots per coefficient).  Each is within ~1-2 ulp.
//
// Near-minimax (Chebyshev-fitted, coefficients rounded to fp64; scripts/minimax_coeffs.py)
// polynomials in u = r^2, highest degree first.  Max relative error with these fp64
// coefficients (50-digit check): sin(r)/r 1.3e-17 and cos(r) 7.2e-18 on |r| <= pi/4.
// (cosh/sinh: masw_exp_table.h.)
static __constant__ double c_sin[6] = {1.5894736651849094e-10, -2.5050716974102745e-08,
                                       2.755731337640013e-06, -0.000198412698286503,
                                       0.008333333333320363, -0.16666666666666616};
static __constant__ double c_cos[7] = {-1.1353379638297575e-11, 2.0875582380663952e-09,
                                       -2.7557313097790086e-07, 2.4801587283881152e-05,
                                       -0.0013888888888861095, 0.04166666666666645, -0.5};

constexpr double kShifter = 6755399441055744.0;         // 1.5 * 2^52: round-to-integer trick
// Split constants whose leading part has <= 21 significant bits (low word zero), so the
// leading part is an instruction immediate (no register materialisation) and n * part is
// exact for the n that occur; the trailing parts come from the constant bank (c_k).
constexpr double kPio2Hi = 1.570796012878418;           // pi/2 = kPio2Hi + c_k[1] + c_k[2]
static __constant__ double c_k[4] = {
    0.6366197723675814,        // 0: 2 / pi
    3.139164786504813e-07,     // 1: pi/2 - kPio2Hi (53 bits)
    1.0562999066987428e-23,    // 2: the rest (residual 5e-40)
    0.375,                     // 3: rsqrt correction coefficient
};

// cosh/sinh reconstruction table (masw_exp_table.h, generated, correctly rounded): a
// per-CTA copy at the start of the kernel's dynamic shared memory -- (cosh(m d), sinh(m d))
// for m < 5680 (d = 1/16: th < 354.97), 89 KB, read without a branch.  exp_scale_fill()
// copies only the rows the launch can reach (m <= kh_max / d + 1, kh_max = max k h over the
// call's rows and layers).  Lanes of a warp hold neighbouring velocities, so their m mostly
// coincide (broadcast reads).
// shared-memory bytes reserved for the table (the larger of the coarse and fine ones)
constexpr unsigned kExpTabBytes = (kExpTabN > kExpTabNF ? kExpTabN : kExpTabNF) * 16u;

// The fine variant of the table (g_cosh_sinh_fine: d = 1/128, th < 50.55) and its element
// functions are used for calls whose largest k h is at most kFineKhMax: every wave argument
// th = k h x is below k h (x = sqrt(1 - c^2/v^2) < 1), so the fine table covers it.  The
// scans choose per call from the validation pass (ws_fine), all of them by the same test, so
// they stay bitwise identical to one another.  (The scaled elements of MASW_STABLE reach
// th = 354 and always use the coarse table.)
#ifndef MASW_FINE_KH_MAX
#define MASW_FINE_KH_MAX 50.5
#endif
constexpr double kFineKhMax = MASW_FINE_KH_MAX;
struct FineTab {
    unsigned a;   // 32-bit shared address of the fine rows
};
template <class TabT> struct TabTraits {
    static constexpr double inv_d = kExpInvD;
    static constexpr int n = kExpTabN;
    static __device__ __forceinline__ const double2 *rows() { return g_cosh_sinh; }
    static __device__ __forceinline__ unsigned make(unsigned a) { return a; }
};
template <> struct TabTraits<FineTab> {
    static constexpr double inv_d = kExpFInvD;
    static constexpr int n = kExpTabNF;
    static __device__ __forceinline__ const double2 *rows() { return g_cosh_sinh_fine; }
    static __device__ __forceinline__ FineTab make(unsigned a) { return FineTab{a}; }
};

// rows of the table a launch can reach (m <= kh_max / d + 1)
template <class TabT = unsigned>
__device__ __forceinline__ int exp_rows_needed(double kh_max)
{
    constexpr int n = TabTraits<TabT>::n;
    const double m = kh_max * TabTraits<TabT>::inv_d + 2.0;
    return (m < (double)n) ? (int)m : n;   // (NaN -> all rows)
}

template <class TabT = unsigned>
__device__ __forceinline__ void exp_scale_fill(void *tab, int rows)
{
    double2 *t2 = reinterpret_cast<double2 *>(tab);
    const double2 *src = TabTraits<TabT>::rows();
    for (int m = threadIdx.x; m < rows; m += blockDim.x) t2[m] = src[m];
}

// Shared-memory addressing with 32-bit shared-window addresses held in registers.  The
// compiler otherwise re-derives the (cluster-qualified) shared address of a table or a
// per-warp array from special registers and the launch parameters at every use inside the
// hot loop (measured: ~25 integer instructions per node in the model-major kernel).
// opaque() hides a value's origin so it stays in a register; its memory clobber also orders
// the loads below after the stores that filled the memory.
__device__ __forceinline__ unsigned smem_addr(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned opaque(unsigned x)
{
    asm volatile("" : "+r"(x) : : "memory");
    return x;
}
__device__ __forceinline__ double2 lds_v2(unsigned a)
{
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a)
{
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a)
{
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_s32(unsigned a, int v)
{
    asm volatile("st.shared.s32 [%0], %1;" : : "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int lds_s8(unsigned a)
{
    int v;
    asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_s8(unsigned a, int v)
{
    asm volatile("st.shared.s8 [%0], %1;" : : "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ LayerConst load_lc_at(unsigned a)
{
    const double2 p = lds_v2(a), q = lds_v2(a + 16), r = lds_v2(a + 32);
    LayerConst L;
    L.kh = p.x;
    L.ia2 = p.y;
    L.ib2 = q.x;
    L.krho = q.y;
    L.b2 = r.x;
    L.aux = r.y;
    return L;
}

// The cosh/sinh table (below) as the element functions read it: a 32-bit shared-memory
// address (every scan copies the table into shared memory).
__device__ __forceinline__ double2 tab_load(unsigned tab, unsigned m) { return lds_v2(tab + m * 16u); }

// The MUFU fp64 seeds (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64) have relative error
// e <= 2^-20.1 on sm_100a (scripts/mufu_accuracy.cu, measured on B200), so ONE higher-order
// correction reaches full precision: its truncation error is O(e^3) ~ 2^-60.

// 1/x for finite normal x: y0 (1 + e + e^2), e = 1 - x y0 (max 0.999 * 2^-53 relative,
// measured; the same as two Newton steps, one DFMA fewer).  0 -> NaN (callers guard).
__device__ __forceinline__ double rcp_fast(double x)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}

// 1/sqrt(q) for finite q > 0: y0 (1 + e/2 + 3e^2/8), e = 1 - q y0^2 (max 1.005 * 2^-53
// relative, measured; two Newton steps give 1.24 * 2^-53 in eight FP64 ops, this five).
__device__ __forceinline__ double rsqrt_fast(double q)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
    const double e = fma(-q * y, y, 1.0);
    return fma(y * e, fma(e, c_k[3], 0.5), y);
}

// sqrt(q) and 1/sqrt(q) for finite q > 0: x = q * (1/sqrt q) (~1.5 ulp).  No residual
// correction: det K is ~1e4 times less sensitive to 1-ulp errors in the square roots r, s
// than to errors in the cosh values (kappa analysis, reading S15'), measured per term.
__device__ __forceinline__ void sqrt_rsqrt(double q, double &x, double &rx)
{
    rx = rsqrt_fast(q);
    x = q * rx;
}

// cosh and sinh of th in [0, 350] (the range guard S9 bounds k h_e by 350 and x <= 1).
// th = m d + r with d = 1/16 (m = round(16 th); r = th - m/16 is exact), |r| <= 1/32; with
// A = cosh(m d), B = sinh(m d) from the table and E = cosh r - 1, O = sinh r (near-minimax
// polynomials in r^2: degree 2 for E / r^2, abs. err of E < 8e-19; degree 3 for O / r, rel.
// err < 5e-20):
//   cosh th = A (1 + E) + B O,   sinh th = B (1 + E) + A O.
// At m = 0 (A = 1, B = 0) sinh th = O exactly structured (no cancellation at small th); for
// m >= 1, B and A O do not cancel (th >= m d / 2).  15 FP64 operations, no branch (the
// table covers th < 354.97; the index is clamped so a NaN argument stays in bounds).
template <class TabT>
__device__ __forceinline__ void cosh_sinh(double th, double &ch, double &sh, TabT tab)
{
    // th + 1.5 * 2^52 d rounds th to the nearest multiple of d (ulp d); its low word is m.
    // Three DADDs with immediate operands (no constant materialisation); r is exact
    // (md is within a factor 2 of th, or 0).
    static_assert(kExpD * 16.0 == 1.0, "shifter below assumes d = 1/16");
    constexpr double kShifterD = kShifter * kExpD;        // 1.5 * 2^48 (low word zero)
    const double t = th + kShifterD;
    const double md = t - kShifterD;                       // m d
    const unsigned m = min((unsigned)__double2loint(t), (unsigned)(kExpTabN - 1));
    const double r = th - md;                              // exact
    const double u = r * r;
    double pe = fma(kExpE2_0, u, c_expE2[1]);              // E / r^2
    double po = fma(kExpO3_0, u, c_expO3[1]);              // O / r
    pe = fma(pe, u, c_expE2[2]);
#pragma unroll
    for (int i = 2; i < 4; ++i) po = fma(po, u, c_expO3[i]);
    const double E = pe * u, O = po * r;
    const double2 ab = tab_load(tab, m);
    const double A = ab.x, B = ab.y;
    ch = fma(A, E, fma(B, O, A));
    sh = fma(B, E, fma(A, O, B));
}

// The fine variant (FineTab: calls with k h <= kFineKhMax, see there): d = 1/128, |r| <= 1/256,
// E = u (c0 u + c1) and O = r (c0' u^2 + c1' u + 1) (masw_exp_table.h: the same accuracy as
// the coarse polynomials above): 13 FP64 operations instead of 15.
__device__ __forceinline__ void cosh_sinh_fine(double th, double &ch, double &sh, unsigned tab)
{
    constexpr double kShifterF = kShifter * kExpFD;       // 1.5 * 2^45 (low word zero)
    const double t = th + kShifterF;
    const double md = t - kShifterF;                       // m d
    const unsigned m = min((unsigned)__double2loint(t), (unsigned)(kExpTabNF - 1));
    const double r = th - md;                              // exact
    const double u = r * r;
    const double pe = fma(kExpFE1_0, u, c_expFE1[1]);      // E / r^2
    double po = fma(kExpFO2_0, u, c_expFO2[1]);            // O / r
    po = fma(po, u, c_expFO2[2]);
    const double E = pe * u, O = po * r;
    const double2 ab = lds_v2(tab + m * 16u);
    const double A = ab.x, B = ab.y;
    ch = fma(A, E, fma(B, O, A));
    sh = fma(B, E, fma(A, O, B));
}

__device__ __forceinline__ void cosh_sinh(double th, double &ch, double &sh, FineTab tab)
{
    cosh_sinh_fine(th, ch, sh, tab.a);
}

// sin and cos of th in [0, 8e5] (< 2^19 pi/2: 3-part Cody-Waite reduction, the first product
// exact, each later step one rounding; near-minimax
// polynomials on |r| <= pi/4: sin to r^13, cos to r^14).  No branches; the caller
// routes larger arguments to sin_cos_large.
constexpr double kTrigMax = 8.0e5;

// Sign / range tests on the high word in the integer pipe (a DSETP occupies the FP64 pipe):
// is_pos(x) == (x > 0) for every x the scans test (nonzero by S4, or NaN -> either branch
// gives NaN); trig_fast(th) == (th < 2^19) for th >= 0 (NaN -> the large-argument path).
__device__ __forceinline__ bool is_pos(double x) { return __double2hiint(x) > 0; }
__device__ __forceinline__ bool trig_fast(double th)
{
    return (unsigned)__double2hiint(th) < 0x41200000u;   // 2^19 < kTrigMax
}
// pi/2 in five parts, the first four of <= 23 significant bits: n * part is exact for
// n < 2^30, so the large-argument reduction below is accurate for th < 2^30 * pi/2.
constexpr double kPio2L_1 = 1.570796251296997;
constexpr double kPio2L_2 = 7.549789415861596e-08;
constexpr double kPio2L_3 = 5.390302529957765e-15;
constexpr double kPio2L_4 = 3.2820036682434026e-22;
constexpr double kPio2L_5 = -1.2536990206932499e-29;

__device__ __forceinline__ void sin_cos_reduced(double r, int n, double &sn, double &cs);

__device__ __forceinline__ void sin_cos(double th, double &sn, double &cs)
{
    const double t = fma(th, c_k[0], kShifter);
    const double nd = t - kShifter;
    const int n = __double2loint(t);
    double r = fma(nd, -kPio2Hi, th);          // exact (n * kPio2Hi has <= 40 bits)
    r = fma(nd, -c_k[1], r);
    r = fma(nd, -c_k[2], r);
    sin_cos_reduced(r, n, sn, cs);
}

// Rare path: 8e5 <= th < 2^30 (c >~ 2000 times a layer's wave speed); NaN beyond.
static __device__ __noinline__ void sin_cos_large(double th, double &sn, double &cs)
{
    if (!(th < 1073741824.0)) {
        sn = cs = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    const double nd = rint(th * 0.6366197723675814);
    const int n = (int)nd;
    double r = th - nd * kPio2L_1;           // exact (Sterbenz)
    r = r - nd * kPio2L_2;
    r = r - nd * kPio2L_3;
    r = r - nd * kPio2L_4;
    r = fma(-nd, kPio2L_5, r);
    sin_cos_reduced(r, n, sn, cs);
}

__device__ __forceinline__ void sin_cos_reduced(double r, int n, double &sn, double &cs)
{
    const double r2 = r * r;
    double ps = c_sin[0];
    double pc = c_cos[0];
#pragma unroll
    for (int i = 1; i < 6; ++i) {
        ps = fma(ps, r2, c_sin[i]);
        pc = fma(pc, r2, c_cos[i]);
    }
    pc = fma(pc, r2, c_cos[6]);
    const double s = fma(r * r2, ps, r);
    const double c = fma(r2, pc, 1.0);
    // quadrant n mod 4: (sin, cos) = (s, c), (c, -s), (-s, -c), (-c, s)
    const bool swap = n & 1;
    const unsigned sgn_s = ((unsigned)n & 2u) << 30;         // sign bit for sin
    const unsigned sgn_c = ((unsigned)(n + 1) & 2u) << 30;   // sign bit for cos
    const double a = swap ? c : s;
    const double b = swap ? s : c;
    sn = __hiloint2double((int)((unsigned)__double2hiint(a) ^ sgn_s), __double2loint(a));
    cs = __hiloint2double((int)((unsigned)__double2hiint(b) ^ sgn_c), __double2loint(b));
}

// -------------------------------------------------------------- wave triples
// (C, XS, SX) of one wave: q = 1 - c^2/v^2 (!= 0 by S4) and kh = k*h; see header comment.
template <class TabT>
__device__ __forceinline__ void wave_hyp(double q, double kh, double &C, double &XS, double &SX,
                                         TabT tab)
{
    double x, rq;                      // x, 1/x
    sqrt_rsqrt(q, x, rq);
    double ch, sh;
    cosh_sinh(kh * x, ch, sh, tab);
    C = ch;
    XS = x * sh;
    SX = sh * rq;
}

__device__ __forceinline__ void wave_trig(double q, double kh, double &C, double &XS, double &SX)
{
    double xi, rq;                     // xi, 1/xi
    sqrt_rsqrt(-q, xi, rq);
    const double th = kh * xi;
    double sn, cs;
    if (trig_fast(th)) {
        sin_cos(th, sn, cs);
    } else {
        sin_cos_large(th, sn, cs);
    }
    C = cs;
    XS = -xi * sn;
    SX = sn * rq;
}

template <class TabT>
__device__ __forceinline__ void wave_triple(double q, double kh, double &C, double &XS,
                                            double &SX, TabT tab)
{
    if (q > 0.0) {
        wave_hyp(q, kh, C, XS, SX, tab);
    } else {
        wave_trig(q, kh, C, XS, SX);
    }
}

// -------------------------------------------------------------- perturbation (reading S4)
// while c' is within 1e-4 m/s of any alpha_e / beta_e (e = 0..N): c' *= (1 - 1e-4).
__device__ __forceinline__ double perturb_velocity(const double *__restrict__ vel, int nvel,
                                                   double c)
{
    for (;;) {
        bool near = false;
        for (int e = 0; e < nvel; ++e) near |= (fabs(c - vel[e]) < kPerturbTol);
        if (!near) return c;
        c = c * kPerturbFactor;
    }
}

// The same for velocities held as separate alpha[0..n) and beta[0..n) arrays (the result
// depends only on the set of velocities, so it equals perturb_velocity's bit for bit).
__device__ __forceinline__ double perturb_velocity_ab(const double *__restrict__ al,
                                                      const double *__restrict__ be, int n,
                                                      double c)
{
    for (;;) {
        bool near = false;
        for (int e = 0; e < n; ++e)
            near |= (fabs(c - al[e]) < kPerturbTol) | (fabs(c - be[e]) < kPerturbTol);
        if (!near) return c;
        c = c * kPerturbFactor;
    }
}

// -------------------------------------------------------------- layer element
// Six unique real entries of the Kausel-Roesset layer element (reading S1) from the wave
// triples: with (C, XS, SX) of the P (r) and S (s) waves,
//   D   = 2(1 - Cr Cs) + SXr SXs + XSr XSs,  f = k rho c^2 / D
//   k11 = f (Cr SXs - XSr Cs)    k12 = f (Cr Cs - XSr XSs - 1) - mu (1 + s^2)
//   k13 = f (XSr - SXs)          k14 = f (Cs - Cr)
//   k22 = f (SXr Cs - Cr XSs)    k24 = f (XSs - SXr)
// Element layout (DOFs u_top, w_top, u_bot, w_bot):
//   [[k11, k12, k13, k14], [k12, k22, -k14, k24], [k13, -k14, k11, -k12], [k14, k24, -k12, k22]]
// Evaluation: Cr Cs - 1 is one fused op (exact product, one rounding; it is -(1 - Cr Cs) in
// both D and k12), and mu (1 + s^2) = k rho (2 beta^2 - c^2) = 2 mu - k rho c^2 reuses k rho c^2.
struct Elem {
    double k11, k12, k13, k14, k22, k24;
};

__device__ __forceinline__ Elem elem_from_triples(double Cr, double XSr, double SXr, double Cs,
                                                  double XSs, double SXs, double krho, double mu,
                                                  double c2)
{
    const double cm1 = fma(Cr, Cs, -1.0);                              // Cr Cs - 1
    const double D = fma(XSr, XSs, fma(-2.0, cm1, SXr * SXs));
    const double kc2 = krho * c2;
    const double f = kc2 * rcp_fast(D);
    Elem E;
    E.k11 = f * fma(Cr, SXs, -XSr * Cs);
    E.k12 = fma(f, fma(-XSr, XSs, cm1), fma(-2.0, mu, kc2));
    E.k13 = f * (XSr - SXs);
    E.k14 = f * (Cs - Cr);
    E.k22 = f * fma(SXr, Cs, -Cr * XSs);
    E.k24 = f * (XSs - SXr);
    return E;
}

// The same element without its scalar factor, for the sign scan: E = f U with f = k rho c^2 / D
// and, since mu (1 + s^2) = k rho (2 beta^2 - c^2) = f D (2 beta^2 / c^2 - 1),
//   U = the element's brackets, with k12's  g12 = Cr Cs - XSr XSs - 1 + kappa D,
//   kappa = 1 - 2 beta^2 / c^2  (per layer and velocity; from b2 = 2 beta^2 and 1/c^2).
// No reciprocal and no scaling products: det_sign_block_u carries f through the recursion
// as ratios f_e / f_(e+1) = (rho_e / rho_(e+1)) D_(e+1) / D_e (rr = rho_e / rho_(e+1)).
struct ElemU {
    double g11, g12, g13, g14, g22, g24, D, rr;
};

__device__ __forceinline__ ElemU elemu_from_triples(double Cr, double XSr, double SXr, double Cs,
                                                    double XSs, double SXs, double kap, double rr)
{
    const double cm1 = fma(Cr, Cs, -1.0);                              // Cr Cs - 1
    ElemU U;
    U.D = fma(XSr, XSs, fma(-2.0, cm1, SXr * SXs));
    U.g11 = fma(Cr, SXs, -XSr * Cs);
    U.g12 = fma(kap, U.D, fma(-XSr, XSs, cm1));
    U.g13 = XSr - SXs;
    U.g14 = Cs - Cr;
    U.g22 = fma(SXr, Cs, -Cr * XSs);
    U.g24 = XSs - SXr;
    U.rr = rr;
    return U;
}

// kappa_e = 1 - 2 beta_e^2 / c^2
__device__ __forceinline__ double lc_kappa(const LayerConst &L, double ic2)
{
    return fma(-L.b2, ic2, 1.0);
}

// Rare case c > alpha_e (both waves possibly trigonometric): kept out of line so the hot
// loop's code stays small (instruction-cache pressure was measured: no_instruction stalls).
template <class TabT>
static __device__ __noinline__ void waves_general(double qa, double qb, double kh, double *t,
                                                  TabT tab)
{
    wave_triple(qa, kh, t[0], t[1], t[2], tab);
    wave_triple(qb, kh, t[3], t[4], t[5], tab);
}

template <class TabT>
__device__ __forceinline__ Elem layer_elem(const LayerConst &L, double c2,
                                           TabT tab)
{
    const double qa = fma(-c2, L.ia2, 1.0);   // r^2
    const double qb = fma(-c2, L.ib2, 1.0);   // s^2
    double Cr, XSr, SXr, Cs, XSs, SXs;
    // The P wave is hyperbolic unless c exceeds alpha (rare); each S-wave branch carries its
    // own branch-free copy of the P wave so the two independent chains interleave (ILP).
    if (is_pos(qa)) {
        if (is_pos(qb)) {
            wave_hyp(qa, L.kh, Cr, XSr, SXr, tab);
            wave_hyp(qb, L.kh, Cs, XSs, SXs, tab);
        } else {
            wave_hyp(qa, L.kh, Cr, XSr, SXr, tab);
            wave_trig(qb, L.kh, Cs, XSs, SXs);
        }
    } else {
        double t[6];
        waves_general(qa, qb, L.kh, t, tab);
        Cr = t[0]; XSr = t[1]; SXr = t[2];
        Cs = t[3]; XSs = t[4]; SXs = t[5];
    }
    return elem_from_triples(Cr, XSr, SXr, Cs, XSs, SXs, L.krho, lc_mu(L), c2);
}

// layer_elem without the factor f (ElemU; ic2 = 1/c^2 of the same c2).
template <class TabT>
__device__ __forceinline__ ElemU layer_elem_u(const LayerConst &L, double c2, double ic2,
                                              TabT tab)
{
    const double qa = fma(-c2, L.ia2, 1.0);   // r^2
    const double qb = fma(-c2, L.ib2, 1.0);   // s^2
    double Cr, XSr, SXr, Cs, XSs, SXs;
    if (is_pos(qa)) {
        if (is_pos(qb)) {
            wave_hyp(qa, L.kh, Cr, XSr, SXr, tab);
            wave_hyp(qb, L.kh, Cs, XSs, SXs, tab);
        } else {
            wave_hyp(qa, L.kh, Cr, XSr, SXr, tab);
            wave_trig(qb, L.kh, Cs, XSs, SXs);
        }
    } else {
        double t[6];
        waves_general(qa, qb, L.kh, t, tab);
        Cr = t[0]; XSr = t[1]; SXr = t[2];
        Cs = t[3]; XSs = t[4]; SXs = t[5];
    }
    return elemu_from_triples(Cr, XSr, SXr, Cs, XSs, SXs, lc_kappa(L, ic2), L.aux);
}

// -------------------------------------------------------------- stable element (f3)
// SURVEY.md §8(f) f3, opt-in (MASW_STABLE): an element evaluation without the two fp64
// failure modes of the direct App. A formulas (readings S9, S15):
//  * c -> 0 with both waves hyperbolic: D = 2(1 - Cr Cs) + Sr Ss (1/(rs) + rs) and the
//    entries' brackets are O(c^4) / O(c^2) differences of O(cosh^2) terms.  With
//    delta = (th_r - th_s)/2 = k h (r - s)/2, r - s = (b - a)/(r + s), w = 1 - rs =
//    (a + b - ab)/(1 + rs) (a = c^2/alpha^2, b = c^2/beta^2), the exact identities
//      D = -4 sinh^2(delta) + (w^2/(rs)) Sr Ss,
//      Cr Cs - rs Sr Ss - 1 = 2 sinh^2(delta) + w Sr Ss,
//      Cr Ss - rs Sr Cs = -sinh(2 delta) + w Sr Cs,   Sr Cs - rs Cr Ss = sinh(2 delta) + w Cr Ss,
//      Sr - Ss = 2 cosh(sigma) sinh(delta),  Cs - Cr = -2 sinh(sigma) sinh(delta),
//    (sigma = th_s + delta) turn every bracket into terms without cancellation at small c;
//  * thick layers (k h > 350, cosh overflow): every term carries e^(th_r + th_s) (or e^th_r
//    in the mixed case), so with scaled functions c^ = cosh(x) e^-x, s^ = sinh(x) e^-x and
//    e^-x the element is evaluated for k h up to 700 (range guard raised under MASW_STABLE).
// Validated against 50-digit mpmath (tests/test_gpu_stable.py), not the naive oracle.
constexpr double kMaxKHStable = 700.0;
constexpr double kExpSplit = 354.0;                      // within the cosh/sinh table
constexpr double kExpNeg354 = 0x1.381ea37bd35b3p-511;    // e^-354 (correctly rounded)

struct ExpScaled {
    double c, s, e;   // cosh(x) e^-x, sinh(x) e^-x, e^-x   (x in [0, 700])
};

template <class TabT>
__device__ __forceinline__ ExpScaled exp_scaled(double x, TabT tab)
{
    ExpScaled o;
    if (x <= kExpSplit) {
        double C, S;
        cosh_sinh(x, C, S, tab);
        o.e = rcp_fast(C + S);
        o.c = C * o.e;
        o.s = S * o.e;
    } else {   // e^-2x < 1e-307: c^ = s^ = 1/2 in fp64
        double C, S;
        cosh_sinh(x - kExpSplit, C, S, tab);
        o.e = rcp_fast(C + S) * kExpNeg354;
        o.c = 0.5;
        o.s = 0.5;
    }
    return o;
}

// Both waves hyperbolic (c < beta_e < alpha_e); entries as described above, all scaled by
// e^-(th_r + th_s) in numerator and denominator (f = f^ e^-(th_r + th_s)).
template <class TabT>
__device__ __forceinline__ Elem elem_stable_hh(double kh, double c2, double ia2, double ib2,
                                               double krho, double mu, TabT tab)
{
    const double a = c2 * ia2, b = c2 * ib2;
    double r, rr, s, rsn;
    sqrt_rsqrt(1.0 - a, r, rr);
    sqrt_rsqrt(1.0 - b, s, rsn);
    const double rs = r * s;
    const double w = fma(-a, b, a + b) * rcp_fast(1.0 + rs);          // 1 - rs
    const double dl = 0.5 * kh * ((b - a) * rcp_fast(r + s));          // (th_r - th_s)/2
    const ExpScaled R = exp_scaled(kh * r, tab), S = exp_scaled(kh * s, tab);
    const ExpScaled Dl = exp_scaled(dl, tab);
    const double es2 = S.e * S.e;                                      // e^-2 th_s
    const double sd2 = Dl.s * Dl.s;
    const double sdcd2 = 2.0 * Dl.s * Dl.c;
    const double csig = fma(S.c, Dl.c, S.s * Dl.s);                    // cosh(sigma) e^-sigma
    const double ssig = fma(S.s, Dl.c, S.c * Dl.s);                    // sinh(sigma) e^-sigma
    const double Dh = fma((w * w) * (rr * rsn), R.s * S.s, -4.0 * sd2 * es2);
    const double fh = (krho * c2) * rcp_fast(Dh);
    Elem E;
    E.k11 = (fh * rsn) * fma(w * R.s, S.c, -sdcd2 * es2);
    E.k12 = fma(fh, fma(2.0 * sd2, es2, w * (R.s * S.s)), -mu * (2.0 - b));
    E.k13 = (fh * rsn) * (S.e * fma(2.0 * csig, Dl.s, -w * R.s));
    E.k14 = -2.0 * fh * ssig * Dl.s * S.e;
    E.k22 = (fh * rr) * fma(sdcd2, es2, w * (R.c * S.s));
    E.k24 = -(fh * rr) * fma(2.0 * csig * Dl.s, S.e, w * S.s * R.e);
    return E;
}

// P wave hyperbolic, S wave trigonometric (beta_e < c < alpha_e): the direct formulas with
// the P-wave terms scaled by e^-th_r (overflow-free for th_r up to 700).
template <class TabT>
__device__ __forceinline__ Elem elem_stable_ht(double kh, double c2, double ia2, double ib2,
                                               double krho, double mu, TabT tab)
{
    double r, rr;
    sqrt_rsqrt(fma(-c2, ia2, 1.0), r, rr);
    const double qb = fma(-c2, ib2, 1.0);
    const ExpScaled R = exp_scaled(kh * r, tab);
    const double Cr = R.c, XSr = r * R.s, SXr = R.s * rr, er = R.e;
    double Cs, XSs, SXs;
    wave_trig(qb, kh, Cs, XSs, SXs);
    const double Dh = fma(SXr, SXs, fma(XSr, XSs, 2.0 * fma(-Cr, Cs, er)));
    const double fh = (krho * c2) * rcp_fast(Dh);
    Elem E;
    E.k11 = fh * fma(Cr, SXs, -XSr * Cs);
    E.k12 = fma(fh, fma(-XSr, XSs, fma(Cr, Cs, -er)), -mu * (1.0 + qb));
    E.k13 = fh * fma(-er, SXs, XSr);
    E.k14 = fh * fma(er, Cs, -Cr);
    E.k22 = fh * fma(SXr, Cs, -Cr * XSs);
    E.k24 = fh * fma(er, XSs, -SXr);
    return E;
}

template <class TabT>
__device__ __forceinline__ Elem layer_elem_stable(const LayerConst &L, double c2, TabT tab)
{
    const double qa = fma(-c2, L.ia2, 1.0), qb = fma(-c2, L.ib2, 1.0);
    if (qa > 0.0 && qb > 0.0) return elem_stable_hh(L.kh, c2, L.ia2, L.ib2, L.krho, lc_mu(L), tab);
    if (qa > 0.0) return elem_stable_ht(L.kh, c2, L.ia2, L.ib2, L.krho, lc_mu(L), tab);
    double t[6];   // both trigonometric: bounded functions, the direct formulas
    waves_general(qa, qb, L.kh, t, tab);
    return elem_from_triples(t[0], t[1], t[2], t[3], t[4], t[5], L.krho, lc_mu(L), c2);
}

// The stable element without its factor (ElemU, as layer_elem_u for the direct one): the
// scaled brackets and the scaled D^ are one consistent pair (f^ D^ = k rho c^2), so U = the
// brackets with k12's correction as kappa D^ -- the f-free recursion runs on them unchanged,
// and every entry stays O(1) for k h up to 700 (no overflow in D_t d_t either).
template <class TabT>
__device__ __forceinline__ ElemU elemu_stable_hh(double kh, double c2, double ia2, double ib2,
                                                 double kap, double rratio, TabT tab)
{
    const double a = c2 * ia2, b = c2 * ib2;
    double r, rr, s, rsn;
    sqrt_rsqrt(1.0 - a, r, rr);
    sqrt_rsqrt(1.0 - b, s, rsn);
    const double rs = r * s;
    const double w = fma(-a, b, a + b) * rcp_fast(1.0 + rs);          // 1 - rs
    const double dl = 0.5 * kh * ((b - a) * rcp_fast(r + s));          // (th_r - th_s)/2
    const ExpScaled R = exp_scaled(kh * r, tab), S = exp_scaled(kh * s, tab);
    const ExpScaled Dl = exp_scaled(dl, tab);
    const double es2 = S.e * S.e;
    const double sd2 = Dl.s * Dl.s;
    const double sdcd2 = 2.0 * Dl.s * Dl.c;
    const double csig = fma(S.c, Dl.c, S.s * Dl.s);
    const double ssig = fma(S.s, Dl.c, S.c * Dl.s);
    ElemU U;
    U.D = fma((w * w) * (rr * rsn), R.s * S.s, -4.0 * sd2 * es2);
    U.g11 = rsn * fma(w * R.s, S.c, -sdcd2 * es2);
    U.g12 = fma(kap, U.D, fma(2.0 * sd2, es2, w * (R.s * S.s)));
    U.g13 = rsn * (S.e * fma(2.0 * csig, Dl.s, -w * R.s));
    U.g14 = -2.0 * ssig * Dl.s * S.e;
    U.g22 = rr * fma(sdcd2, es2, w * (R.c * S.s));
    U.g24 = -rr * fma(2.0 * csig * Dl.s, S.e, w * S.s * R.e);
    U.rr = rratio;
    return U;
}

template <class TabT>
__device__ __forceinline__ ElemU elemu_stable_ht(double kh, double c2, double ia2, double ib2,
                                                 double kap, double rratio, TabT tab)
{
    double r, rr;
    sqrt_rsqrt(fma(-c2, ia2, 1.0), r, rr);
    const double qb = fma(-c2, ib2, 1.0);
    const ExpScaled R = exp_scaled(kh * r, tab);
    const double Cr = R.c, XSr = r * R.s, SXr = R.s * rr, er = R.e;
    double Cs, XSs, SXs;
    wave_trig(qb, kh, Cs, XSs, SXs);
    ElemU U;
    U.D = fma(SXr, SXs, fma(XSr, XSs, 2.0 * fma(-Cr, Cs, er)));
    U.g11 = fma(Cr, SXs, -XSr * Cs);
    U.g12 = fma(kap, U.D, fma(-XSr, XSs, fma(Cr, Cs, -er)));
    U.g13 = fma(-er, SXs, XSr);
    U.g14 = fma(er, Cs, -Cr);
    U.g22 = fma(SXr, Cs, -Cr * XSs);
    U.g24 = fma(er, XSs, -SXr);
    U.rr = rratio;
    return U;
}

// layer_elem_stable without the factor; L.kh = k h (row scan) -- the model-major and pair
// scans pass a copy with k h formed from their k-free h (the same product).
template <class TabT>
__device__ __forceinline__ ElemU layer_elemu_stable(const LayerConst &L, double c2, double ic2,
                                                    TabT tab)
{
    const double qa = fma(-c2, L.ia2, 1.0), qb = fma(-c2, L.ib2, 1.0);
    const double kap = lc_kappa(L, ic2);
    if (qa > 0.0 && qb > 0.0) return elemu_stable_hh(L.kh, c2, L.ia2, L.ib2, kap, L.aux, tab);
    if (qa > 0.0) return elemu_stable_ht(L.kh, c2, L.ia2, L.ib2, kap, L.aux, tab);
    double t[6];   // both trigonometric: bounded functions, the direct formulas
    waves_general(qa, qb, L.kh, t, tab);
    return elemu_from_triples(t[0], t[1], t[2], t[3], t[4], t[5], kap, L.aux);
}

// -------------------------------------------------------------- wavelength-free terms
// The square roots r_e = sqrt(1 - c^2/alpha_e^2), s_e = sqrt(1 - c^2/beta_e^2) and the
// half-space's k-free factors depend on the model and c but NOT on the wavelength, so the
// model-major scan (scan_models_kernel) computes them once per (model, c) for all of a
// model's wavelengths.  Everything downstream is evaluated with the same operations in the
// same order as in the row scan, so both give bitwise-identical determinants.  A root is
// stored as (x, 1/|x|) with x = +sqrt(q) for a hyperbolic wave (q > 0) and x = -sqrt(-q)
// for a trigonometric one.
__device__ __forceinline__ double2 wave_root(double q)
{
    double x, rx;
    sqrt_rsqrt(fabs(q), x, rx);
    return make_double2(q > 0.0 ? x : -x, rx);
}

template <class TabT>
__device__ __forceinline__ void wave_hyp_root(double x, double rx, double kh, double &C,
                                              double &XS, double &SX,
                                              TabT tab)
{
    double ch, sh;
    cosh_sinh(kh * x, ch, sh, tab);
    C = ch;
    XS = x * sh;
    SX = sh * rx;
}

__device__ __forceinline__ void wave_trig_root(double xneg, double rx, double kh, double &C,
                                               double &XS, double &SX)
{
    const double xi = -xneg;
    const double th = kh * xi;
    double sn, cs;
    if (trig_fast(th)) {
        sin_cos(th, sn, cs);
    } else {
        sin_cos_large(th, sn, cs);
    }
    C = cs;
    XS = -xi * sn;
    SX = sn * rx;
}

// Element of K / k for layer M at wavenumber k from the cached roots a (P wave) and b (S wave).
// M holds the model's k-free constants: M.kh = h, M.krho = rho, M.b2 = 2 beta^2; only
// k h = k * M.kh depends on the wavelength (formed exactly as the row scan's LayerConst
// fill forms it, so both scans compute bitwise-identical elements).
template <class TabT>
__device__ __forceinline__ Elem layer_elem_root(const LayerConst &M, double k, double2 a,
                                                double2 b, double c2,
                                                TabT tab)
{
    const double kh = k * M.kh;
    double Cr, XSr, SXr, Cs, XSs, SXs;
    if (is_pos(a.x)) {
        if (is_pos(b.x)) {
            wave_hyp_root(a.x, a.y, kh, Cr, XSr, SXr, tab);
            wave_hyp_root(b.x, b.y, kh, Cs, XSs, SXs, tab);
        } else {
            wave_hyp_root(a.x, a.y, kh, Cr, XSr, SXr, tab);
            wave_trig_root(b.x, b.y, kh, Cs, XSs, SXs);
        }
    } else {
        double t[6];
        waves_general(fma(-c2, M.ia2, 1.0), fma(-c2, M.ib2, 1.0), kh, t, tab);
        Cr = t[0]; XSr = t[1]; SXr = t[2];
        Cs = t[3]; XSs = t[4]; SXs = t[5];
    }
    return elem_from_triples(Cr, XSr, SXr, Cs, XSs, SXs, M.krho, lc_mu(M), c2);
}

// Elements of layer M for two wavenumbers ka, kb (two wavelengths of one model) at the same
// velocity: one branch on the wave types, both rows' waves interleaved inside it.  Each
// row's arithmetic is exactly layer_elem_root's (bitwise-identical elements).
template <class TabT>
__device__ __forceinline__ void layer_elem_root2(const LayerConst &M, double ka, double kb,
                                                 double2 a, double2 b, double c2, TabT tab,
                                                 Elem &Ea, Elem &Eb)
{
    const double kha = ka * M.kh, khb = kb * M.kh;
    double Cra, XSra, SXra, Csa, XSsa, SXsa;
    double Crb, XSrb, SXrb, Csb, XSsb, SXsb;
    if (is_pos(a.x)) {
        if (is_pos(b.x)) {
            wave_hyp_root(a.x, a.y, kha, Cra, XSra, SXra, tab);
            wave_hyp_root(a.x, a.y, khb, Crb, XSrb, SXrb, tab);
            wave_hyp_root(b.x, b.y, kha, Csa, XSsa, SXsa, tab);
            wave_hyp_root(b.x, b.y, khb, Csb, XSsb, SXsb, tab);
        } else {
            wave_hyp_root(a.x, a.y, kha, Cra, XSra, SXra, tab);
            wave_hyp_root(a.x, a.y, khb, Crb, XSrb, SXrb, tab);
            wave_trig_root(b.x, b.y, kha, Csa, XSsa, SXsa);
            wave_trig_root(b.x, b.y, khb, Csb, XSsb, SXsb);
        }
    } else {
        double t[6];
        const double qa = fma(-c2, M.ia2, 1.0), qb = fma(-c2, M.ib2, 1.0);
        waves_general(qa, qb, kha, t, tab);
        Cra = t[0]; XSra = t[1]; SXra = t[2];
        Csa = t[3]; XSsa = t[4]; SXsa = t[5];
        waves_general(qa, qb, khb, t, tab);
        Crb = t[0]; XSrb = t[1]; SXrb = t[2];
        Csb = t[3]; XSsb = t[4]; SXsb = t[5];
    }
    Ea = elem_from_triples(Cra, XSra, SXra, Csa, XSsa, SXsa, M.krho, lc_mu(M), c2);
    Eb = elem_from_triples(Crb, XSrb, SXrb, Csb, XSsb, SXsb, M.krho, lc_mu(M), c2);
}

// layer_elem_root / layer_elem_root2 without the factor f (ElemU), for the sign scans.
template <class TabT>
__device__ __forceinline__ ElemU layer_elem_root_u(const LayerConst &M, double k, double2 a,
                                                   double2 b, double c2, double ic2,
                                                   TabT tab)
{
    const double kh = k * M.kh;
    double Cr, XSr, SXr, Cs, XSs, SXs;
    if (is_pos(a.x)) {
        if (is_pos(b.x)) {
            wave_hyp_root(a.x, a.y, kh, Cr, XSr, SXr, tab);
            wave_hyp_root(b.x, b.y, kh, Cs, XSs, SXs, tab);
        } else {
            wave_hyp_root(a.x, a.y, kh, Cr, XSr, SXr, tab);
            wave_trig_root(b.x, b.y, kh, Cs, XSs, SXs);
        }
    } else {
        double t[6];
        waves_general(fma(-c2, M.ia2, 1.0), fma(-c2, M.ib2, 1.0), kh, t, tab);
        Cr = t[0]; XSr = t[1]; SXr = t[2];
        Cs = t[3]; XSs = t[4]; SXs = t[5];
    }
    return elemu_from_triples(Cr, XSr, SXr, Cs, XSs, SXs, lc_kappa(M, ic2), M.aux);
}

template <class TabT>
__device__ __forceinline__ void layer_elem_root2_u(const LayerConst &M, double ka, double kb,
                                                   double2 a, double2 b, double c2, double ic2,
                                                   TabT tab, ElemU &Ea, ElemU &Eb)
{
    const double kha = ka * M.kh, khb = kb * M.kh;
    double Cra, XSra, SXra, Csa, XSsa, SXsa;
    double Crb, XSrb, SXrb, Csb, XSsb, SXsb;
    if (is_pos(a.x)) {
        if (is_pos(b.x)) {
            wave_hyp_root(a.x, a.y, kha, Cra, XSra, SXra, tab);
            wave_hyp_root(a.x, a.y, khb, Crb, XSrb, SXrb, tab);
            wave_hyp_root(b.x, b.y, kha, Csa, XSsa, SXsa, tab);
            wave_hyp_root(b.x, b.y, khb, Csb, XSsb, SXsb, tab);
        } else {
            wave_hyp_root(a.x, a.y, kha, Cra, XSra, SXra, tab);
            wave_hyp_root(a.x, a.y, khb, Crb, XSrb, SXrb, tab);
            wave_trig_root(b.x, b.y, kha, Csa, XSsa, SXsa);
            wave_trig_root(b.x, b.y, khb, Csb, XSsb, SXsb);
        }
    } else {
        double t[6];
        const double qa = fma(-c2, M.ia2, 1.0), qb = fma(-c2, M.ib2, 1.0);
        waves_general(qa, qb, kha, t, tab);
        Cra = t[0]; XSra = t[1]; SXra = t[2];
        Csa = t[3]; XSsa = t[4]; SXsa = t[5];
        waves_general(qa, qb, khb, t, tab);
        Crb = t[0]; XSrb = t[1]; SXrb = t[2];
        Csb = t[3]; XSsb = t[4]; SXsb = t[5];
    }
    const double kap = lc_kappa(M, ic2);
    Ea = elemu_from_triples(Cra, XSra, SXra, Csa, XSsa, SXsa, kap, M.aux);
    Eb = elemu_from_triples(Crb, XSrb, SXrb, Csb, XSsb, SXsb, kap, M.aux);
}

// Half-space element K_hs = mu [[r w/(1-rs), w/(1-rs) - 2], [., s w/(1-rs)]], w = 1 - s^2 =
// c^2/beta_N^2 (real), mu = k rho_N beta_N^2; cases by the branch of r, s (reading S3).
// Split into the k-free factors (HsRoot: the roots, gw = w/(1 - r s) or its analogue, and
// the case) and the mu-dependent entries.
struct HalfSpace {
    double h11r, h11i, h12r, h12i, h22r, h22i;
    bool real;   // all imaginary parts zero (c < beta_N)
};
struct HsRoot {
    double r, s, gw, t;
    int kase;   // 0: c < beta_N (r, s real); 1: beta_N < c < alpha_N (s = i xs); 2: c > alpha_N
};

__device__ __forceinline__ HsRoot halfspace_root(double ia2, double ib2, double c2)
{
    HsRoot R;
    const double qa = fma(-c2, ia2, 1.0), qb = fma(-c2, ib2, 1.0);
    const double w = c2 * ib2;
    if (qb > 0.0) {
        R.r = qa * rsqrt_fast(qa);
        R.s = qb * rsqrt_fast(qb);
        // 1 - rs = (a + b - ab)/(1 + rs), a = c^2/alpha^2, b = c^2/beta^2 = w: no cancellation
        // as c -> 0 (the direct 1 - rs loses ~log10(1/(1-rs)) digits there)
        const double a = c2 * ia2;
        R.gw = (w * (1.0 + R.r * R.s)) * rcp_fast(fma(-a, w, a + w));
        R.t = 0.0;
        R.kase = 0;
    } else if (qa > 0.0) {
        R.r = qa * rsqrt_fast(qa);
        R.s = -qb * rsqrt_fast(-qb);          // xs
        R.t = R.r * R.s;                       // 1/(1 - i t) = (1 + i t)/(1 + t^2)
        R.gw = w * rcp_fast(fma(R.t, R.t, 1.0));
        R.kase = 1;
    } else {
        R.r = -qa * rsqrt_fast(-qa);          // xr
        R.s = -qb * rsqrt_fast(-qb);          // xs
        R.gw = w * rcp_fast(fma(R.r, R.s, 1.0));
        R.t = 0.0;
        R.kase = 2;
    }
    return R;
}

__device__ __forceinline__ HalfSpace halfspace_k(const HsRoot &R, double mu)
{
    HalfSpace H;
    H.real = R.kase == 0;
    if (R.kase == 0) {
        const double g = mu * R.gw;
        H.h11r = R.r * g; H.h11i = 0.0;
        H.h12r = g - 2.0 * mu; H.h12i = 0.0;
        H.h22r = R.s * g; H.h22i = 0.0;
    } else if (R.kase == 1) {
        const double gre = mu * R.gw, gim = gre * R.t;
        H.h11r = R.r * gre; H.h11i = R.r * gim;
        H.h12r = gre - 2.0 * mu; H.h12i = gim;
        H.h22r = -R.s * gim; H.h22i = R.s * gre;
    } else {
        const double g = mu * R.gw;
        H.h11r = 0.0; H.h11i = R.r * g;
        H.h12r = g - 2.0 * mu; H.h12i = 0.0;
        H.h22r = 0.0; H.h22i = R.s * g;
    }
    return H;
}

// -------------------------------------------------------------- determinant
// Mantissa/exponent accumulator for the debug det grid (exact sign, no overflow).
struct DetAcc {
    double m;
    int e;
    __device__ __forceinline__ void mul(double x)
    {
        m *= x;
        int ex;
        m = frexp(m, &ex);
        e += ex;
    }
};

struct DetOut {
    int sign;      // sgn(Re det K) in {-1, 0, +1}
    bool bad;      // a pivot or Re det was NaN/Inf (reading S9)
    double mre, mim;
    int e2;        // det = (mre + i mim) * 2^e2 (only when WANT_VALUE)
};

// -------------------------------------------------------------- banded GEPP step
// One step of banded Gaussian elimination with partial pivoting over the 4 rows that can
// hold nonzeros in the current node's two columns (reading S10/S11): rows R[0], R[1] are the
// two rows left by the previous step (matrix positions 2t, 2t+1), R[2], R[3] the two rows
// of the next node (positions 2t+2, 2t+3); columns are [node t | node t+1 | node t+2].
// Every other row of K is zero in these columns, so choosing the largest |entry| among the
// four and swapping it to the top is the pivot sequence of dense GEPP on K -- the oracle's
// algorithm -- up to near-ties (magnitudes compared to 2^-20, see mag_key).
//
// The pivot rows are resolved by BRANCHING on (p, q) into statically indexed code instead
// of selecting rows through the index: along a warp's 32 consecutive velocities the pivot
// pattern is uniform in ~90% of (chunk, step) pairs (measured on C5), so the branches are
// mostly convergent and no per-element select instructions are issued.  NR = number of
// trailing complex columns (2 in the last step, whose node-N columns carry K_hs).
struct StepOut {
    double piv0, piv1;
    int key0, key1;   // mag_key of the two pivots (0 <=> zero pivot, >= 0x7ff00000 <=> Inf/NaN)
    int parity;       // parity of the two GEPP row swaps
};

// |x| ordering key: the high word without the sign bit (exponent + top 20 mantissa bits).
// Comparing keys picks a pivot within 2^-20 of the largest magnitude -- as stable as exact
// partial pivoting -- with one integer op per candidate instead of an FP64-pipe DSETP.
__device__ __forceinline__ int mag_key(double x) { return __double2hiint(x) & 0x7fffffff; }

// Entries known to be ZERO at compile time, so their updates are skipped (fma(-l, 0, x) is
// x for finite l; a non-finite l already poisons the row's other columns, so the Inf/NaN
// bookkeeping is unchanged).  Before the step, rows 0, 1 (left over from node t-1) are zero
// in node t+2's columns (c >= 4 when NC = 6) and have no imaginary part; rows 2, 3 are
// imaginary only in the trailing NR columns.  After column 0 is eliminated with pivot row P,
// row i keeps a zero iff it and row P both had one.  With P in {0, 1} (3/4 of the steps on
// C5) this removes 6-10 of the step's 23 DFMAs.
template <int NC, int NR>
__device__ __forceinline__ constexpr bool zre0(int i, int c) { return NC == 6 && i < 2 && c >= 4; }
template <int NC, int NR>
__device__ __forceinline__ constexpr bool zim0(int i, int c) { return i < 2 || c < NC - NR; }

template <int NC, int NR, int P, int Q>
__device__ __forceinline__ void gepp_finish(double (&R)[4][NC], double (&Ri)[4][NC],
                                            StepOut &o, double (&X)[2][NC - 2],
                                            double (&Xi)[2][NC - 2])
{
    // positions after swap(0, P): pos[1..3]; after swap(1, Q): leftover = positions 2, 3
    constexpr int pos1 = (P == 1) ? 0 : 1;
    constexpr int pos2 = (P == 2) ? 0 : 2;
    constexpr int pos3 = (P == 3) ? 0 : 3;
    constexpr int prow = (Q == 1) ? pos1 : (Q == 2 ? pos2 : pos3);   // column-1 pivot row
    constexpr int lo = (Q == 2) ? pos1 : pos2;
    constexpr int hi = (Q == 3) ? pos1 : pos3;
    o.piv1 = R[prow][1];
    const double inv1 = rcp_fast(o.piv1);
    const double l_lo = R[lo][1] * inv1, l_hi = R[hi][1] * inv1;
    // zero pattern after the column-0 elimination (rows != P)
    constexpr auto zr = [](int i, int c) { return zre0<NC, NR>(i, c) && zre0<NC, NR>(P, c); };
    constexpr auto zi = [](int i, int c) { return zim0<NC, NR>(i, c) && zim0<NC, NR>(P, c); };
#pragma unroll
    for (int c = 2; c < NC; ++c) {
        if (zr(prow, c)) {
            X[0][c - 2] = zr(lo, c) ? 0.0 : R[lo][c];
            X[1][c - 2] = zr(hi, c) ? 0.0 : R[hi][c];
        } else {
            X[0][c - 2] = fma(-l_lo, R[prow][c], R[lo][c]);
            X[1][c - 2] = fma(-l_hi, R[prow][c], R[hi][c]);
        }
        if (zi(prow, c)) {
            Xi[0][c - 2] = zi(lo, c) ? 0.0 : Ri[lo][c];
            Xi[1][c - 2] = zi(hi, c) ? 0.0 : Ri[hi][c];
        } else {
            Xi[0][c - 2] = zi(lo, c) ? -l_lo * Ri[prow][c] : fma(-l_lo, Ri[prow][c], Ri[lo][c]);
            Xi[1][c - 2] = zi(hi, c) ? -l_hi * Ri[prow][c] : fma(-l_hi, Ri[prow][c], Ri[hi][c]);
        }
    }
    o.parity = (P != 0) ^ (Q != 1);
}

template <int NC, int NR, int P>
__device__ __forceinline__ void gepp_after_p(double (&R)[4][NC], double (&Ri)[4][NC],
                                             StepOut &o, double (&X)[2][NC - 2],
                                             double (&Xi)[2][NC - 2])
{
    o.piv0 = R[P][0];
    const double inv0 = rcp_fast(o.piv0);
    // eliminate column 0 from the three other rows with pivot row P (skipping the pivot
    // row's known zeros)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i == P) continue;
        const double l = R[i][0] * inv0;
#pragma unroll
        for (int c = 1; c < NC; ++c) {
            if (!zre0<NC, NR>(P, c))
                R[i][c] = zre0<NC, NR>(i, c) ? -l * R[P][c] : fma(-l, R[P][c], R[i][c]);
            if (!zim0<NC, NR>(P, c))
                Ri[i][c] = zim0<NC, NR>(i, c) ? -l * Ri[P][c] : fma(-l, Ri[P][c], Ri[i][c]);
        }
    }
    // column-1 pivot among positions 1..3 (rows pos1, pos2, pos3), first max wins
    constexpr int pos1 = (P == 1) ? 0 : 1;
    constexpr int pos2 = (P == 2) ? 0 : 2;
    constexpr int pos3 = (P == 3) ? 0 : 3;
    const int b1 = mag_key(R[pos1][1]), b2 = mag_key(R[pos2][1]), b3 = mag_key(R[pos3][1]);
    const int b23 = max(b2, b3);
    o.key1 = max(b1, b23);
    // first maximum in position order; the common no-swap case (position 1) is tested first
    if (b1 >= b23) {
        gepp_finish<NC, NR, P, 1>(R, Ri, o, X, Xi);
    } else if (b2 >= b3) {
        gepp_finish<NC, NR, P, 2>(R, Ri, o, X, Xi);
    } else {
        gepp_finish<NC, NR, P, 3>(R, Ri, o, X, Xi);
    }
}

template <int NC, int NR>
__device__ __forceinline__ StepOut gepp_step(double (&R)[4][NC], double (&Ri)[4][NC],
                                             double (&X)[2][NC - 2], double (&Xi)[2][NC - 2])
{
    StepOut o;
    const int a0 = mag_key(R[0][0]), a1 = mag_key(R[1][0]), a2 = mag_key(R[2][0]),
              a3 = mag_key(R[3][0]);
    int p = 0;
    int best = a0;
    if (a1 > best) { best = a1; p = 1; }
    if (a2 > best) { best = a2; p = 2; }
    if (a3 > best) { best = a3; p = 3; }
    o.key0 = best;
    // most frequent first (C5, oracle's dense GEPP: p = 0 63 %, 3 24 %, 1 12 %, 2 1 %)
    if (p == 0) {
        gepp_after_p<NC, NR, 0>(R, Ri, o, X, Xi);
    } else if (p == 3) {
        gepp_after_p<NC, NR, 3>(R, Ri, o, X, Xi);
    } else if (p == 1) {
        gepp_after_p<NC, NR, 1>(R, Ri, o, X, Xi);
    } else {
        gepp_after_p<NC, NR, 2>(R, Ri, o, X, Xi);
    }
    return o;
}

// Determinant core (sign, optionally value) of K for N layers.  elem(e) returns the element
// of layer e (0 <= e < N), hs() the half-space element.
//
// Elimination (reading S10/S11): banded GEPP streamed node by node.  The nodes' rows hold
//   node 0:     [ top_0 | B_0 ]
//   node t:     [ B_{t-1}^T | bottom_{t-1} + top_t | B_t ]
//   node N:     [ B_{N-1}^T | bottom_{N-1} + K_hs ]
// with top = [[k11, k12], [k12, k22]], bottom = [[k11, -k12], [-k12, k22]],
// B = [[k13, k14], [-k14, k24]].  Step t eliminates node t's two columns from the two rows
// left over by step t-1 and the two rows of node t+1.  Every column of nodes < N is real
// (reading S3/S5), so the pivots and all but the last node's columns are real fp64; only
// node N's columns (K_hs) are complex.  det K = (-1)^parity * prod pivots * det(last 2x2).
// Cost per node: one layer element + one 4-row GEPP step, O(N) in total.
// NFIX > 0 compiles the determinant for exactly NFIX layers (fully unrolled); NFIX = 0 takes
// N at run time, its node loop unrolled UNROLL times (measured on B200: 2 is 1.7 % faster
// for the model-major kernel at N = 6, 1 is 4 % faster for the row kernel at N = 10).
// State of one streamed banded-GEPP determinant: the previous layer's element P, the two
// rows X left over by the last step, and the sign / zero / non-finite bookkeeping.
//
// Sign, zero and non-finite bookkeeping in integer ops on the pivots' high words (off the FP64
// pipe): sgn accumulates the XOR of the pivots' sign bits; a zero pivot has key 0, an Inf/NaN
// pivot a key >= 0x7ff00000 (NaN keys exceed every finite key, so a NaN entry is always picked
// as a pivot or reaches the last 2x2 through the updates).
template <bool WANT_VALUE>
struct DetState {
    Elem P;
    double X[2][4];
    int perm;
    unsigned sgn, kmin, kmax;
    DetAcc acc;

    __device__ __forceinline__ void init(const Elem &E)
    {
        P = E;
        X[0][0] = E.k11; X[0][1] = E.k12; X[0][2] = E.k13; X[0][3] = E.k14;
        X[1][0] = E.k12; X[1][1] = E.k22; X[1][2] = -E.k14; X[1][3] = E.k24;
        perm = 0;
        sgn = 0u;
        kmin = 0x7fffffffu;
        kmax = 0u;
        acc = DetAcc{1.0, 0};
    }

    __device__ __forceinline__ void book(const StepOut &so)
    {
        sgn ^= (unsigned)(__double2hiint(so.piv0) ^ __double2hiint(so.piv1));
        kmin = min(kmin, min((unsigned)so.key0, (unsigned)so.key1));
        kmax = max(kmax, max((unsigned)so.key0, (unsigned)so.key1));
        perm ^= so.parity;
        if (WANT_VALUE) {
            acc.mul(so.piv0);
            acc.mul(so.piv1);
        }
    }

    // one node step with the next layer's element Q
    __device__ __forceinline__ void step(const Elem &Q)
    {
        double R[4][6] = {
            {X[0][0], X[0][1], X[0][2], X[0][3], 0.0, 0.0},
            {X[1][0], X[1][1], X[1][2], X[1][3], 0.0, 0.0},
            {P.k13, -P.k14, P.k11 + Q.k11, Q.k12 - P.k12, Q.k13, Q.k14},
            {P.k14, P.k24, Q.k12 - P.k12, P.k22 + Q.k22, -Q.k14, Q.k24}};
        double Ri[4][6];   // unused (real step): NR = 0
        double Xi[2][4];
        book(gepp_step<6, 0>(R, Ri, X, Xi));
        P = Q;
    }

    // last step with the half-space element: node N-1 columns real, node N columns complex
    // (NR = 2) -- or real when c < beta_N (K_hs real, the common case)
    __device__ __forceinline__ DetOut finish(const HalfSpace &H)
    {
        double dre, dim;
        if (H.real) {
            double R[4][4] = {{X[0][0], X[0][1], X[0][2], X[0][3]},
                              {X[1][0], X[1][1], X[1][2], X[1][3]},
                              {P.k13, -P.k14, P.k11 + H.h11r, H.h12r - P.k12},
                              {P.k14, P.k24, H.h12r - P.k12, P.k22 + H.h22r}};
            double Ri[4][4];   // unused: NR = 0
            double Y[2][2], Yi[2][2];
            book(gepp_step<4, 0>(R, Ri, Y, Yi));
            dre = fma(Y[0][0], Y[1][1], -Y[0][1] * Y[1][0]);
            dim = 0.0;
        } else {
            double R[4][4] = {{X[0][0], X[0][1], X[0][2], X[0][3]},
                              {X[1][0], X[1][1], X[1][2], X[1][3]},
                              {P.k13, -P.k14, P.k11 + H.h11r, H.h12r - P.k12},
                              {P.k14, P.k24, H.h12r - P.k12, P.k22 + H.h22r}};
            double Ri[4][4] = {{0.0, 0.0, 0.0, 0.0},
                               {0.0, 0.0, 0.0, 0.0},
                               {0.0, 0.0, H.h11i, H.h12i},
                               {0.0, 0.0, H.h12i, H.h22i}};
            double Y[2][2], Yi[2][2];
            book(gepp_step<4, 2>(R, Ri, Y, Yi));
            // det of the last complex 2x2
            dre = fma(Y[0][0], Y[1][1], -Yi[0][0] * Yi[1][1]) -
                  fma(Y[0][1], Y[1][0], -Yi[0][1] * Yi[1][0]);
            dim = fma(Y[0][0], Yi[1][1], Yi[0][0] * Y[1][1]) -
                  fma(Y[0][1], Yi[1][0], Yi[0][1] * Y[1][0]);
        }
        kmax = max(kmax, max((unsigned)mag_key(dre), (unsigned)mag_key(dim)));
        // A zero pivot (key 0: the pivot column is zero, det K = 0 exactly) makes every later
        // pivot NaN through the unguarded reciprocal; it takes precedence, as in the oracle's
        // elimination, which stops there with det = 0.  Inputs are finite and the range
        // guard S9 keeps every entry finite, so no Inf/NaN can precede a zero pivot.
        const bool zero = (kmin == 0u) || (dre == 0.0);
        const bool bad = (kmax >= 0x7ff00000u) && (kmin != 0u);
        const bool neg = (perm != 0) ^ ((sgn >> 31) != 0) ^ (dre < 0.0);

        DetOut out;
        out.bad = bad;
        out.sign = zero ? 0 : (neg ? -1 : 1);
        out.mre = 0.0;
        out.mim = 0.0;
        out.e2 = 0;
        if (WANT_VALUE && kmin != 0u) {
            // value = (-1)^permutation * (prod pivots) * (dre + i dim)
            const double ps = perm ? -acc.m : acc.m;
            double re = ps * dre, im = ps * dim;
            const double t = fmax(fabs(re), fabs(im));
            if (t == 0.0 || !isfinite(t)) {
                out.mre = re;
                out.mim = im;
                out.e2 = (t == 0.0) ? 0 : acc.e;
            } else {
                int ex;
                frexp(t, &ex);
                out.mre = ldexp(re, -ex);
                out.mim = ldexp(im, -ex);
                out.e2 = acc.e + ex;
            }
        }
        return out;
    }
};

// Determinant core (sign, optionally value) of K for N layers.  elem(e) returns the element
// of layer e (0 <= e < N), hs() the half-space element.
//
// Elimination (reading S10/S11): banded GEPP streamed node by node.  The nodes' rows hold
//   node 0:     [ top_0 | B_0 ]
//   node t:     [ B_{t-1}^T | bottom_{t-1} + top_t | B_t ]
//   node N:     [ B_{N-1}^T | bottom_{N-1} + K_hs ]
// with top = [[k11, k12], [k12, k22]], bottom = [[k11, -k12], [-k12, k22]],
// B = [[k13, k14], [-k14, k24]].  Step t eliminates node t's two columns from the two rows
// left over by step t-1 and the two rows of node t+1.  Every column of nodes < N is real
// (reading S3/S5), so the pivots and all but the last node's columns are real fp64; only
// node N's columns (K_hs) are complex.  det K = (-1)^parity * prod pivots * det(last 2x2).
// Cost per node: one layer element + one 4-row GEPP step, O(N) in total.
// NFIX > 0 compiles the determinant for exactly NFIX layers (fully unrolled); NFIX = 0 takes
// N at run time, its node loop unrolled UNROLL times (measured on B200: 2 is 1.7 % faster
// for the model-major kernel at N = 6, 1 is 4 % faster for the row kernel at N = 10).
template <bool WANT_VALUE, int NFIX, int UNROLL, class ElemFn, class HsFn>
__device__ __forceinline__ DetOut det_core(int Nrt, ElemFn &&elem, HsFn &&hs)
{
    const int N = NFIX > 0 ? NFIX : Nrt;
    DetState<WANT_VALUE> st;
    st.init(elem(0));
    if constexpr (NFIX > 0) {
#pragma unroll
        for (int t = 0; t + 1 < NFIX; ++t) st.step(elem(t + 1));
    } else {
        constexpr int kLayerUnroll = UNROLL;
#pragma unroll kLayerUnroll
        for (int t = 0; t + 1 < N; ++t) st.step(elem(t + 1));
    }
    return st.finish(hs());
}

// -------------------------------------------------------------- sign by block recursion
// The scan needs only sgn(Re det K).  K is symmetric 2x2-block tridiagonal, so the block
// LDL^T recursion  S_0 = A_0,  S_{t+1} = A_{t+1} - B_t^T S_t^{-1} B_t,  det K = prod det S_t
// gives the sign with no pivot search, no branches and no row bookkeeping (~25 FP64 ops
// per node, like one banded-GEPP step, but ~45 fewer integer / move / branch instructions).
// Unpivoted elimination is backward stable when its multipliers W_t = S_t^{-1} B_t stay
// bounded (threshold pivoting: then |L||U| <= (1 + |W|) |K| block-wise; the bound and the
// measured agreement with GEPP are in DESIGN.md §5); every step checks max|W_t| <=
// 2^kBlockMultExp (exponent arithmetic on the high words) and that every det S_t is nonzero
// and finite (BlockSignU: every scaling p_t normal with a normal reciprocal).  A determinant that fails
// the check (a leading block S_t nearly singular: rare, measured in DESIGN.md) is re-evaluated
// by the caller with the banded GEPP (det_core), so the result always follows partial
// pivoting where the unpivoted recursion is not certified.  (Reading S11: the values of
// det K -- masw_det_grid, parity -- always come from the GEPP.)
#ifndef MASW_BLOCK_MULT_EXP
#define MASW_BLOCK_MULT_EXP 12
#endif
constexpr int kBlockMultExp = MASW_BLOCK_MULT_EXP;   // multipliers up to 4096 (variant builds: -D)

struct SignOut {
    int sign;   // sgn(Re det K)
    bool bad;   // non-finite (only from the GEPP re-evaluation)
    bool ok;    // certified (else re-evaluate with GEPP)
};

// exponent field of |x| (0 for zero/denormal, 0x7ff for Inf/NaN)
__device__ __forceinline__ int exp_of(double x) { return (__double2hiint(x) >> 20) & 0x7ff; }

// (mag_key, above: (exponent << 20) | top 20 mantissa bits of |x|, one LOP3 where exp_of
// needs two.)
// BlockSignU's certificate in key units (integer pipe, ~7 instructions per node fewer than
// exponent fields): key(max|W'|) - key(d) <= kBlockMultExp << 20, i.e. the exponent
// difference is at most kBlockMultExp and at most kBlockMultExp - 1 unless the top mantissa
// bits of W' do not exceed d's (|W| < 2^13, typically <= 2^12: never looser than BlockSign's
// exponent test); and every p normal with a normal reciprocal, DBL_MIN <= |p| < 2^1022:
// key(p) - key(DBL_MIN) < key(2^1022) - key(DBL_MIN) as unsigned.  (The reciprocal of p is
// taken with rcp.approx.ftz, which flushes a subnormal result to zero: for 2^1022 <= |p| <
// 2^1024 the recursion would silently drop the coupling to the layer above -- measured on
// thick layers, k h ~ 140, where p = D d ~ e^(3 (th_r + th_s)) approaches the fp64 range;
// such a determinant now goes to the GEPP re-evaluation like an overflowing one.)
constexpr int kKeyMultMax = kBlockMultExp << 20;
#ifndef MASW_KEY_PMAX
#define MASW_KEY_PMAX 0x7fd00000u   // key(2^1022) (variant builds: 0x7ff00000u, the old bound)
#endif
constexpr unsigned kKeyNormMin = 0x00100000u, kKeyRange = MASW_KEY_PMAX - 0x00100000u;

// State of one block-recursion sign evaluation (see det_sign_block).
struct BlockSign {
    Elem P;                 // the previous layer's element
    double s11, s12, s22;   // current leading block S_t (symmetric)
    unsigned sgn;           // XOR of the det S_t sign bits
    int worst;              // max over steps of exponent(max|W'|) - exponent(det S)
    int dmin, dmax;         // min / max exponent of det S (0: zero/denormal, 0x7ff: Inf/NaN)

    __device__ __forceinline__ void init(const Elem &E)
    {
        P = E;
        s11 = E.k11;   // S_0 = top block of layer 0
        s12 = E.k12;
        s22 = E.k22;
        sgn = 0u;
        worst = -4096;
        dmin = 0x7ff;
        dmax = 0;
    }

    // eliminate the current node with block S and coupling B = [[b11, b12], [-b12, b22]]
    // (layer P's k13, k14, k24): M' = B^T adj(S) B and 1/det S (M = M' / det S is applied by
    // the callers inside their subtraction, one fused operation per entry)
    __device__ __forceinline__ void eliminate(double &m11, double &m12, double &m22, double &id)
    {
        const double b11 = P.k13, b12 = P.k14, b22 = P.k24;
        const double d = fma(s11, s22, -(s12 * s12));
        // W' = adj(S) B, adj(S) = [[s22, -s12], [-s12, s11]], b21 = -b12
        const double w11 = fma(s22, b11, s12 * b12);
        const double w12 = fma(s22, b12, -s12 * b22);
        const double w21 = fma(-s12, b11, -s11 * b12);
        const double w22 = fma(-s12, b12, s11 * b22);
        id = rcp_fast(d);
        // M' = B^T W' (symmetric)
        m11 = fma(b11, w11, -b12 * w21);
        m12 = fma(b11, w12, -b12 * w22);
        m22 = fma(b12, w12, b22 * w22);
        sgn ^= (unsigned)__double2hiint(d);
        const int ed = exp_of(d);
        const int ew = max(max(exp_of(w11), exp_of(w12)), max(exp_of(w21), exp_of(w22)));
        worst = max(worst, ew - ed);
        dmin = min(dmin, ed);
        dmax = max(dmax, ed);
    }

    // one node, in two halves so that the previous element P is dead before the next one is
    // computed (no loop-carried copies of P, fewer live registers during the element):
    //   pre():   T = bottom(P) - B^T S_t^{-1} B      (needs S_t and P only)
    //   post(Q): S_{t+1} = T + top(Q),  P = Q
    double t11, t12, t22;
    __device__ __forceinline__ void pre()
    {
        double m11, m12, m22, id;
        eliminate(m11, m12, m22, id);
        t11 = fma(-m11, id, P.k11);
        t12 = fma(-m12, id, -P.k12);
        t22 = fma(-m22, id, P.k22);
    }
    __device__ __forceinline__ void post(const Elem &Q)
    {
        s11 = t11 + Q.k11;
        s12 = t12 + Q.k12;
        s22 = t22 + Q.k22;
        P = Q;
    }

    // last node: S_N = bottom(P) + K_hs - M (complex when c > beta_N); sign of Re det K
    __device__ __forceinline__ SignOut finish(const HalfSpace &H)
    {
        double m11, m12, m22, id;
        eliminate(m11, m12, m22, id);
        const double r11 = fma(-m11, id, P.k11 + H.h11r), r12 = fma(-m12, id, H.h12r - P.k12),
                     r22 = fma(-m22, id, P.k22 + H.h22r);
        double dre;
        if (H.real) {
            dre = fma(r11, r22, -(r12 * r12));
        } else {
            // Re[(r11 + i h11i)(r22 + i h22i) - (r12 + i h12i)^2]
            dre = fma(r11, r22, -H.h11i * H.h22i) - fma(r12, r12, -H.h12i * H.h12i);
        }
        SignOut o;
        o.ok = (worst <= kBlockMultExp) && (dmin > 0) && (dmax < 0x7ff) && (exp_of(dre) < 0x7ff);
        o.bad = false;
        const int hi = __double2hiint(dre);
        const bool neg = ((sgn >> 31) != 0) ^ (hi < 0);
        const bool zero = ((hi & 0x7fffffff) | __double2loint(dre)) == 0;
        o.sign = zero ? 0 : (neg ? -1 : 1);
        return o;
    }
};

// The same recursion on the f-free elements (ElemU, E_e = f_e U_e): with S_t = f_t S^_t
// (node t's leading block over its lower layer's factor; det S_t = f_t^2 det S^_t has the
// sign of det S^_t, and the multipliers S_t^-1 B_t = S^_t^-1 G_t are unchanged),
//   S^_0 = top(U_0),
//   S^_(t+1) = (f_t / f_(t+1)) X_t / d_t + top(U_(t+1)),  X_t = d_t bot(U_t) - G_t^T adj(S^_t) G_t,
//   d_t = det S^_t,   f_t / f_(t+1) = rr_t D_(t+1) / D_t,
// i.e. one reciprocal of p_t = D_t d_t per node and none per element; the last node
// S_N = f_(N-1) X / d + K_hs is scaled by the real d / f_(N-1):  Z = X + p K_hs / (rho_(N-1) c^2)
// (same sign of Re det).  The half-space is passed pre-scaled (halfspace_k with
// mu' = rho_N beta_N^2 / (rho_(N-1) c^2)).  p_t is also certified (normal, with a normal
// reciprocal: D_t = 0 is a pole of the element, which the GEPP re-evaluation reports as
// non-finite).
struct BlockSignU {
    ElemU P;                // the previous layer's element
    double s11, s12, s22;   // S^_t
    unsigned sgn;
    int worst;              // max over nodes of key(max|W'|) - key(d)
    unsigned prange;        // max over nodes of key(p) - kKeyNormMin (unsigned)
    double x11, x12, x22, rg;

    __device__ __forceinline__ void init(const ElemU &E)
    {
        P = E;
        s11 = E.g11;
        s12 = E.g12;
        s22 = E.g22;
        sgn = 0u;
        worst = -(1 << 30);
        prange = 0u;
    }

    // X = d bot(P) - G^T adj(S^) G, p = D_P d
    __device__ __forceinline__ double eliminate()
    {
        const double b11 = P.g13, b12 = P.g14, b22 = P.g24;
        const double d = fma(s11, s22, -(s12 * s12));
        const double w11 = fma(s22, b11, s12 * b12);
        const double w12 = fma(s22, b12, -s12 * b22);
        const double w21 = fma(-s12, b11, -s11 * b12);
        const double w22 = fma(-s12, b12, s11 * b22);
        const double m11 = fma(b11, w11, -b12 * w21);
        const double m12 = fma(b11, w12, -b12 * w22);
        const double m22 = fma(b12, w12, b22 * w22);
        x11 = fma(P.g11, d, -m11);
        x12 = fma(-P.g12, d, -m12);
        x22 = fma(P.g22, d, -m22);
        const double p = P.D * d;
        sgn ^= (unsigned)__double2hiint(d);
        const int kw = max(max(mag_key(w11), mag_key(w12)), max(mag_key(w21), mag_key(w22)));
        worst = max(worst, kw - mag_key(d));
        prange = max(prange, (unsigned)mag_key(p) - kKeyNormMin);
        return p;
    }
    // rr / p with rr folded into the reciprocal's correction: y0 (1 + e + e^2) rr as
    // fma(rr y0, e + e^2, rr y0) -- rr y0 forms beside e, one dependent step fewer (as
    // accurate as rcp_fast; C5 -0.25 %)
    __device__ __forceinline__ void pre()
    {
        const double p = eliminate();
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
        const double e = fma(-p, y, 1.0);
        const double ry = P.rr * y;
        rg = fma(ry, fma(e, e, e), ry);
    }
    __device__ __forceinline__ void post(const ElemU &Q)
    {
        const double g = rg * Q.D;
        s11 = fma(g, x11, Q.g11);
        s12 = fma(g, x12, Q.g12);
        s22 = fma(g, x22, Q.g22);
        P = Q;
    }

    // H: K_hs scaled by 1 / (rho_(N-1) c^2)
    __device__ __forceinline__ SignOut finish(const HalfSpace &H)
    {
        const double p = eliminate();
        const double z11 = fma(p, H.h11r, x11), z12 = fma(p, H.h12r, x12),
                     z22 = fma(p, H.h22r, x22);
        double dre;
        if (H.real) {
            dre = fma(z11, z22, -(z12 * z12));
        } else {
            const double i11 = p * H.h11i, i12 = p * H.h12i, i22 = p * H.h22i;
            dre = fma(z11, z22, -i11 * i22) - fma(z12, z12, -i12 * i12);
        }
        SignOut o;
        o.ok = (worst <= kKeyMultMax) && (prange < kKeyRange) && (exp_of(dre) < 0x7ff);
        o.bad = false;
        const int hi = __double2hiint(dre);
        const bool neg = ((sgn >> 31) != 0) ^ (hi < 0);
        const bool zero = ((hi & 0x7fffffff) | __double2loint(dre)) == 0;
        o.sign = zero ? 0 : (neg ? -1 : 1);
        return o;
    }
};

template <int UNROLL, class ElemFn, class HsFn>
__device__ __forceinline__ SignOut det_sign_block_u(int N, ElemFn &&elem, HsFn &&hs)
{
    BlockSignU st;
    st.init(elem(0));
    constexpr int kU = UNROLL;
#pragma unroll kU
    for (int t = 0; t + 1 < N; ++t) {
        st.pre();
        st.post(elem(t + 1));
    }
    return st.finish(hs());
}

template <int UNROLL, class Elem2Fn, class Hs2Fn>
__device__ __forceinline__ void det_sign_block_u_pair(int N, Elem2Fn &&elem2, Hs2Fn &&hs2,
                                                      SignOut &oa, SignOut &ob)
{
    BlockSignU A, B;
    {
        ElemU ea, eb;
        elem2(0, ea, eb);
        A.init(ea);
        B.init(eb);
    }
    constexpr int kU = UNROLL;
#pragma unroll kU
    for (int t = 0; t + 1 < N; ++t) {
        A.pre();
        B.pre();
        ElemU qa, qb;
        elem2(t + 1, qa, qb);
        A.post(qa);
        B.post(qb);
    }
    HalfSpace ha, hb;
    hs2(ha, hb);
    oa = A.finish(ha);
    ob = B.finish(hb);
}

template <int UNROLL, class ElemFn, class HsFn>
__device__ __forceinline__ SignOut det_sign_block(int N, ElemFn &&elem, HsFn &&hs)
{
    BlockSign st;
    st.init(elem(0));
    constexpr int kU = UNROLL;
#pragma unroll kU
    for (int t = 0; t + 1 < N; ++t) {
        st.pre();
        st.post(elem(t + 1));
    }
    return st.finish(hs());
}

// Two signs whose element evaluations share every branch (two wavelengths of one model at
// the same velocity): with the branch-free block recursion the two evaluations interleave
// completely (twice the instruction-level parallelism).
template <int UNROLL, class Elem2Fn, class Hs2Fn>
__device__ __forceinline__ void det_sign_block_pair(int N, Elem2Fn &&elem2, Hs2Fn &&hs2,
                                                    SignOut &oa, SignOut &ob)
{
    BlockSign A, B;
    {
        Elem ea, eb;
        elem2(0, ea, eb);
        A.init(ea);
        B.init(eb);
    }
    constexpr int kU = UNROLL;
#pragma unroll kU
    for (int t = 0; t + 1 < N; ++t) {
        A.pre();
        B.pre();
        Elem qa, qb;
        elem2(t + 1, qa, qb);
        A.post(qa);
        B.post(qb);
    }
    HalfSpace ha, hb;
    hs2(ha, hb);
    oa = A.finish(ha);
    ob = B.finish(hb);
}

// det K(k, c) for one row whose LayerConst[0..N] (k-scaled) and velocity list are in `lc`,
// `vel` (shared memory).  `maybe_near` = false means c is already the S4-perturbed velocity
// (the scan resolves S4 per warp for its 32 velocities, see scan_kernel), which skips the
// per-lane S4 loop.
template <bool WANT_VALUE, int NFIX = 0, bool STABLE = false, class TabT = unsigned>
__device__ __forceinline__ DetOut det_K(const LayerConst *__restrict__ lc,
                                        const double *__restrict__ vel,
                                        TabT tab, int Nrt, double c,
                                        bool maybe_near = true)
{
    const int N = NFIX > 0 ? NFIX : Nrt;
    const double cp = maybe_near ? perturb_velocity(vel, 2 * (N + 1), c) : c;
    const double c2 = cp * cp;
    return det_core<WANT_VALUE, NFIX, MASW_LAYER_UNROLL>(
        N,
        [&](int e) {
            if constexpr (STABLE) return layer_elem_stable(load_lc(lc + e), c2, tab);
            else return layer_elem(load_lc(lc + e), c2, tab);
        },
        [&] {
            const LayerConst H = load_lc(lc + N);
            return halfspace_k(halfspace_root(H.ia2, H.ib2, c2), lc_mu(H));
        });
}


}  // namespace masw
