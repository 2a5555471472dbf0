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

namespace masw {

constexpr double kTwoPi = 6.283185307179586;   // reading S2 / O1
constexpr double kMaxKH = 350.0;               // reading S9 range guard
constexpr double kPerturbTol = 1e-4;           // reading S4
constexpr double kPerturbFactor = 1.0 - 1e-4;  // reading S4

// Per-row constants of one finite layer e (index N holds the half-space's ia2, ib2, mu).
struct LayerConst {
    double kh;    // k * h_e
    double ia2;   // 1 / alpha_e^2
    double ib2;   // 1 / beta_e^2
    double krho;  // k * rho_e
    double mu;    // k * rho_e * beta_e^2
};
static_assert(sizeof(LayerConst) == 40, "LayerConst layout");

// -------------------------------------------------------------- wave triple
// cosh/sinh of th >= 0.  Small arguments use the Taylor series (no cancellation in
// sinh ~ th, reading "Transcendental accuracy"); large ones exp and 1/exp.
__device__ __forceinline__ void cosh_sinh(double th, double &ch, double &sh)
{
    if (th < 0.5) {
        const double t2 = th * th;
        // sinh(t)/t = sum t^{2n}/(2n+1)!, n <= 7: truncation < 5e-17 for t < 0.5
        double ps = 1.0 / 1307674368000.0;                 // 1/15!
        ps = fma(ps, t2, 1.0 / 6227020800.0);              // 1/13!
        ps = fma(ps, t2, 1.0 / 39916800.0);                // 1/11!
        ps = fma(ps, t2, 1.0 / 362880.0);                  // 1/9!
        ps = fma(ps, t2, 1.0 / 5040.0);                    // 1/7!
        ps = fma(ps, t2, 1.0 / 120.0);                     // 1/5!
        ps = fma(ps, t2, 1.0 / 6.0);                       // 1/3!
        ps = fma(ps, t2, 1.0);
        // cosh(t) = sum t^{2n}/(2n)!, n <= 8: truncation < 1e-18
        double pc = 1.0 / 20922789888000.0;                // 1/16!
        pc = fma(pc, t2, 1.0 / 87178291200.0);             // 1/14!
        pc = fma(pc, t2, 1.0 / 479001600.0);               // 1/12!
        pc = fma(pc, t2, 1.0 / 3628800.0);                 // 1/10!
        pc = fma(pc, t2, 1.0 / 40320.0);                   // 1/8!
        pc = fma(pc, t2, 1.0 / 720.0);                     // 1/6!
        pc = fma(pc, t2, 1.0 / 24.0);                      // 1/4!
        pc = fma(pc, t2, 0.5);                             // 1/2!
        pc = fma(pc, t2, 1.0);
        sh = th * ps;
        ch = pc;
    } else {
        const double e = exp(th);
        const double ie = 1.0 / e;
        ch = 0.5 * (e + ie);
        sh = 0.5 * (e - ie);
    }
}

// (C, XS, SX) for q = 1 - c^2/v^2 != 0 and kh = k*h.  See header comment.
__device__ __forceinline__ void wave_triple(double q, double kh, double &C, double &XS,
                                            double &SX)
{
    if (q > 0.0) {
        const double rq = rsqrt(q);   // 1/x
        const double x = q * rq;      // x
        double ch, sh;
        cosh_sinh(kh * x, ch, sh);
        C = ch;
        XS = x * sh;
        SX = sh * rq;
    } else {
        const double nq = -q;
        const double rq = rsqrt(nq);  // 1/xi
        const double xi = nq * rq;    // xi
        double sn, cs;
        sincos(kh * xi, &sn, &cs);
        C = cs;
        XS = -xi * sn;
        SX = sn * rq;
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

// -------------------------------------------------------------- layer element
// Six unique real entries of the Kausel-Roesset layer element (reading S1) from the wave
// triples: with (C, XS, SX) of the P (r) and S (s) waves,
//   D   = 2(1 - Cr Cs) + SXr SXs + XSr XSs,  f = k rho c^2 / D
//   k11 = f (Cr SXs - XSr Cs)    k12 = f (Cr Cs - XSr XSs - 1) - mu (1 + s^2)
//   k13 = f (XSr - SXs)          k14 = f (Cs - Cr)
//   k22 = f (SXr Cs - Cr XSs)    k24 = f (XSs - SXr)
// Element layout (DOFs u_top, w_top, u_bot, w_bot):
//   [[k11, k12, k13, k14], [k12, k22, -k14, k24], [k13, -k14, k11, -k12], [k14, k24, -k12, k22]]
struct Elem {
    double k11, k12, k13, k14, k22, k24;
};

__device__ __forceinline__ Elem layer_elem(const LayerConst &L, double c2)
{
    const double qa = fma(-c2, L.ia2, 1.0);   // r^2
    const double qb = fma(-c2, L.ib2, 1.0);   // s^2
    double Cr, XSr, SXr, Cs, XSs, SXs;
    wave_triple(qa, L.kh, Cr, XSr, SXr);
    wave_triple(qb, L.kh, Cs, XSs, SXs);
    const double CC = Cr * Cs;
    const double D = fma(SXr, SXs, fma(XSr, XSs, 2.0 * (1.0 - CC)));
    const double f = (L.krho * c2) / D;
    Elem E;
    E.k11 = f * fma(Cr, SXs, -XSr * Cs);
    E.k12 = fma(f, fma(-XSr, XSs, CC - 1.0), -L.mu * (1.0 + qb));
    E.k13 = f * (XSr - SXs);
    E.k14 = f * (Cs - Cr);
    E.k22 = f * fma(SXr, Cs, -Cr * XSs);
    E.k24 = f * (XSs - SXr);
    return E;
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

template <int NC>
__device__ __forceinline__ double sel4(int p, const double (&R)[4][NC], int c)
{
    return p == 0 ? R[0][c] : (p == 1 ? R[1][c] : (p == 2 ? R[2][c] : R[3][c]));
}

// One step of banded Gaussian elimination with partial pivoting over the 4 rows that can
// hold nonzeros in the current node's two columns (reading S10/S11: 2 leftover rows of the
// previous node + the 2 rows of the next node).  Columns: [node t | node t+1 | node t+2].
// The pivot for each column is the row of largest magnitude (first in row order on ties),
// exactly as dense GEPP picks it (the oracle), because every other row of K is
// zero in these columns.  Rows are not moved: the pivot row is read through a select and
// every other live row is updated with multiplier l_i (l = 0 for used rows).  The two rows
// left over are returned in row order as the next step's first two rows.
// parity = parity of the permutation (p, q, rest...) of the four rows.
template <int NC, int NR>
__device__ __forceinline__ void gepp_step(double (&R)[4][NC], double (&Ri)[4][NC], double &piv0,
                                          double &piv1, int &parity, double (&X)[2][NC - 2],
                                          double (&Xi)[2][NC - 2])
{
    // ---- column 0
    int p = 0;
    double best = fabs(R[0][0]);
#pragma unroll
    for (int i = 1; i < 4; ++i) {
        const double a = fabs(R[i][0]);
        if (a > best) {
            best = a;
            p = i;
        }
    }
    piv0 = sel4<NC>(p, R, 0);
    const double inv0 = (piv0 != 0.0) ? 1.0 / piv0 : 0.0;
    double PR[NC], PRi[NC];
#pragma unroll
    for (int c = 1; c < NC; ++c) {
        PR[c] = sel4<NC>(p, R, c);
        if (c >= NC - NR) PRi[c] = sel4<NC>(p, Ri, c);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double l = (i == p) ? 0.0 : R[i][0] * inv0;
#pragma unroll
        for (int c = 1; c < NC; ++c) {
            R[i][c] = fma(-l, PR[c], R[i][c]);
            if (c >= NC - NR) Ri[i][c] = fma(-l, PRi[c], Ri[i][c]);
        }
    }
    // ---- column 1 (rows other than p)
    int q = -1;
    best = -1.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double a = (i == p) ? -1.0 : fabs(R[i][1]);
        if (a > best) {
            best = a;
            q = i;
        }
    }
    piv1 = sel4<NC>(q, R, 1);
    const double inv1 = (piv1 != 0.0) ? 1.0 / piv1 : 0.0;
#pragma unroll
    for (int c = 2; c < NC; ++c) {
        PR[c] = sel4<NC>(q, R, c);
        if (c >= NC - NR) PRi[c] = sel4<NC>(q, Ri, c);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double l = (i == p || i == q) ? 0.0 : R[i][1] * inv1;
#pragma unroll
        for (int c = 2; c < NC; ++c) {
            R[i][c] = fma(-l, PR[c], R[i][c]);
            if (c >= NC - NR) Ri[i][c] = fma(-l, PRi[c], Ri[i][c]);
        }
    }
    // ---- the two leftover rows, in row order
    const int lo = (p != 0 && q != 0) ? 0 : ((p != 1 && q != 1) ? 1 : 2);
    const int hi = (p != 3 && q != 3) ? 3 : ((p != 2 && q != 2) ? 2 : 1);
#pragma unroll
    for (int c = 2; c < NC; ++c) {
        X[0][c - 2] = sel4<NC>(lo, R, c);
        X[1][c - 2] = sel4<NC>(hi, R, c);
        if (c >= NC - NR) {
            Xi[0][c - 2] = sel4<NC>(lo, Ri, c);
            Xi[1][c - 2] = sel4<NC>(hi, Ri, c);
        } else {
            Xi[0][c - 2] = 0.0;
            Xi[1][c - 2] = 0.0;
        }
    }
    parity = (p + q - (p < q ? 1 : 0)) & 1;
}

// Determinant of K(k, c) for one row whose LayerConst[0..N] and velocity list are in `lc`,
// `vel` (shared memory).  c is the unperturbed grid value.
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
template <bool WANT_VALUE>
__device__ __forceinline__ DetOut det_K(const LayerConst *__restrict__ lc,
                                        const double *__restrict__ vel, int N, double c)
{
    const double cp = perturb_velocity(vel, 2 * (N + 1), c);
    const double c2 = cp * cp;

    int neg = 0, perm = 0;
    bool zero = false, bad = false;
    DetAcc acc{1.0, 0};

    Elem P = layer_elem(lc[0], c2);
    double X[2][4] = {{P.k11, P.k12, P.k13, P.k14}, {P.k12, P.k22, -P.k14, P.k24}};

#pragma unroll 1
    for (int t = 0; t + 1 < N; ++t) {
        const Elem Q = layer_elem(lc[t + 1], c2);
        double R[4][6] = {
            {X[0][0], X[0][1], X[0][2], X[0][3], 0.0, 0.0},
            {X[1][0], X[1][1], X[1][2], X[1][3], 0.0, 0.0},
            {P.k13, -P.k14, P.k11 + Q.k11, Q.k12 - P.k12, Q.k13, Q.k14},
            {P.k14, P.k24, Q.k12 - P.k12, P.k22 + Q.k22, -Q.k14, Q.k24}};
        double Ri[4][6];   // unused (real step): NR = 0
        double Xi[2][4];
        double piv0, piv1;
        int par;
        gepp_step<6, 0>(R, Ri, piv0, piv1, par, X, Xi);
        neg ^= par ^ (piv0 < 0.0) ^ (piv1 < 0.0);
        perm ^= par;
        zero |= (piv0 == 0.0) | (piv1 == 0.0);
        bad |= !isfinite(piv0) | !isfinite(piv1);
        if (WANT_VALUE) {
            acc.mul(piv0);
            acc.mul(piv1);
        }
        P = Q;
    }

    // Half-space K_hs = mu [[r w/(1-rs), w/(1-rs) - 2], [., s w/(1-rs)]], w = 1 - s^2 =
    // c^2/beta_N^2 (real); cases by the branch of r, s (reading S3).
    double h11r, h11i, h12r, h12i, h22r, h22i;
    {
        const double ia2 = lc[N].ia2, ib2 = lc[N].ib2, mu = lc[N].mu;
        const double qa = fma(-c2, ia2, 1.0), qb = fma(-c2, ib2, 1.0);
        const double w = c2 * ib2;
        if (qb > 0.0) {                     // c < beta_N < alpha_N: r, s real
            const double r = sqrt(qa), s = sqrt(qb);
            const double g = mu * (w / (1.0 - r * s));
            h11r = r * g; h11i = 0.0;
            h12r = g - 2.0 * mu; h12i = 0.0;
            h22r = s * g; h22i = 0.0;
        } else if (qa > 0.0) {              // beta_N < c < alpha_N: r real, s = i xs
            const double r = sqrt(qa), xs = sqrt(-qb);
            const double t = r * xs;        // 1/(1 - i t) = (1 + i t)/(1 + t^2)
            const double gre = mu * (w / fma(t, t, 1.0)), gim = gre * t;
            h11r = r * gre; h11i = r * gim;
            h12r = gre - 2.0 * mu; h12i = gim;
            h22r = -xs * gim; h22i = xs * gre;
        } else {                            // c > alpha_N: r = i xr, s = i xs
            const double xr = sqrt(-qa), xs = sqrt(-qb);
            const double g = mu * (w / fma(xr, xs, 1.0));
            h11r = 0.0; h11i = xr * g;
            h12r = g - 2.0 * mu; h12i = 0.0;
            h22r = 0.0; h22i = xs * g;
        }
    }

    // Last step: node N-1 columns real, node N columns complex (NR = 2).
    double R[4][4] = {{X[0][0], X[0][1], X[0][2], X[0][3]},
                      {X[1][0], X[1][1], X[1][2], X[1][3]},
                      {P.k13, -P.k14, P.k11 + h11r, h12r - P.k12},
                      {P.k14, P.k24, h12r - P.k12, P.k22 + h22r}};
    double Ri[4][4] = {{0.0, 0.0, 0.0, 0.0},
                       {0.0, 0.0, 0.0, 0.0},
                       {0.0, 0.0, h11i, h12i},
                       {0.0, 0.0, h12i, h22i}};
    double Y[2][2], Yi[2][2];
    double piv0, piv1;
    int par;
    gepp_step<4, 2>(R, Ri, piv0, piv1, par, Y, Yi);
    neg ^= par ^ (piv0 < 0.0) ^ (piv1 < 0.0);
    perm ^= par;
    zero |= (piv0 == 0.0) | (piv1 == 0.0);
    bad |= !isfinite(piv0) | !isfinite(piv1);
    if (WANT_VALUE) {
        acc.mul(piv0);
        acc.mul(piv1);
    }
    // det of the last complex 2x2
    const double dre = fma(Y[0][0], Y[1][1], -Yi[0][0] * Yi[1][1]) -
                       fma(Y[0][1], Y[1][0], -Yi[0][1] * Yi[1][0]);
    const double dim = fma(Y[0][0], Yi[1][1], Yi[0][0] * Y[1][1]) -
                       fma(Y[0][1], Yi[1][0], Yi[0][1] * Y[1][0]);
    bad |= !isfinite(dre) || !isfinite(dim);
    zero |= (dre == 0.0);
    neg ^= (dre < 0.0);

    DetOut out;
    out.bad = bad;
    out.sign = zero ? 0 : (neg ? -1 : 1);
    out.mre = 0.0;
    out.mim = 0.0;
    out.e2 = 0;
    if (WANT_VALUE) {
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

}  // namespace masw
