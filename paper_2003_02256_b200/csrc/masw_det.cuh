// masw_det.cuh -- per-(lambda, c) stiffness determinant, assembled and eliminated in
// registers (sm_100a).  Product code; shares nothing with oracle/.
//
// What it computes (readings S1-S16 in DESIGN.md):
//   K(k, c) of order 2(N+1) is the sum of N Kausel-Roesset 4x4 layer elements overlapping
//   in 2x2 blocks plus the 2x2 half-space element, i.e. a symmetric 2x2 BLOCK-TRIDIAGONAL
//   matrix (the paper's "heptadiagonal" band, reading S10):
//       A_i = bottom(layer i-1) + top(layer i) (+ K_hs at i = N),  B_i = coupling of layer i.
//   det K = prod_i det S_i with S_0 = A_0, S_i = A_i - B_{i-1}^T S_{i-1}^{-1} B_{i-1}
//   (block Gaussian elimination without pivoting, reading S11; O(N)).
//
// Arithmetic design (B200):
//   * Every layer entry is an even function of r and s, hence exactly REAL for real (k, c)
//     (reading S3/S5): each wave contributes the real triple (C, x*S, S/x) =
//        (cosh th, x sinh th, sinh th / x),  x = sqrt(1 - c^2/v^2),   th = k h x   (x real)
//        (cos th, -xi sin th, sin th / xi),  xi = sqrt(c^2/v^2 - 1),  th = k h xi  (x = i xi)
//     so the N interior blocks are eliminated in fp64 REAL arithmetic; only the last node
//     (with the half-space) is complex, and only when c > beta_N.
//   * Nothing is stored: K never exists in memory (the paper kept 3136 B per matrix in
//     global memory).  Per layer the kernel keeps 3 doubles of carried Schur
//     complement; parameters come from shared memory (broadcast).
//   * The sign of Re det K is the product of the signs of the N real block determinants and
//     of Re det S_N, so the scan never multiplies determinants and cannot overflow (S14).
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
    bool bad;      // some block determinant or Re det was NaN/Inf (reading S9)
    double mre, mim;
    int e2;        // det = (mre + i mim) * 2^e2 (only when WANT_VALUE)
};

// Determinant of K(k, c) for one row whose LayerConst[0..N] and velocity list are in `lc`,
// `vel` (shared memory).  c is the unperturbed grid value.
template <bool WANT_VALUE>
__device__ __forceinline__ DetOut det_K(const LayerConst *__restrict__ lc,
                                        const double *__restrict__ vel, int N, double c)
{
    const double cp = perturb_velocity(vel, 2 * (N + 1), c);
    const double c2 = cp * cp;

    double P11 = 0.0, P12 = 0.0, P22 = 0.0;   // carried bottom(e-1) - B^T S^{-1} B
    int neg = 0;
    bool zero = false, bad = false;
    DetAcc acc{1.0, 0};

#pragma unroll 1
    for (int e = 0; e < N; ++e) {
        const double kh = lc[e].kh, ia2 = lc[e].ia2, ib2 = lc[e].ib2;
        const double krho = lc[e].krho, mu = lc[e].mu;
        const double qa = fma(-c2, ia2, 1.0);   // r^2
        const double qb = fma(-c2, ib2, 1.0);   // s^2
        double Cr, XSr, SXr, Cs, XSs, SXs;
        wave_triple(qa, kh, Cr, XSr, SXr);
        wave_triple(qb, kh, Cs, XSs, SXs);
        const double CC = Cr * Cs;
        // D = 2(1 - Cr Cs) + (1/(rs)) Sr Ss + rs Sr Ss
        const double D = fma(SXr, SXs, fma(XSr, XSs, 2.0 * (1.0 - CC)));
        const double f = (krho * c2) / D;
        const double k11 = f * fma(Cr, SXs, -XSr * Cs);
        const double k12 = fma(f, fma(-XSr, XSs, CC - 1.0), -mu * (1.0 + qb));
        const double k13 = f * (XSr - SXs);
        const double k14 = f * (Cs - Cr);
        const double k22 = f * fma(SXr, Cs, -Cr * XSs);
        const double k24 = f * (XSs - SXr);
        // S_e = P + top(layer e)
        const double S11 = P11 + k11, S12 = P12 + k12, S22 = P22 + k22;
        const double dS = fma(S11, S22, -S12 * S12);
        neg ^= (dS < 0.0);
        zero |= (dS == 0.0);
        bad |= !isfinite(dS);
        if (WANT_VALUE) acc.mul(dS);
        const double inv = 1.0 / dS;
        // B = [[k13, k14], [-k14, k24]]: columns b1 = (k13, -k14), b2 = (k14, k24).
        // y = adj(S) b, adj(S) = [[S22, -S12], [-S12, S11]]
        const double y1x = fma(S22, k13, S12 * k14), y1y = -fma(S12, k13, S11 * k14);
        const double y2x = fma(S22, k14, -S12 * k24), y2y = fma(S11, k24, -S12 * k14);
        const double q11 = fma(k13, y1x, -k14 * y1y);
        const double q12 = fma(k13, y2x, -k14 * y2y);
        const double q22 = fma(k14, y2x, k24 * y2y);
        // bottom(layer e) = [[k11, -k12], [-k12, k22]]
        P11 = fma(-inv, q11, k11);
        P12 = fma(-inv, q12, -k12);
        P22 = fma(-inv, q22, k22);
    }

    // Half-space node: S_N = P + K_hs, K_hs = mu [[r w/(1-rs), w/(1-rs) - 2], [., s w/(1-rs)]]
    // with w = 1 - s^2 = c^2/beta_N^2 (real).  Cases by the branch of r, s (reading S3).
    const double ia2 = lc[N].ia2, ib2 = lc[N].ib2, mu = lc[N].mu;
    const double qa = fma(-c2, ia2, 1.0), qb = fma(-c2, ib2, 1.0);
    const double w = c2 * ib2;
    double dre, dim;
    if (qb > 0.0) {                     // c < beta_N < alpha_N: r, s real
        const double r = sqrt(qa), s = sqrt(qb);
        const double g = mu * (w / (1.0 - r * s));
        const double S11 = P11 + r * g, S12 = P12 + (g - 2.0 * mu), S22 = P22 + s * g;
        dre = fma(S11, S22, -S12 * S12);
        dim = 0.0;
    } else if (qa > 0.0) {              // beta_N < c < alpha_N: r real, s = i*xs
        const double r = sqrt(qa), xs = sqrt(-qb);
        // 1/(1 - i r xs) = (1 + i r xs) / (1 + r^2 xs^2)
        const double t = r * xs;
        const double den = fma(t, t, 1.0);
        const double gre = mu * (w / den), gim = gre * t;       // g = mu w /(1 - rs)
        const double a11r = P11 + r * gre, a11i = r * gim;       // r g
        const double a12r = P12 + (gre - 2.0 * mu), a12i = gim;  // g - 2 mu
        const double a22r = P22 - xs * gim, a22i = xs * gre;     // i xs g
        dre = fma(a11r, a22r, -a11i * a22i) - fma(a12r, a12r, -a12i * a12i);
        dim = fma(a11r, a22i, a11i * a22r) - 2.0 * a12r * a12i;
    } else {                            // c > alpha_N: r = i*xr, s = i*xs, 1 - rs = 1 + xr xs
        const double xr = sqrt(-qa), xs = sqrt(-qb);
        const double g = mu * (w / fma(xr, xs, 1.0));
        const double a11r = P11, a11i = xr * g;
        const double a12 = P12 + (g - 2.0 * mu);
        const double a22r = P22, a22i = xs * g;
        dre = fma(a11r, a22r, -a11i * a22i) - a12 * a12;
        dim = fma(a11r, a22i, a11i * a22r);
    }
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
        // (acc.m * 2^acc.e) * (dre + i dim), normalised by max(|re|, |im|) in [0.5, 1)
        double re = acc.m * dre, im = acc.m * dim;
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
