/*
 * oracle/masw_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU fp64 reference for the MASW theoretical
 * dispersion curve of Kump & Martin, "MASWAccelerated" (arXiv:2003.02256), written
 * from the paper and the readings listed in DESIGN.md ("Readings").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load this library.  It shares no code, header, table or constant generator
 * with the CUDA product (paper_2003_02256_b200/csrc); neither side includes the other.
 *
 * What it computes, step by step:
 *   O0 validate            oracle_validate()
 *   O1 wavenumber          k = 2*pi/lambda                          (reading S2)
 *   O2 velocity perturb    c' = c*(1-1e-4) while near a layer velocity (reading S4)
 *   O3 layer element       Kausel-Roesset 4x4 element, complex arithmetic
 *   O4 half-space element  2x2 element ("size 2(N+1)", S1, S22)
 *   O5 determinant         DENSE complex LU with partial pivoting, det kept as
 *                          (complex mantissa, binary exponent)
 *   O6 sign                sgn(Re det)
 *   O7 scan                Algorithm 1, lazily in ascending c, first change -> V[n]
 *                                                                         (PAPER.md:50-71, S6-S9)
 *   O8 misfit              Algorithm 2, index-order sum / l
 *   O9 ensemble            O7+O8 per model, argmin ties -> lowest id
 *   O10 det grid           every (lambda, c) det, no early exit
 *
 * Deliberately unlike the product: the product never forms K and eliminates 2x2 blocks
 * in real arithmetic; this file scatters every element into a dense complex n x n matrix
 * (n = 2(N+1)) and factors it with pivoting, O(n^3) per determinant, the way
 * MASWaves does ("banded structure ... not utilized").
 *
 * Parity status per function: every function here is pinned by tests/test_oracle_pins.py
 * (pins P1-P13, P15 of SURVEY.md §8(c)); see DESIGN.md "Oracle pins".
 *
 * Threads: rows (one (model, lambda) pair each) are independent ("no
 * dependence on other wavelength values"), so oracle_curve/oracle_ensemble run rows on
 * pthreads; each row's arithmetic is exactly the serial Algorithm 1.
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <quadmath.h>

typedef double complex cplx;

/* Status codes (same numeric meaning as documented in DESIGN.md; defined independently). */
#define OR_OK 0
#define OR_WARN_NO_SIGN_CHANGE 1
#define OR_E_ARG (-1)
#define OR_E_MODEL (-2)
#define OR_E_GRID (-3)
#define OR_E_RANGE (-4)
#define OR_E_NONFINITE (-5)

#define OR_IDX_NO_CHANGE (-1)
#define OR_IDX_NONFINITE (-2)

/* O1: 2*pi as the fp64 literal of reading S2/O1. */
static const double OR_TWO_PI = 6.283185307179586;
/* O0: overflow guard, reading S9: k*h must not exceed this. */
static const double OR_MAX_KH = 350.0;
/* O2: reading S4 (MASWaves rule). */
static const double OR_PERTURB_TOL = 1e-4;
static const double OR_PERTURB_FACTOR = 1e-4;

/* ------------------------------------------------------------------ O0 validation */

static int finite_all(const double *x, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* Validate one model (SPEC.md:36 invariants: h>0, rho>0, beta>0, alpha>beta). */
int oracle_validate_model(int32_t N, const double *h, const double *alpha,
                          const double *beta, const double *rho)
{
    if (N < 1 || !h || !alpha || !beta || !rho) return OR_E_ARG;
    if (!finite_all(h, N) || !finite_all(alpha, N + 1) || !finite_all(beta, N + 1) ||
        !finite_all(rho, N + 1))
        return OR_E_NONFINITE;
    for (int e = 0; e < N; ++e)
        if (!(h[e] > 0.0)) return OR_E_MODEL;
    for (int e = 0; e <= N; ++e) {
        if (!(rho[e] > 0.0) || !(beta[e] > 0.0) || !(alpha[e] > beta[e])) return OR_E_MODEL;
    }
    return OR_OK;
}

/* Validate the (lambda, c) grid: L>=1, lambda>0; V>=2, c strictly increasing, c0>0
 * (reading S9), and the range guard k*h <= 350 (S9). */
static int validate_grid(const double *lam, int64_t L, const double *c, int64_t V)
{
    if (!lam || !c || L < 1 || V < 2) return OR_E_ARG;
    if (!finite_all(lam, L) || !finite_all(c, V)) return OR_E_NONFINITE;
    for (int64_t i = 0; i < L; ++i)
        if (!(lam[i] > 0.0)) return OR_E_GRID;
    if (!(c[0] > 0.0)) return OR_E_GRID;
    for (int64_t j = 1; j < V; ++j)
        if (!(c[j] > c[j - 1])) return OR_E_GRID;
    return OR_OK;
}

static int validate_range(int32_t N, const double *h, const double *lam, int64_t L)
{
    for (int64_t i = 0; i < L; ++i) {
        double k = OR_TWO_PI / lam[i];
        for (int e = 0; e < N; ++e)
            if (k * h[e] > OR_MAX_KH) return OR_E_RANGE;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ O1, O2 */

double oracle_wavenumber(double lambda) { return OR_TWO_PI / lambda; }

/* O2 (reading S4): while c' lies within 1e-4 m/s of any alpha_e or beta_e (e = 0..N,
 * half-space included), c' <- c' * (1 - 1e-4).  The reported C_t stays the grid value. */
double oracle_perturb_velocity(int32_t N, const double *alpha, const double *beta, double c)
{
    for (;;) {
        int near = 0;
        for (int e = 0; e <= N; ++e) {
            if (fabs(c - alpha[e]) < OR_PERTURB_TOL || fabs(c - beta[e]) < OR_PERTURB_TOL) {
                near = 1;
                break;
            }
        }
        if (!near) return c;
        c = c * (1.0 - OR_PERTURB_FACTOR);
    }
}

/* ------------------------------------------------------------------ O3-O5
 * The element / assembly / dense-LU steps live in masw_det_core.h, instantiated for fp64
 * (the oracle), for long double (its rounding-error audit, reading S15') and for binary128
 * (the points where fp64 cannot resolve the sign, reading S15'', below).  The math macros
 * name each type's libm / libquadmath functions.
 */
#define REAL double
#define OR_CTYPE double complex
#define SFX d
#define OR_CSQRT csqrt
#define OR_CCOSH ccosh
#define OR_CSINH csinh
#define OR_CABS cabs
#define OR_CRE creal
#define OR_CIM cimag
#define OR_RABS fabs
#define OR_RMAX fmax
#define OR_FREXP frexp
#define OR_LDEXP ldexp
#define OR_FINITE isfinite
#define OR_CMPLX(a, b) CMPLX(a, b)
#include "masw_det_core.h"
#undef REAL
#undef OR_CTYPE
#undef SFX
#undef OR_CSQRT
#undef OR_CCOSH
#undef OR_CSINH
#undef OR_CABS
#undef OR_CRE
#undef OR_CIM
#undef OR_RABS
#undef OR_RMAX
#undef OR_FREXP
#undef OR_LDEXP
#undef OR_FINITE
#undef OR_CMPLX
#define REAL long double
#define OR_CTYPE long double complex
#define SFX ld
#define OR_CSQRT csqrtl
#define OR_CCOSH ccoshl
#define OR_CSINH csinhl
#define OR_CABS cabsl
#define OR_CRE creall
#define OR_CIM cimagl
#define OR_RABS fabsl
#define OR_RMAX fmaxl
#define OR_FREXP frexpl
#define OR_LDEXP ldexpl
#define OR_FINITE isfinite
#define OR_CMPLX(a, b) CMPLXL(a, b)
#include "masw_det_core.h"
#undef REAL
#undef OR_CTYPE
#undef SFX
#undef OR_CSQRT
#undef OR_CCOSH
#undef OR_CSINH
#undef OR_CABS
#undef OR_CRE
#undef OR_CIM
#undef OR_RABS
#undef OR_RMAX
#undef OR_FREXP
#undef OR_LDEXP
#undef OR_FINITE
#undef OR_CMPLX
#define REAL __float128
#define OR_CTYPE __complex128
#define SFX q
#define OR_CSQRT csqrtq
#define OR_CCOSH ccoshq
#define OR_CSINH csinhq
#define OR_CABS cabsq
#define OR_CRE crealq
#define OR_CIM cimagq
#define OR_RABS fabsq
#define OR_RMAX fmaxq
#define OR_FREXP frexpq
#define OR_LDEXP ldexpq
#define OR_FINITE finiteq
#define OR_CMPLX(a, b) __builtin_complex((__float128)(a), (__float128)(b))
#include "masw_det_core.h"
#undef REAL
#undef OR_CTYPE
#undef SFX
#undef OR_CSQRT
#undef OR_CCOSH
#undef OR_CSINH
#undef OR_CABS
#undef OR_CRE
#undef OR_CIM
#undef OR_RABS
#undef OR_RMAX
#undef OR_FREXP
#undef OR_LDEXP
#undef OR_FINITE
#undef OR_CMPLX

typedef __complex128 cplx_q;
typedef long double complex cplx_ld;
_Static_assert(sizeof(cplx_ld) <= sizeof(cplx_q), "scratch reuse");

/* ------------------------------------------------------------------ reading S15''
 * Where the fp64 evaluation cannot resolve the sign.  As c -> 0 (all waves evanescent) the
 * App. A brackets are O(c^2) .. O(c^4) differences of O(cosh^2) terms: D -> a b (k h)^2 for
 * small k h (a = c^2/alpha^2, b = c^2/beta^2), with absolute rounding ~u in cosh ~ 1, and the
 * element's soft part is a further (k h)^2 below its stiff part; for thick layers the
 * relative error of D tends to ~16 u (beta/c)^4.  So the relative error of an fp64 det K is
 * of the order of
 *     P(c, k) = u max_e [ 16 (beta_e/c)^4 + (alpha_e beta_e / c^2)^2 / (k h_e)^4 ],
 * u = 2^-53 (measured against 60-digit mpmath on random layered models: error / P <= 30,
 * median ~1; tests/test_oracle_pins.py pins the bound and the binary128 values).  Where
 * P > OR_QUAD_TAU the oracle evaluates the same formulas in a wider type: x87 long double
 * (u = 2^-64) while P 2^-11 <= OR_QUAD_TAU, else binary128 (u = 2^-113, error scale P 2^-60).
 * So every oracle determinant has an error scale below OR_QUAD_TAU.
 */
static const double OR_QUAD_TAU = 1e-6;

double oracle_fp64_error_bound(int32_t N, const double *h, const double *alpha,
                               const double *beta, double k, double c)
{
    const double c2 = c * c, c4 = c2 * c2;
    double worst = 0.0;
    for (int e = 0; e < N; ++e) {
        const double b2 = beta[e] * beta[e];
        const double ab = alpha[e] * beta[e];
        const double kh = k * h[e];
        const double kh2 = kh * kh;
        const double t = (16.0 * b2 * b2 + (ab * ab) / (kh2 * kh2)) / c4;
        if (t > worst) worst = t;
    }
    return ldexp(worst, -53);
}

/* O5 at one (lambda, c) as the oracle evaluates it (reading S15''): the fp64 instance, or the
 * long double / binary128 instance of the same formulas where P(c', k) > OR_QUAD_TAU (c' the
 * perturbed velocity the matrix is assembled at).  Kq: scratch of n*n binary128 entries (also
 * used as the long double scratch: sizeof(cplx_ld) <= sizeof(cplx_q)). */
static int det_at(int32_t N, const double *h, const double *alpha, const double *beta,
                  const double *rho, double lambda, double c, cplx *K, cplx_q *Kq, cplx *mant,
                  int *exp2)
{
    const double k = OR_TWO_PI / lambda;
    const double cp = oracle_perturb_velocity(N, alpha, beta, c);
    const double P = oracle_fp64_error_bound(N, h, alpha, beta, k, cp);
    if (P <= OR_QUAD_TAU) return det_at_d(N, h, alpha, beta, rho, lambda, c, K, mant, exp2);
    if (ldexp(P, -11) <= OR_QUAD_TAU) {
        cplx_ld ml = 0.0;
        const int st = det_at_ld(N, h, alpha, beta, rho, lambda, c, (cplx_ld *)Kq, &ml, exp2);
        *mant = CMPLX((double)creall(ml), (double)cimagl(ml));
        return st;
    }
    cplx_q mq = 0.0;
    const int st = det_at_q(N, h, alpha, beta, rho, lambda, c, Kq, &mq, exp2);
    *mant = CMPLX((double)crealq(mq), (double)cimagq(mq));
    return st;
}


/* Exported for the pins: Ke as 16 complex numbers, row-major, (re, im) interleaved. */
void oracle_layer_element(double h, double alpha, double beta, double rho, double k, double c,
                          double *out32)
{
    cplx Ke[4][4];
    layer_element_d(h, alpha, beta, rho, k, c, Ke, -1, 1.0);
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            out32[2 * (4 * a + b)] = creal(Ke[a][b]);
            out32[2 * (4 * a + b) + 1] = cimag(Ke[a][b]);
        }
}

void oracle_halfspace_element(double alpha, double beta, double rho, double k, double c,
                              double *out8)
{
    cplx Kh[2][2];
    halfspace_element_d(alpha, beta, rho, k, c, Kh, -1, 1.0);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            out8[2 * (2 * a + b)] = creal(Kh[a][b]);
            out8[2 * (2 * a + b) + 1] = cimag(Kh[a][b]);
        }
}

void oracle_assemble(int32_t N, const double *h, const double *alpha, const double *beta,
                     const double *rho, double k, double c, double *out /* [n*n*2] */)
{
    int n = 2 * (N + 1);
    cplx *K = (cplx *)malloc(sizeof(cplx) * n * n);
    assemble_d(N, h, alpha, beta, rho, k, c, K, -1, -1, 1.0);
    for (int i = 0; i < n * n; ++i) {
        out[2 * i] = creal(K[i]);
        out[2 * i + 1] = cimag(K[i]);
    }
    free(K);
}

/* Exported for the pins: determinant of a dense complex matrix ((re, im) interleaved). */
int oracle_det_dense(int32_t n, const double *a /* [n*n*2] */, double *mant2, int32_t *exp2)
{
    cplx *A = (cplx *)malloc(sizeof(cplx) * n * n);
    for (int i = 0; i < n * n; ++i) A[i] = a[2 * i] + I * a[2 * i + 1];
    cplx m = 0.0;
    int e = 0;
    int st = det_lu_d(n, A, &m, &e);
    free(A);
    mant2[0] = creal(m);
    mant2[1] = cimag(m);
    *exp2 = e;
    return st;
}

int oracle_det(int32_t N, const double *h, const double *alpha, const double *beta,
               const double *rho, double lambda, double c, double *mant2, int32_t *exp2)
{
    int n = 2 * (N + 1);
    cplx *K = (cplx *)malloc(sizeof(cplx) * n * n);
    cplx_q *Kq = (cplx_q *)malloc(sizeof(cplx_q) * n * n);
    cplx m = 0.0;
    int e = 0;
    int st = det_at(N, h, alpha, beta, rho, lambda, c, K, Kq, &m, &e);
    free(K);
    free(Kq);
    mant2[0] = creal(m);
    mant2[1] = cimag(m);
    *exp2 = e;
    return st;
}

/* The fp64 instance alone (what oracle_det returned before reading S15''; for the pins). */
int oracle_det_fp64(int32_t N, const double *h, const double *alpha, const double *beta,
                    const double *rho, double lambda, double c, double *mant2, int32_t *exp2)
{
    int n = 2 * (N + 1);
    cplx *K = (cplx *)malloc(sizeof(cplx) * n * n);
    cplx m = 0.0;
    int e = 0;
    int st = det_at_d(N, h, alpha, beta, rho, lambda, c, K, &m, &e);
    free(K);
    mant2[0] = creal(m);
    mant2[1] = cimag(m);
    *exp2 = e;
    return st;
}

/* The binary128 instance alone: mantissa as (hi, lo) double pairs of re and im
 * (mant4 = [re_hi, re_lo, im_hi, im_lo]), for the pins against mpmath. */
int oracle_det_q(int32_t N, const double *h, const double *alpha, const double *beta,
                 const double *rho, double lambda, double c, double *mant4, int32_t *exp2)
{
    int n = 2 * (N + 1);
    cplx_q *K = (cplx_q *)malloc(sizeof(cplx_q) * n * n);
    cplx_q m = 0.0;
    int e = 0;
    int st = det_at_q(N, h, alpha, beta, rho, lambda, c, K, &m, &e);
    free(K);
    const __float128 re = crealq(m), im = cimagq(m);
    mant4[0] = (double)re;
    mant4[1] = (double)(re - (__float128)mant4[0]);
    mant4[2] = (double)im;
    mant4[3] = (double)(im - (__float128)mant4[2]);
    *exp2 = e;
    return st;
}

/* Conditioning of det K with respect to the rounding of the elementary-function values that
 * every fp64 evaluation of the Kausel-Roesset formulas must compute (reading S15'):
 *   kappa = 2^-53 * sum over layers e, values v in {cosh, sinh of both waves, r, s} (and r, s
 *           of the half-space) of |d ln det / d ln v|,
 * i.e. the first-order relative change of det K when each such value is off by one unit
 * roundoff.  Derivatives by finite differences (relative step 2^-30) in long double. */
static long double det_ld_value(int32_t N, const double *h, const double *alpha,
                                const double *beta, const double *rho, double lambda,
                                double c, cplx_ld *K, int pe, int pw, long double pf, int *st,
                                cplx_ld *m_out, int *e_out)
{
    cplx_ld m = 0.0;
    int e = 0;
    *st = det_at_p_ld(N, h, alpha, beta, rho, lambda, c, K, &m, &e, pe, pw, pf);
    *m_out = m;
    *e_out = e;
    return 0.0L;
}

int oracle_det_kappa(int32_t N, const double *h, const double *alpha, const double *beta,
                     const double *rho, double lambda, double c, double *kappa)
{
    int n = 2 * (N + 1);
    cplx_ld *K = (cplx_ld *)malloc(sizeof(cplx_ld) * n * n);
    cplx_ld m0, m1;
    int e0, e1, st;
    det_ld_value(N, h, alpha, beta, rho, lambda, c, K, -1, -1, 1.0L, &st, &m0, &e0);
    if (st != OR_OK || creall(m0) == 0.0L) {
        free(K);
        *kappa = INFINITY;
        return st;
    }
    const long double step = ldexpl(1.0L, -30), unit = ldexpl(1.0L, -53);
    long double sum = 0.0L;
    for (int pe = 0; pe <= N; ++pe) {
        for (int pw = (pe == N ? 4 : 0); pw < 6; ++pw) {
            det_ld_value(N, h, alpha, beta, rho, lambda, c, K, pe, pw, 1.0L + step, &st, &m1, &e1);
            if (st != OR_OK) {
                free(K);
                *kappa = INFINITY;
                return st;
            }
            /* d = (m1 2^e1 - m0 2^e0) / (m0 2^e0) */
            cplx_ld ratio = (m1 / m0) * ldexpl(1.0L, e1 - e0);
            sum += cabsl(ratio - 1.0L) / step;
        }
    }
    free(K);
    *kappa = (double)(sum * unit);
    return OR_OK;
}

/* The same determinant carried in long double (reading S15'): mantissa rounded to double. */
int oracle_det_ld(int32_t N, const double *h, const double *alpha, const double *beta,
                  const double *rho, double lambda, double c, double *mant2, int32_t *exp2)
{
    int n = 2 * (N + 1);
    cplx_ld *K = (cplx_ld *)malloc(sizeof(cplx_ld) * n * n);
    cplx_ld m = 0.0;
    int e = 0;
    int st = det_at_ld(N, h, alpha, beta, rho, lambda, c, K, &m, &e);
    free(K);
    mant2[0] = (double)creall(m);
    mant2[1] = (double)cimagl(m);
    *exp2 = e;
    return st;
}

/* ------------------------------------------------------------------ O6 sign */
static int sign_re(cplx m)
{
    double re = creal(m);
    return (re > 0.0) - (re < 0.0);
}

/* ------------------------------------------------------------------ O7 scan (Algorithm 1)
 * d_old = det(V[0]); d_new = det(V[1]); n = 1;
 *   while sign(d_old) == sign(d_new): n++, d_old = d_new, d_new = det(V[n]);  C_t = V[n].
 * Readings: 0 is a sign of its own (S6); returned velocity is the unperturbed V[n] (S7);
 * no change over the grid -> idx -1, C_t NaN (S8); a non-finite det -> idx -2 (S9).
 * *ndet counts the determinants evaluated.
 */
static void scan_row(int32_t N, const double *h, const double *alpha, const double *beta,
                     const double *rho, double lambda, const double *c, int64_t V, cplx *K,
                     cplx_q *Kq, double *ct, int32_t *idx, int64_t *ndet)
{
    int64_t count = 0;
    int s_old = 0;
    for (int64_t j = 0; j < V; ++j) {
        cplx m = 0.0;
        int e;
        int st = det_at(N, h, alpha, beta, rho, lambda, c[j], K, Kq, &m, &e);
        ++count;
        if (st != OR_OK) {
            *idx = OR_IDX_NONFINITE;
            *ct = NAN;
            *ndet = count;
            return;
        }
        int s_new = sign_re(m);
        if (j > 0 && s_new != s_old) {
            *idx = (int32_t)j;
            *ct = c[j];
            *ndet = count;
            return;
        }
        s_old = s_new;
    }
    *idx = OR_IDX_NO_CHANGE;
    *ct = NAN;
    *ndet = count;
}

/* ------------------------------------------------------------------ row threads */
typedef struct {
    int64_t M, L, V;
    int32_t N;
    const double *h, *alpha, *beta, *rho; /* SoA [M][N], [M][N+1] */
    const double *lam, *c;
    double *ct;     /* [M][L] */
    int32_t *idx;   /* [M][L] */
    int64_t *ndet;  /* [M][L] or NULL */
    atomic_llong next;
} rows_job;

static void *rows_worker(void *arg)
{
    rows_job *J = (rows_job *)arg;
    int n = 2 * (J->N + 1);
    cplx *K = (cplx *)malloc(sizeof(cplx) * n * n);
    cplx_q *Kq = (cplx_q *)malloc(sizeof(cplx_q) * n * n);
    const int64_t total = J->M * J->L;
    for (;;) {
        int64_t r = atomic_fetch_add(&J->next, 1);
        if (r >= total) break;
        int64_t m = r / J->L, i = r % J->L;
        int32_t N = J->N;
        int64_t nd = 0;
        scan_row(N, J->h + m * N, J->alpha + m * (N + 1), J->beta + m * (N + 1),
                 J->rho + m * (N + 1), J->lam[i], J->c, J->V, K, Kq, &J->ct[r], &J->idx[r], &nd);
        if (J->ndet) J->ndet[r] = nd;
    }
    free(K);
    free(Kq);
    return NULL;
}

static void run_rows(rows_job *J, int nthreads)
{
    atomic_init(&J->next, 0);
    if (nthreads <= 1) {
        rows_worker(J);
        return;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, rows_worker, J) == 0) ++started;
    if (started == 0) rows_worker(J);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
}

/* ------------------------------------------------------------------ O8 misfit (Algorithm 2)
 * e = 0; for i = 1..l: e += |C_t[i] - C_e[i]| / C_e[i];  m = e / l.
 * Readings: e starts at 0, index order (S12); any non-finite C_t -> +inf (S8).
 * Errors: l < 1 -> OR_E_ARG; C_e not finite -> OR_E_NONFINITE; C_e <= 0 -> OR_E_ARG.
 */
int oracle_misfit(const double *ct, const double *ce, int64_t L, double *out)
{
    if (!ct || !ce || !out || L < 1) return OR_E_ARG;
    if (!finite_all(ce, L)) return OR_E_NONFINITE;
    for (int64_t i = 0; i < L; ++i)
        if (!(ce[i] > 0.0)) return OR_E_ARG;
    double e = 0.0;
    for (int64_t i = 0; i < L; ++i) {
        if (!isfinite(ct[i])) {
            *out = INFINITY;
            return OR_OK;
        }
        e = e + fabs(ct[i] - ce[i]) / ce[i];
    }
    *out = e / (double)L;
    return OR_OK;
}

/* Same sum in long double, for tolerance audits. */
int oracle_misfit_ld(const double *ct, const double *ce, int64_t L, double *out)
{
    if (!ct || !ce || !out || L < 1) return OR_E_ARG;
    long double e = 0.0L;
    for (int64_t i = 0; i < L; ++i) {
        if (!isfinite(ct[i])) {
            *out = INFINITY;
            return OR_OK;
        }
        e += fabsl((long double)ct[i] - (long double)ce[i]) / (long double)ce[i];
    }
    *out = (double)(e / (long double)L);
    return OR_OK;
}

/* ------------------------------------------------------------------ public: one curve */
static int validate_all(int64_t M, int32_t N, const double *h, const double *alpha,
                        const double *beta, const double *rho, const double *lam, int64_t L,
                        const double *c, int64_t V)
{
    if (M < 0 || N < 1) return OR_E_ARG;
    int st = validate_grid(lam, L, c, V);
    if (st != OR_OK) return st;
    for (int64_t m = 0; m < M; ++m) {
        st = oracle_validate_model(N, h + m * N, alpha + m * (N + 1), beta + m * (N + 1),
                                   rho + m * (N + 1));
        if (st != OR_OK) return st;
    }
    for (int64_t m = 0; m < M; ++m) {
        st = validate_range(N, h + m * N, lam, L);
        if (st != OR_OK) return st;
    }
    return OR_OK;
}

static int worst_row_status(const int32_t *idx, int64_t n)
{
    for (int64_t r = 0; r < n; ++r)
        if (idx[r] < 0) return OR_WARN_NO_SIGN_CHANGE;
    return OR_OK;
}

/* C_t for one model (Algorithm 1 per wavelength).  ndet may be NULL. */
int oracle_curve(int32_t N, const double *h, const double *alpha, const double *beta,
                 const double *rho, const double *lam, int64_t L, const double *c, int64_t V,
                 double *ct, int32_t *idx, int64_t *ndet, int32_t nthreads)
{
    int st = validate_all(1, N, h, alpha, beta, rho, lam, L, c, V);
    if (st != OR_OK) return st;
    rows_job J;
    J.M = 1; J.L = L; J.V = V; J.N = N;
    J.h = h; J.alpha = alpha; J.beta = beta; J.rho = rho;
    J.lam = lam; J.c = c; J.ct = ct; J.idx = idx; J.ndet = ndet;
    run_rows(&J, nthreads);
    return worst_row_status(idx, L);
}

/* ------------------------------------------------------------------ O9 ensemble */
int oracle_ensemble(int64_t M, int32_t N, const double *h, const double *alpha,
                    const double *beta, const double *rho, const double *lam, int64_t L,
                    const double *c, int64_t V, const double *ce, double *ct, int32_t *idx,
                    double *misfit, int64_t *ndet, int64_t *best, int32_t nthreads)
{
    int st = validate_all(M, N, h, alpha, beta, rho, lam, L, c, V);
    if (st != OR_OK) return st;
    if (ce) {
        if (!finite_all(ce, L)) return OR_E_NONFINITE;
        for (int64_t i = 0; i < L; ++i)
            if (!(ce[i] > 0.0)) return OR_E_ARG;
    }
    if (M == 0) {
        if (best) *best = -1;
        return OR_OK;
    }
    rows_job J;
    J.M = M; J.L = L; J.V = V; J.N = N;
    J.h = h; J.alpha = alpha; J.beta = beta; J.rho = rho;
    J.lam = lam; J.c = c; J.ct = ct; J.idx = idx; J.ndet = ndet;
    run_rows(&J, nthreads);
    if (ce && misfit) {
        for (int64_t m = 0; m < M; ++m) oracle_misfit(ct + m * L, ce, L, &misfit[m]);
        if (best) {
            int64_t b = 0;
            for (int64_t m = 1; m < M; ++m)
                if (misfit[m] < misfit[b]) b = m; /* strict: ties -> lowest id */
            *best = b;
        }
    }
    return worst_row_status(idx, M * L);
}

/* ------------------------------------------------------------------ O10 det grid
 * Every (lambda_i, c_j) determinant, no early exit ("grid" view).
 * Outputs [L][V]: mantissa (re, im) and exponent; status[L][V] (0 or OR_E_NONFINITE).
 */
typedef struct {
    int32_t N;
    const double *h, *alpha, *beta, *rho, *lam, *c;
    int64_t L, V;
    double *mre, *mim;
    int32_t *ex, *status;
    int extended; /* 1: long double audit instance, 2: conditioning kappa (reading S15') */
    atomic_llong next;
} grid_job;

static void *grid_worker(void *arg)
{
    grid_job *G = (grid_job *)arg;
    int n = 2 * (G->N + 1);
    cplx *K = (cplx *)malloc(sizeof(cplx) * n * n);
    cplx_ld *Kl = (cplx_ld *)malloc(sizeof(cplx_ld) * n * n);
    cplx_q *Kq = (cplx_q *)malloc(sizeof(cplx_q) * n * n);
    for (;;) {
        int64_t i = atomic_fetch_add(&G->next, 1);
        if (i >= G->L) break;
        for (int64_t j = 0; j < G->V; ++j) {
            double re, im;
            int e = 0, st;
            if (G->extended == 2) {
                double kap = 0.0;
                st = oracle_det_kappa(G->N, G->h, G->alpha, G->beta, G->rho, G->lam[i], G->c[j], &kap);
                re = kap;
                im = 0.0;
            } else if (G->extended) {
                cplx_ld m = 0.0;
                st = det_at_ld(G->N, G->h, G->alpha, G->beta, G->rho, G->lam[i], G->c[j], Kl, &m, &e);
                re = (double)creall(m);
                im = (double)cimagl(m);
            } else {
                cplx m = 0.0;
                st = det_at(G->N, G->h, G->alpha, G->beta, G->rho, G->lam[i], G->c[j], K, Kq, &m, &e);
                re = creal(m);
                im = cimag(m);
            }
            int64_t o = i * G->V + j;
            G->mre[o] = re;
            G->mim[o] = im;
            G->ex[o] = e;
            if (G->status) G->status[o] = st;
        }
    }
    free(K);
    free(Kl);
    free(Kq);
    return NULL;
}

static int det_grid_impl(int extended, int32_t N, const double *h, const double *alpha,
                         const double *beta, const double *rho, const double *lam, int64_t L,
                         const double *c, int64_t V, double *mant_re, double *mant_im,
                         int32_t *exp2, int32_t *status, int32_t nthreads);

int oracle_det_grid(int32_t N, const double *h, const double *alpha, const double *beta,
                    const double *rho, const double *lam, int64_t L, const double *c, int64_t V,
                    double *mant_re, double *mant_im, int32_t *exp2, int32_t *status,
                    int32_t nthreads)
{
    return det_grid_impl(0, N, h, alpha, beta, rho, lam, L, c, V, mant_re, mant_im, exp2,
                         status, nthreads);
}

/* kappa (oracle_det_kappa) on the grid, written to mant_re (reading S15'). */
int oracle_det_grid_kappa(int32_t N, const double *h, const double *alpha, const double *beta,
                          const double *rho, const double *lam, int64_t L, const double *c,
                          int64_t V, double *kappa, int32_t *status, int32_t nthreads)
{
    double *im = (double *)malloc(sizeof(double) * L * V);
    int32_t *ex = (int32_t *)malloc(sizeof(int32_t) * L * V);
    int st = det_grid_impl(2, N, h, alpha, beta, rho, lam, L, c, V, kappa, im, ex, status,
                           nthreads);
    free(im);
    free(ex);
    return st;
}

/* The grid in long double (reading S15': measures the fp64 oracle's rounding error). */
int oracle_det_grid_ld(int32_t N, const double *h, const double *alpha, const double *beta,
                       const double *rho, const double *lam, int64_t L, const double *c,
                       int64_t V, double *mant_re, double *mant_im, int32_t *exp2,
                       int32_t *status, int32_t nthreads)
{
    return det_grid_impl(1, N, h, alpha, beta, rho, lam, L, c, V, mant_re, mant_im, exp2,
                         status, nthreads);
}

static int det_grid_impl(int extended, int32_t N, const double *h, const double *alpha,
                         const double *beta, const double *rho, const double *lam, int64_t L,
                         const double *c, int64_t V, double *mant_re, double *mant_im,
                         int32_t *exp2, int32_t *status, int32_t nthreads)
{
    int st = validate_all(1, N, h, alpha, beta, rho, lam, L, c, V);
    if (st != OR_OK) return st;
    grid_job G;
    G.N = N; G.h = h; G.alpha = alpha; G.beta = beta; G.rho = rho;
    G.lam = lam; G.c = c; G.L = L; G.V = V;
    G.mre = mant_re; G.mim = mant_im; G.ex = exp2; G.status = status;
    G.extended = extended;
    atomic_init(&G.next, 0);
    if (nthreads <= 1) {
        grid_worker(&G);
        return OR_OK;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, grid_worker, &G) == 0) ++started;
    if (started == 0) grid_worker(&G);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
    return OR_OK;
}
