/*
 * oracle/masw_det_core.h -- TEST INFRASTRUCTURE ONLY (part of the oracle; see masw_oracle.c).
 *
 * Steps O3-O5 of the oracle (layer element, half-space element, dense assembly, dense
 * partial-pivot LU determinant), written once over a generic real type and included three
 * times by masw_oracle.c:
 *   REAL = double       the oracle proper (fp64, the paper's precision: cuDoubleComplex,
 *                       PAPER.md:248);
 *   REAL = long double  the same arithmetic carried in x87 extended precision, used only to
 *                       measure the fp64 oracle's own rounding error (reading S15');
 *   REAL = __float128   the same arithmetic in IEEE binary128 (libquadmath), used where the
 *                       fp64 evaluation of these formulas cannot resolve the sign of det K
 *                       (reading S15'': c^4 small against (alpha beta)^2 / (k h)^4).
 * Inputs (k, c', model) are doubles in every instance: all three evaluate the same matrix
 * K(fl(2 pi / lambda), c'), they differ only in the rounding of the arithmetic.
 *
 * Expects: REAL, SFX (name suffix) and the math macros of masw_oracle.c (OR_CSQRT, OR_CCOSH,
 * OR_CSINH, OR_CABS, OR_CRE, OR_CIM, OR_RABS, OR_RMAX, OR_FREXP, OR_LDEXP, OR_FINITE,
 * OR_CMPLX) and its complex type OR_CTYPE defined for that type.
 */
#define OR_CAT2(a, b) a##_##b
#define OR_CAT(a, b) OR_CAT2(a, b)
#define OR_NAME(x) OR_CAT(x, SFX)
#define CREAL_T OR_CTYPE

/* ------------------------------------------------------------------ O3 layer element
 * Kausel-Roesset / MASWaves layer stiffness (the paper cites the
 * method only, "stiffness matrix method (Kausel, 1981)"; reading S1).
 * Complex arithmetic throughout, principal square roots (reading S3):
 *   r = sqrt(1 - c^2/alpha^2), s = sqrt(1 - c^2/beta^2)
 *   Cr = cosh(k r h), Sr = sinh(k r h), Cs = cosh(k s h), Ss = sinh(k s h)
 *   D  = 2(1 - Cr Cs) + (1/(r s) + r s) Sr Ss,   f = k rho c^2 / D
 *   k11 = f (Cr Ss/s - r Sr Cs)          k12 = f (Cr Cs - r s Sr Ss - 1) - k rho beta^2 (1 + s^2)
 *   k13 = f (r Sr - Ss/s)                k14 = f (Cs - Cr)
 *   k22 = f (Sr Cs/r - s Cr Ss)          k24 = f (s Ss - Sr/r)
 *   Ke = [[k11, k12, k13, k14], [k12, k22, -k14, k24], [k13, -k14, k11, -k12], [k14, k24, -k12, k22]]
 * Local DOFs (u_top, w_top, u_bot, w_bot).
 */
/* pw >= 0 multiplies one intermediate value by pf (0: Cr, 1: Sr, 2: Cs, 3: Ss, 4: r, 5: s)
 * -- used only by the conditioning measure (reading S15'); pw < 0 leaves the arithmetic
 * untouched. */
static void OR_NAME(layer_element)(REAL h, REAL alpha, REAL beta, REAL rho, REAL k, REAL c,
                                   CREAL_T Ke[4][4], int pw, REAL pf)
{
    CREAL_T r = OR_CSQRT((CREAL_T)(1.0 - (c * c) / (alpha * alpha)));
    CREAL_T s = OR_CSQRT((CREAL_T)(1.0 - (c * c) / (beta * beta)));
    if (pw == 4) r = r * pf;
    if (pw == 5) s = s * pf;
    CREAL_T Cr = OR_CCOSH(k * r * h), Sr = OR_CSINH(k * r * h);
    CREAL_T Cs = OR_CCOSH(k * s * h), Ss = OR_CSINH(k * s * h);
    if (pw == 0) Cr = Cr * pf;
    if (pw == 1) Sr = Sr * pf;
    if (pw == 2) Cs = Cs * pf;
    if (pw == 3) Ss = Ss * pf;
    CREAL_T D = 2.0 * (1.0 - Cr * Cs) + (1.0 / (r * s) + r * s) * Sr * Ss;
    CREAL_T f = k * rho * c * c / D;
    CREAL_T k11 = f * (Cr * Ss / s - r * Sr * Cs);
    CREAL_T k12 = f * (Cr * Cs - r * s * Sr * Ss - 1.0) - k * rho * beta * beta * (1.0 + s * s);
    CREAL_T k13 = f * (r * Sr - Ss / s);
    CREAL_T k14 = f * (Cs - Cr);
    CREAL_T k22 = f * (Sr * Cs / r - s * Cr * Ss);
    CREAL_T k24 = f * (s * Ss - Sr / r);
    CREAL_T M[4][4] = {{k11, k12, k13, k14},
                       {k12, k22, -k14, k24},
                       {k13, -k14, k11, -k12},
                       {k14, k24, -k12, k22}};
    memcpy(Ke, M, sizeof(M));
}

/* ------------------------------------------------------------------ O4 half-space element
 *   K_hs = k rho beta^2 [[ r(1-s^2)/(1-rs),    (1-s^2)/(1-rs) - 2 ],
 *                        [ (1-s^2)/(1-rs) - 2, s(1-s^2)/(1-rs)    ]]
 * (reading S1, S22.)
 */
static void OR_NAME(halfspace_element)(REAL alpha, REAL beta, REAL rho, REAL k, REAL c,
                                       CREAL_T Kh[2][2], int pw, REAL pf)
{
    CREAL_T r = OR_CSQRT((CREAL_T)(1.0 - (c * c) / (alpha * alpha)));
    CREAL_T s = OR_CSQRT((CREAL_T)(1.0 - (c * c) / (beta * beta)));
    if (pw == 4) r = r * pf;
    if (pw == 5) s = s * pf;
    REAL mu = k * rho * beta * beta;
    CREAL_T q = (1.0 - s * s) / (1.0 - r * s);
    Kh[0][0] = mu * r * q;
    Kh[0][1] = mu * q - 2.0 * mu;
    Kh[1][0] = Kh[0][1];
    Kh[1][1] = mu * s * q;
}

/* Dense global assembly: layer e adds Ke into rows/cols 2e..2e+3, the half-space adds
 * K_hs into rows/cols 2N, 2N+1 (PAPER.md:78 order 2(N+1)).  c is used as
 * given (callers pass the perturbed c'). */
/* pe: element whose intermediate value pw is scaled by pf (pe == N: the half-space, pw 4/5);
 * pe < 0: no perturbation (the oracle proper). */
static void OR_NAME(assemble)(int32_t N, const double *h, const double *alpha,
                              const double *beta, const double *rho, double k, double c,
                              CREAL_T *K /* [n*n] */, int pe, int pw, REAL pf)
{
    int n = 2 * (N + 1);
    for (int i = 0; i < n * n; ++i) K[i] = 0.0;
    for (int e = 0; e < N; ++e) {
        CREAL_T Ke[4][4];
        OR_NAME(layer_element)(h[e], alpha[e], beta[e], rho[e], k, c, Ke, e == pe ? pw : -1, pf);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) K[(2 * e + a) * n + (2 * e + b)] += Ke[a][b];
    }
    CREAL_T Kh[2][2];
    OR_NAME(halfspace_element)(alpha[N], beta[N], rho[N], k, c, Kh, pe == N ? pw : -1, pf);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) K[(2 * N + a) * n + (2 * N + b)] += Kh[a][b];
}

/* ------------------------------------------------------------------ O5 determinant
 * Dense LU with partial pivoting (row of largest |a_ik|).  det = (-1)^swaps * prod u_kk,
 * accumulated as mant * 2^exp2 with max(|Re mant|, |Im mant|) in [0.5, 1) (reading S14).
 * Returns OR_OK, or OR_E_NONFINITE if any entry or pivot is not finite.  An all-zero
 * pivot column gives det = 0 exactly (mant = 0, exp2 = 0).
 */
static int OR_NAME(det_lu)(int n, CREAL_T *A, CREAL_T *mant, int *exp2)
{
    for (int i = 0; i < n * n; ++i)
        if (!OR_FINITE(OR_CRE(A[i])) || !OR_FINITE(OR_CIM(A[i]))) return OR_E_NONFINITE;
    CREAL_T m = 1.0;
    int ex = 0;
    for (int kk = 0; kk < n; ++kk) {
        int p = kk;
        REAL best = OR_CABS(A[kk * n + kk]);
        for (int i = kk + 1; i < n; ++i) {
            REAL v = OR_CABS(A[i * n + kk]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        if (best == 0.0) {
            *mant = 0.0;
            *exp2 = 0;
            return OR_OK;
        }
        if (p != kk) {
            for (int j = 0; j < n; ++j) {
                CREAL_T t = A[kk * n + j];
                A[kk * n + j] = A[p * n + j];
                A[p * n + j] = t;
            }
            m = -m;
        }
        CREAL_T piv = A[kk * n + kk];
        for (int i = kk + 1; i < n; ++i) {
            CREAL_T l = A[i * n + kk] / piv;
            for (int j = kk; j < n; ++j) A[i * n + j] -= l * A[kk * n + j];
        }
        m *= piv;
        REAL t = OR_RMAX(OR_RABS(OR_CRE(m)), OR_RABS(OR_CIM(m)));
        if (!OR_FINITE(t)) return OR_E_NONFINITE;
        if (t == 0.0) {
            *mant = 0.0;
            *exp2 = 0;
            return OR_OK;
        }
        int e2;
        OR_FREXP(t, &e2);
        m = OR_CMPLX(OR_LDEXP(OR_CRE(m), -e2), OR_LDEXP(OR_CIM(m), -e2));
        ex += e2;
    }
    *mant = m;
    *exp2 = ex;
    return OR_OK;
}

/* O1-O5 for one (model, lambda, c): k, perturb, assemble, dense det. */
static int OR_NAME(det_at_p)(int32_t N, const double *h, const double *alpha,
                             const double *beta, const double *rho, double lambda, double c,
                             CREAL_T *K, CREAL_T *mant, int *exp2, int pe, int pw, REAL pf)
{
    double k = OR_TWO_PI / lambda;
    double cp = oracle_perturb_velocity(N, alpha, beta, c);
    OR_NAME(assemble)(N, h, alpha, beta, rho, k, cp, K, pe, pw, pf);
    return OR_NAME(det_lu)(2 * (N + 1), K, mant, exp2);
}

static int OR_NAME(det_at)(int32_t N, const double *h, const double *alpha, const double *beta,
                           const double *rho, double lambda, double c, CREAL_T *K,
                           CREAL_T *mant, int *exp2)
{
    return OR_NAME(det_at_p)(N, h, alpha, beta, rho, lambda, c, K, mant, exp2, -1, -1, 1.0);
}

#undef OR_CAT2
#undef OR_CAT
#undef OR_NAME
#undef CREAL_T
