// Accuracy of the sm_100a MUFU fp64 seeds (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64) and of
// the refinement sequences built on them (development aid for masw_det.cuh).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mufu_accuracy scripts/mufu_accuracy.cu
//   ./scripts/mufu_accuracy
//
// For x = m * 2^e over a dense sweep of mantissas m in [1, 4) and a spread of exponents, the
// GPU writes the seed and the refined values; the host measures relative errors against
// long-double references (64-bit significand), in units of 2^-53.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ double rcp_seed(double x)
{
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_seed(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

__global__ void kern(const double *x, int n, double *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    // rcp: seed, two Newton steps, one cubic step (y (1 + e + e^2)), cubic + Newton
    const double y0 = rcp_seed(v);
    double e = fma(-v, y0, 1.0);
    double y = fma(y0, e, y0);
    double e2 = fma(-v, y, 1.0);
    const double nn = fma(y, e2, y);
    const double p = fma(e, e, e);
    const double cub = fma(y0, p, y0);
    // rsqrt: seed, two Newton steps (the kernel's), one 2nd-order step
    //   y1 = y0 (1 + e/2 + 3 e^2 / 8),  e = 1 - q y0^2
    const double r0 = rsqrt_seed(v);
    double h = 0.5 * r0;
    double ee = fma(-v * r0, r0, 1.0);
    double r = fma(h, ee, r0);
    h = 0.5 * r;
    double ee2 = fma(-v * r, r, 1.0);
    const double rnn = fma(h, ee2, r);
    const double t = v * r0;
    const double er = fma(-t, r0, 1.0);
    const double pr = fma(er, 0.375, 0.5);
    const double r2o = fma(r0 * er, pr, r0);
    // 3rd-order: y0 (1 + e/2 + 3e^2/8 + 5e^3/16)
    const double pr3 = fma(er, fma(er, 0.3125, 0.375), 0.5);
    const double r3o = fma(r0 * er, pr3, r0);
    double *o = out + 8 * (size_t)i;
    o[0] = y0; o[1] = nn; o[2] = cub; o[3] = r0; o[4] = rnn; o[5] = r2o; o[6] = r3o;
    o[7] = v * rnn;   // sqrt as q * rsqrt
}

int main()
{
    const int nm = 1 << 20;
    const int exps[] = {-40, -13, -3, -1, 0, 1, 2, 7, 20, 33, 60};
    const int ne = sizeof(exps) / sizeof(exps[0]);
    const int n = nm * ne;
    std::vector<double> x(n);
    for (int k = 0; k < ne; ++k)
        for (int i = 0; i < nm; ++i) x[(size_t)k * nm + i] = std::ldexp(1.0 + 3.0 * (i + 0.5) / nm, exps[k]);
    double *dx, *dout;
    cudaMalloc(&dx, n * sizeof(double));
    cudaMalloc(&dout, (size_t)n * 8 * sizeof(double));
    cudaMemcpy(dx, x.data(), n * sizeof(double), cudaMemcpyHostToDevice);
    kern<<<(n + 255) / 256, 256>>>(dx, n, dout);
    std::vector<double> o((size_t)n * 8);
    cudaError_t err = cudaMemcpy(o.data(), dout, o.size() * sizeof(double), cudaMemcpyDeviceToHost);
    if (err != cudaSuccess) {
        printf("cuda error %s\n", cudaGetErrorString(err));
        return 1;
    }
    const char *names[] = {"rcp seed", "rcp 2x Newton", "rcp cubic", "rsqrt seed", "rsqrt 2x Newton",
                           "rsqrt 2nd-order", "rsqrt 3rd-order", "sqrt = q*rsqrt"};
    long double mx[8] = {0};
    const long double ulp = ldexpl(1.0L, -53);
    for (int i = 0; i < n; ++i) {
        const long double v = x[i];
        const long double rc = 1.0L / v, rs = 1.0L / sqrtl(v), sq = sqrtl(v);
        const long double ref[8] = {rc, rc, rc, rs, rs, rs, rs, sq};
        for (int k = 0; k < 8; ++k) {
            long double e = fabsl((long double)o[(size_t)i * 8 + k] / ref[k] - 1.0L);
            if (e > mx[k]) mx[k] = e;
        }
    }
    for (int k = 0; k < 8; ++k)
        printf("%-18s max rel err %.3Le = 2^%.2f = %.3f ulp(2^-53)\n", names[k], mx[k],
               (double)log2l(mx[k]), (double)(mx[k] / ulp));
    return 0;
}
