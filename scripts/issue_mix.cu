// How integer instructions mixed into an FP64 stream cost FP64 throughput on B200 (sm_100a):
// each thread runs 8 independent DFMA chains plus NINT independent integer ops per 8 DFMAs
// (ratio r = NINT / 8), at 16 and 32 warps per SM.  If a warp-wide FP64 instruction occupies
// its SMSP's dispatch for 2 cycles (16 FP64 lanes per SMSP) and an integer one for 1, the FP64
// rate falls as 1 / (1 + r/2); if the integer ops issued in the FP64 pipe's idle cycles for
// free, it would stay flat up to r = 1.  (Development aid for DESIGN.md §5.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/issue_mix scripts/issue_mix.cu
#include <cstdio>

template <int NINT>
__global__ void mix(double *out, unsigned *iout, double a, double b, int iters)
{
    double x[8];
    unsigned v[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = threadIdx.x * 7u + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x[k] = fma(x[k], a, b);
            // NINT / 8 integer ops after each DFMA (spread evenly)
#pragma unroll
            for (int q = 0; q < (NINT + 7) / 8; ++q) {
                const int j = k * ((NINT + 7) / 8) + q;
                if (j < NINT && ((NINT >= 8) || (k % (8 / (NINT ? NINT : 1)) == 0)))
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[j & 15]) : "r"(it), "r"(v[(j + 1) & 15]));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    unsigned t = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) t ^= v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    iout[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int NINT>
void run(double *out, unsigned *iout, int sms, int warps)
{
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mix<NINT><<<sms, 32 * warps>>>(out, iout, 0.999, 1e-3, iters);
    cudaEventRecord(e0);
    mix<NINT><<<sms, 32 * warps>>>(out, iout, 0.999, 1e-3, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * iters * 32.0 * warps * sms;
    const double r = NINT / 8.0;
    printf("int/fp64 %.3f  warps/SM %2d: %6.2f TFLOP/s  (1/(1+r/2) model x %.3f)\n", r, warps,
           flops / (ms * 1e-3) / 1e12, 1.0 / (1.0 + r / 2.0));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main()
{
    double *out;
    unsigned *iout;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&iout, 1 << 24);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {16, 32}) {
        run<0>(out, iout, sms, warps);
        run<1>(out, iout, sms, warps);
        run<2>(out, iout, sms, warps);
        run<4>(out, iout, sms, warps);
        run<6>(out, iout, sms, warps);
        run<8>(out, iout, sms, warps);
        run<16>(out, iout, sms, warps);
    }
    return 0;
}
