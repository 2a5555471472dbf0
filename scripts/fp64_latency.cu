// Dependent-chain latency (cycles) of the FP64 ops the scan kernel is made of, on one warp,
// and the FP64 throughput with 1..16 warps per SM (development aid).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_latency scripts/fp64_latency.cu
#include <cstdio>

#define CHAIN 256

__global__ void lat_dfma(double *out, long long *cyc, double a, double b)
{
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < CHAIN; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_dmul(double *out, long long *cyc, double a, double b)
{
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < CHAIN; ++i) x = x * a;
    long long t1 = clock64();
    out[threadIdx.x] = x + b;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_rcp(double *out, long long *cyc, double a, double b)
{
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < CHAIN; ++i) {
        double y;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        x = y;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + b;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_setp(double *out, long long *cyc, double a, double b)
{
    // DSETP -> predicated select -> next DFMA
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < CHAIN; ++i) x = (x > b) ? fma(x, a, -b) : fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// throughput: 8 independent chains per thread
__global__ void thr_dfma(double *out, double a, double b, int iters)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// throughput with a single dependent chain per thread (latency-bound per warp)
__global__ void thr_dfma1(double *out, double a, double b, int iters)
{
    double x = threadIdx.x * 1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x = fma(x, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main()
{
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 64);
    long long h;
    auto run = [&](const char *name, void (*k)(double *, long long *, double, double)) {
        k<<<1, 32>>>(out, cyc, 0.999, 1e-3);
        k<<<1, 32>>>(out, cyc, 0.999, 1e-3);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-10s latency %.2f cycles\n", name, (double)h / CHAIN);
    };
    run("DFMA", lat_dfma);
    run("DMUL", lat_dmul);
    run("MUFU.RCP64H+mov", lat_rcp);
    run("DSETP+sel+DFMA", lat_setp);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int ilp = 0; ilp < 2; ++ilp) {
        for (int warps = 1; warps <= 32; warps *= 2) {
            auto launch = [&]() {
                if (ilp) thr_dfma<<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
                else thr_dfma1<<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 8 * iters * 32.0 * warps * sms;
            printf("%s warps/SM %2d: %.2f TFLOP/s\n", ilp ? "8 chains/thread" : "1 chain/thread ", warps,
                   flops / (ms * 1e-3) / 1e12);
        }
    }
    printf("SMs %d, clock %d kHz\n", sms, clk);
    return 0;
}
