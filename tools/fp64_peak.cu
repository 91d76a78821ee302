// fp64_peak.cu -- DFMA-chain microbenchmark: the FP64 roofline denominator
// (MEASURED_PEAKS.json has no fp64 entry).  Not part of the product library.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void dfma_chains(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
}

// Returns measured TFLOP/s (2 flops per DFMA), best of `reps` launches.
extern "C" double fp64_peak_tflops(int reps)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    double best = 0.0;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

// ---- latency constants for the latency-bound configs (C1, C2) -------------
// dependent DFMA chain, one warp per SM: clocks per dependent FP64 op
__global__ void dfma_dep(double *out, int iters, double a, double b, long long *cyc)
{
    double x = threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) x = fma(x, a, b);
    long long t1 = clock64();
    if (x == 123.456) out[0] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// shared-memory store -> barrier -> neighbour load round trip (one CTA per SM)
__global__ void bar_trip(double *out, int iters, long long *cyc)
{
    __shared__ double sh[1024];
    double v = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        sh[threadIdx.x] = v;
        __syncthreads();
        v += sh[(threadIdx.x + 1) % blockDim.x];
    }
    long long t1 = clock64();
    if (v == 123.456) out[0] = v;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static double avg_cycles(long long *dcyc, int n)
{
    long long h[1024];
    cudaMemcpy(h, dcyc, sizeof(long long) * n, cudaMemcpyDeviceToHost);
    double a = 0;
    for (int i = 0; i < n; ++i) a += (double)h[i];
    return a / n;
}

// clocks per dependent DFMA (FP64 latency)
extern "C" double fp64_latency_clk(void)
{
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * 1024);
    const int iters = 4096;
    dfma_dep<<<1, 32>>>(out, iters, 0.999999, 1e-7, cyc);
    dfma_dep<<<1, 32>>>(out, iters, 0.999999, 1e-7, cyc);
    cudaDeviceSynchronize();
    const double c = avg_cycles(cyc, 1) / iters;
    cudaFree(out);
    cudaFree(cyc);
    return c;
}

// clocks per smem store + __syncthreads + smem load with `warps` warps per CTA
extern "C" double barrier_trip_clk(int warps)
{
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * 1024);
    const int iters = 4096;
    bar_trip<<<1, 32 * warps>>>(out, iters, cyc);
    bar_trip<<<1, 32 * warps>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    const double c = avg_cycles(cyc, 1) / iters;
    cudaFree(out);
    cudaFree(cyc);
    return c;
}
