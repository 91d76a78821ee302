// probe: the C5 step's DFMA pattern (78 distinct weight registers, 18-value window,
// 12 chains) without any shared memory or barrier: clocks per "step" per SM sub-partition
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256, 1) pat(const double *wsrc, double *out, int iters, long long *cyc)
{
    constexpr int J = 6, NS = 13, W = 18;
    double w[J][NS], x[J], win[W];
    for (int j = 0; j < J; ++j)
        for (int c = 0; c < NS; ++c) w[j][c] = wsrc[(j * NS + c) * 256 + threadIdx.x];
    for (int j = 0; j < J; ++j) x[j] = 1.0 + 1e-3 * j + 1e-6 * threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 6; ++m) win[m] = x[m] * 0.5;
#pragma unroll
        for (int j = 0; j < J; ++j) win[6 + j] = x[j];
#pragma unroll
        for (int m = 0; m < 6; ++m) win[12 + m] = x[m] * 0.25;
        double acc[J], acc2[J];
        if (MODE == 0) {           // two half chains per node, tap-major
            constexpr int H = 7;
#pragma unroll
            for (int j = 0; j < J; ++j) { acc[j] = w[j][0] * win[j]; acc2[j] = w[j][H] * win[j + H]; }
#pragma unroll
            for (int c = 1; c < H; ++c)
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    acc[j] = fma(w[j][c], win[j + c], acc[j]);
                    if (H + c < NS) acc2[j] = fma(w[j][H + c], win[j + H + c], acc2[j]);
                }
#pragma unroll
            for (int j = 0; j < J; ++j) x[j] = acc[j] + acc2[j];
        } else if (MODE == 2 || MODE == 3 || MODE == 4) {   // S partial chains per node (3, 1, 4), tap-major
            constexpr int S = MODE == 2 ? 3 : (MODE == 3 ? 1 : 4);
            constexpr int L = (NS + S - 1) / S;
            double a[J][S];
#pragma unroll
            for (int j = 0; j < J; ++j)
#pragma unroll
                for (int q = 0; q < S; ++q) a[j][q] = 0.0;
#pragma unroll
            for (int c = 0; c < L; ++c)
#pragma unroll
                for (int q = 0; q < S; ++q)
#pragma unroll
                    for (int j = 0; j < J; ++j)
                        if (q * L + c < NS) a[j][q] = fma(w[j][q * L + c], win[j + q * L + c], a[j][q]);
#pragma unroll
            for (int j = 0; j < J; ++j) {
                double t = a[j][0];
#pragma unroll
                for (int q = 1; q < S; ++q) t += a[j][q];
                x[j] = t;
            }
        } else if (MODE == 1) {    // window-major: each window value feeds all its nodes back to back
#pragma unroll
            for (int j = 0; j < J; ++j) acc[j] = 0.0;
#pragma unroll
            for (int i = 0; i < W; ++i)
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const int c = i - j;
                    if (c >= 0 && c < NS) acc[j] = fma(w[j][c], win[i], acc[j]);
                }
#pragma unroll
            for (int j = 0; j < J; ++j) x[j] = acc[j];
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < J; ++j) s += x[j];
    out[blockIdx.x * 256 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// pair-split layout: two threads share 6 nodes, each holds half of every node's taps
// (39 weights), computes 39 products, trades its 6 partial sums with one shuffle each and
// adds: 16 warps per SM at <= 128 registers
__global__ void __launch_bounds__(512, 1) pat_pair(const double *wsrc, double *out, int iters, long long *cyc)
{
    constexpr int J = 6;
    double w[39], x[J], h[6];
    for (int c = 0; c < 39; ++c) w[c] = wsrc[(c * 256 + (threadIdx.x >> 1)) % (78 * 256)];
    for (int j = 0; j < J; ++j) x[j] = 1.0 + 1e-3 * j + 1e-6 * threadIdx.x;
    const bool odd = threadIdx.x & 1;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 6; ++m) h[m] = x[m] * (odd ? 0.25 : 0.5);
        double win[12];
#pragma unroll
        for (int m = 0; m < 6; ++m) { win[m] = odd ? x[m] : h[m]; win[6 + m] = odd ? h[m] : x[m]; }
        double acc[J];
        // nodes 0..2 take 7 taps, nodes 3..5 take 6 (39 products); window slot j + c (c < 7)
        int k = 0;
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = 0.0;
#pragma unroll
        for (int c = 0; c < 7; ++c)
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (c < 6 || j < 3) { acc[j] = fma(w[k], win[(j + c) % 12], acc[j]); ++k; }
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = acc[j] + __shfl_xor_sync(0xffffffffu, acc[j], 1);
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < J; ++j) s += x[j];
    out[blockIdx.x * 512 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    double *w, *o; long long *c;
    cudaMalloc(&w, 78 * 256 * 8); cudaMalloc(&o, 148 * 512 * 8); cudaMalloc(&c, 148 * 8);
    double *h = new double[78 * 256];
    for (int i = 0; i < 78 * 256; ++i) h[i] = 0.05 + 1e-4 * (i % 97);
    cudaMemcpy(w, h, 78 * 256 * 8, cudaMemcpyHostToDevice);
    const int iters = 2000;
    long long hc[148];
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) pat<0><<<148, 256>>>(w, o, iters, c);
            else if (mode == 1) pat<1><<<148, 256>>>(w, o, iters, c);
            else if (mode == 2) pat<2><<<148, 256>>>(w, o, iters, c);
            else if (mode == 3) pat<3><<<148, 256>>>(w, o, iters, c);
            else pat<4><<<148, 256>>>(w, o, iters, c);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(hc, c, 148 * 8, cudaMemcpyDeviceToHost);
        printf("mode %d (0: 2 chains/node, 1: window-major 1 chain, 2: 3 chains, 3: 1 chain tap-major, 4: 4 chains): %.1f clk per step (8 warps/SM; FP64 floor ~336) err=%s\n", mode,
               (double)hc[0] / iters, cudaGetErrorString(cudaGetLastError()));
    }
    for (int rep = 0; rep < 2; ++rep) { pat_pair<<<148, 512>>>(w, o, iters, c); cudaDeviceSynchronize(); }
    cudaMemcpy(hc, c, 148 * 8, cudaMemcpyDeviceToHost);
    printf("pair-split: %.1f clk per step (16 warps/SM, 39 DFMA + 6 DMUL + 6 DADD + 6 SHFL.64 per thread) err=%s\n",
           (double)hc[0] / iters, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
