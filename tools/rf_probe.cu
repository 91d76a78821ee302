// probe: is a DFMA with three fresh register-pair operands register-file bound?
#include <cstdio>
#include <cuda_runtime.h>
#define FMA(acc, w, x) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(w), "d"(x))
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const double *wsrc, double *out, int iters, long long *cyc)
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
        double acc[J];
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = 0.0;
        if (MODE == 0) {            // window-major, pinned by volatile asm
#pragma unroll
            for (int i = 0; i < W; ++i)
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const int c = i - j;
                    if (c >= 0 && c < NS) FMA(acc[j], w[j][c], win[i]);
                }
        } else if (MODE == 1) {     // tap-major, pinned
#pragma unroll
            for (int c = 0; c < NS; ++c)
#pragma unroll
                for (int j = 0; j < J; ++j) FMA(acc[j], w[j][c], win[j + c]);
        } else {                    // NOT the stencil: one shared value per tap (reuse in tap-major order)
#pragma unroll
            for (int c = 0; c < NS; ++c)
#pragma unroll
                for (int j = 0; j < J; ++j) FMA(acc[j], w[j][c], win[c]);
        }
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = acc[j];
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < J; ++j) s += x[j];
    out[blockIdx.x * 256 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main()
{
    double *w, *o; long long *c;
    cudaMalloc(&w, 78 * 256 * 8); cudaMalloc(&o, 148 * 256 * 8); cudaMalloc(&c, 148 * 8);
    double *h = new double[78 * 256];
    for (int i = 0; i < 78 * 256; ++i) h[i] = 0.05 + 1e-4 * (i % 97);
    cudaMemcpy(w, h, 78 * 256 * 8, cudaMemcpyHostToDevice);
    const int iters = 2000;
    long long hc[148];
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148, 256>>>(w, o, iters, c); else if (mode == 1) k<1><<<148, 256>>>(w, o, iters, c); else k<2><<<148, 256>>>(w, o, iters, c);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(hc, c, 148 * 8, cudaMemcpyDeviceToHost);
        printf("mode %d (0 window-major, 1 tap-major, 2 shared value per tap; volatile asm): %.1f clk per step (78 DFMA x 2 warps/scheduler; issue floor 312)\n", mode, (double)hc[0] / iters);
    }
    return 0;
}
