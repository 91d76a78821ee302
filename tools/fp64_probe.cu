// fp64_probe.cu -- DFMA latency / throughput probe: FMA per clock per SM for
// C independent chains per thread and W warps per SM (one CTA of 32*W threads
// per SM).  Tells how many independent DFMA chains an SM sub-partition needs
// to saturate the FP64 pipe.  Not part of the product library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void probe(double *out, int iters, double a, double b, long long *cyc)
{
    double x[C];
#pragma unroll
    for (int i = 0; i < C; ++i) x[i] = threadIdx.x * 1e-9 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// exact-mode tap chain: acc = acc + w*x (separate DMUL / DADD, the reference order)
template <int C>
__global__ void probe_exact(double *out, int iters, double a, double b, long long *cyc)
{
    double x[C];
#pragma unroll
    for (int i = 0; i < C; ++i) x[i] = threadIdx.x * 1e-9 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) x[i] = __dadd_rn(x[i], __dmul_rn(a, b + i));
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += x[i];
    if (s == 123.456) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// barrier round trip: iters x __syncthreads() with a shared-memory store / load
__global__ void probe_bar(double *out, int iters, long long *cyc)
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

template <int C>
void run_exact(int warps, double *out, long long *cyc, int sms)
{
    const int iters = 2048;
    probe_exact<C><<<sms, 32 * warps>>>(out, iters, 0.999999, 1e-7, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("{\"exact_chains\": %d, \"warps_per_sm\": %d, \"mul_add_pairs_per_clk_per_sm\": %.2f, \"clk_per_dep_pair\": %.2f}\n",
           C, warps, (double)C * iters * 32 * warps / avg, avg / iters);
}

void run_bar(int warps, double *out, long long *cyc, int sms)
{
    const int iters = 4096;
    probe_bar<<<sms, 32 * warps>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("{\"barrier_warps\": %d, \"clk_per_sts_bar_lds\": %.2f}\n", warps, avg / iters);
}

template <int C>
void run(int warps, double *out, long long *cyc, int sms)
{
    const int iters = 2048;
    probe<C><<<sms, 32 * warps>>>(out, iters, 0.999999, 1e-7, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    const double fma_per_clk = (double)C * iters * 32 * warps / avg;
    printf("{\"chains\": %d, \"warps_per_sm\": %d, \"fma_per_clk_per_sm\": %.2f, \"clk_per_dep_fma\": %.2f}\n",
           C, warps, fma_per_clk, avg / iters);
}

int main()
{
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * 1024);
    for (int w : {4, 8, 16, 32}) {
        run_exact<1>(w, out, cyc, sms);
        run_exact<4>(w, out, cyc, sms);
        run_exact<8>(w, out, cyc, sms);
        run_bar(w, out, cyc, sms);
        run<1>(w, out, cyc, sms);
        run<2>(w, out, cyc, sms);
        run<4>(w, out, cyc, sms);
        run<6>(w, out, cyc, sms);
        run<8>(w, out, cyc, sms);
        run<12>(w, out, cyc, sms);
    }
    return 0;
}
