// rows.cu -- small device kernels around the harvest / step banks: ordered
// row combinations (harvest.combine), per-item status reduction, and the
// classification of reference-style (N, n) weight arrays into compact rows.
// They keep that glue on the library's own kernels instead of framework ops.
#include "common.cuh"

namespace lmep {

__global__ void status_or_kernel(const int32_t *__restrict__ st, int64_t B, int32_t *flag)
{
    bool bad = false;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    // 16-byte loads over the aligned body, scalar loads over what is left
    const int64_t head = min(B, (int64_t)((16 - ((uintptr_t)st & 15)) & 15) / 4);
    const int64_t nv = (B - head) / 4;
    const int4 *v = reinterpret_cast<const int4 *>(st + head);
    for (int64_t i = tid; i < nv; i += nth) {
        const int4 q = v[i];
        bad |= (q.x | q.y | q.z | q.w) != LMEP_OK;
    }
    for (int64_t i = tid; i < head; i += nth) bad |= st[i] != LMEP_OK;
    for (int64_t i = head + 4 * nv + tid; i < B; i += nth) bad |= st[i] != LMEP_OK;
    if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

__global__ void status_merge_kernel(int32_t *__restrict__ dst, const int32_t *__restrict__ src,
                                    int64_t B)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B;
         i += (int64_t)gridDim.x * blockDim.x)
        if (dst[i] == LMEP_OK) dst[i] = src[i];
}

static unsigned grid_for(int64_t work, int threads)
{
    const int64_t cap = (int64_t)device_sm_count() * 8;
    const int64_t g = (work + threads - 1) / threads;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

int launch_status_or(const int32_t *status, int64_t B, int32_t *flag, cudaStream_t st)
{
    if (B <= 0) return LMEP_OK;
    status_or_kernel<<<grid_for(B, 256), 256, 0, st>>>(status, B, flag);
    return launch_status("status_or_kernel");
}

int launch_status_merge(int32_t *dst, const int32_t *src, int64_t B, cudaStream_t st)
{
    if (B <= 0) return LMEP_OK;
    status_merge_kernel<<<grid_for(B, 256), 256, 0, st>>>(dst, src, B);
    return launch_status("status_merge_kernel");
}

constexpr int kCombineMax = 8;

struct CombineArgs {
    const double *in[kCombineMax];
    int64_t ld[kCombineMax];
    double c[kCombineMax];
    int nterm;
    int64_t rows, cols, ld_out;
    double *out;
};

// out = (((0 + c0 x0) + c1 x1) + ...): numpy's `acc = acc + c * a` from zeros
// (harvest.py:225-235), two roundings per term, list order
__global__ void combine_kernel(const __grid_constant__ CombineArgs a)
{
    const int64_t total = a.rows * a.cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / a.cols, j = e - r * a.cols;
        double acc = 0.0;
        for (int t = 0; t < a.nterm; ++t) acc = xadd(acc, xmul(a.c[t], a.in[t][r * a.ld[t] + j]));
        a.out[r * a.ld_out + j] = acc;
    }
}

// per-row comparison of an (N, n) weight array with row `ref`: the first and
// last equal rows and their count (compact-row classification, _ops.compress)
__global__ void classify_kernel(const double *__restrict__ w, int64_t N, int n, int64_t ref,
                                unsigned long long *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool eq = true;
        for (int j = 0; j < n; ++j) eq &= w[i * n + j] == w[ref * n + j];
        if (eq) {
            atomicMin(out + 0, (unsigned long long)i);
            atomicMax(out + 1, (unsigned long long)i);
            atomicAdd(out + 2, 1ull);
        }
    }
}

__global__ void classify_init(unsigned long long *out)
{
    out[0] = ~0ull;
    out[1] = 0ull;
    out[2] = 0ull;
}

}  // namespace lmep

using namespace lmep;

extern "C" int lmep_combine(int nterm, const double *const *in, const int64_t *ld_in,
                            const double *coef, int64_t rows, int64_t cols, double *out,
                            int64_t ld_out, void *stream)
{
    if (nterm < 1 || nterm > kCombineMax || !in || !ld_in || !coef || !out) return LMEP_INVALID_CONFIG;
    if (rows < 0 || cols < 0 || ld_out < cols) return LMEP_DIMENSION;
    if (rows == 0 || cols == 0) return LMEP_OK;
    CombineArgs a{};
    for (int t = 0; t < nterm; ++t) {
        if (!in[t] || (rows > 1 && ld_in[t] < cols)) return LMEP_INVALID_CONFIG;
        a.in[t] = in[t];
        a.ld[t] = ld_in[t];
        a.c[t] = coef[t];
    }
    a.nterm = nterm;
    a.rows = rows;
    a.cols = cols;
    a.ld_out = ld_out;
    a.out = out;
    combine_kernel<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(a);
    return launch_status("combine_kernel");
}

extern "C" int lmep_status_any(const int32_t *status, int64_t B, int32_t *flag, void *stream)
{
    if (B < 0 || !flag || (B > 0 && !status)) return LMEP_INVALID_CONFIG;
    return launch_status_or(status, B, flag, (cudaStream_t)stream);
}

extern "C" int lmep_rows_classify(const double *rows, int64_t N, int n, int64_t ref,
                                  uint64_t *out3, void *stream)
{
    if (!rows || !out3 || N < 1 || n < 1 || ref < 0 || ref >= N) return LMEP_INVALID_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    auto *o = reinterpret_cast<unsigned long long *>(out3);
    classify_init<<<1, 1, 0, st>>>(o);
    classify_kernel<<<grid_for(N, 256), 256, 0, st>>>(rows, N, n, ref, o);
    return launch_status("classify_kernel");
}

namespace lmep {

struct FootArgs {
    double w[LMEP_MAX_N];
    double oh[LMEP_MAX_N];
    int n, num_k;
    double kstep, kmax, shift;
    double *gre, *gim, *gabs, *disp;
};

// symbol of one weight row (analysis.py:42-64): one thread per wavenumber,
// k_i = i * kstep (the last one exactly pi / h, like numpy.linspace)
__global__ void footprint_kernel(const __grid_constant__ FootArgs a)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.num_k) return;
    const double k = (i == a.num_k - 1 && a.num_k > 1) ? a.kmax : (double)i * a.kstep;
    double re = 0.0, im = 0.0;
    for (int j = 0; j < a.n; ++j) {
        double s, c;
        sincos(k * a.oh[j], &s, &c);
        re = fma(a.w[j], c, re);
        im = fma(a.w[j], s, im);
    }
    double ss, cs;
    sincos(k * a.shift, &ss, &cs);
    a.gre[i] = re;
    a.gim[i] = im;
    a.gabs[i] = hypot(re, im);
    a.disp[i] = atan2(re * ss + im * cs, re * cs - im * ss);
}

}  // namespace lmep

extern "C" int lmep_spectral_footprint(const double *w, const double *offsets_h, int n, double kmax,
                                       int num_k, double shift, double *g_re, double *g_im,
                                       double *g_abs, double *dispersion, void *stream)
{
    if (!w || !offsets_h || n < 1 || n > LMEP_MAX_N || num_k < 1) return LMEP_INVALID_CONFIG;
    if (!g_re || !g_im || !g_abs || !dispersion) return LMEP_INVALID_CONFIG;
    FootArgs a{};
    for (int j = 0; j < n; ++j) {
        a.w[j] = w[j];
        a.oh[j] = offsets_h[j];
    }
    a.n = n;
    a.num_k = num_k;
    a.kmax = kmax;
    a.kstep = num_k > 1 ? kmax / (double)(num_k - 1) : 0.0;
    a.shift = shift;
    a.gre = g_re;
    a.gim = g_im;
    a.gabs = g_abs;
    a.disp = dispersion;
    footprint_kernel<<<(unsigned)((num_k + 127) / 128), 128, 0, (cudaStream_t)stream>>>(a);
    return launch_status("footprint_kernel");
}
