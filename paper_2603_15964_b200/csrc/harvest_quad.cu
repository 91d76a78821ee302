// harvest_quad.cu -- K1 for d <= 16: register-resident expm-multiply harvest.
//
// The harvest needs only a few columns of exp(A) (A = the transposed reduced
// augmentation, harvest.cu): column `row` gives w_lin and columns n..n+s-2 give
// the raw dt^j phi_j rows (harvest.py:119-120).  Instead of forming exp(A)
// (Pade: ~5 d x d products + an LU solve, harvest.cu), each needed column is
// computed as the action exp(A) e_c -- the expm-multiply approach of Al-Mohy &
// Higham (2011, the algorithm behind scipy.sparse.linalg.expm_multiply):
//
//   1. balance A -> B = D^-1 A D (exact powers of two, as expm.py:37 does),
//   2. s = ceil(log2 ||B||_1) so that ||B / 2^s||_1 <= 1,
//   3. x <- T(B/2^s) x applied 2^s times, T the Taylor series truncated when
//      two consecutive terms fall below 2^-53 of the partial sum,
//   4. exp(A) e_c = 2^-e_c D exp(B) e_c.
//
// Mapping: 4 lanes ("quad") own one item; lane q holds rows q, q+4, q+8, q+12
// of B in registers (no shared memory).  A matrix-vector product is R*D FMAs
// per lane plus D quad shuffles to replicate the new vector, so a warp works
// on 8 items at once with the FP64 pipe, not shared memory, as the limiter.
#include <math.h>

#include "harvest.cuh"

namespace lmep {

__constant__ double kInvK[48] = {
    0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9, 1.0 / 10,
    1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19,
    1.0 / 20, 1.0 / 21, 1.0 / 22, 1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28,
    1.0 / 29, 1.0 / 30, 1.0 / 31, 1.0 / 32, 1.0 / 33, 1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37,
    1.0 / 38, 1.0 / 39, 1.0 / 40, 1.0 / 41, 1.0 / 42, 1.0 / 43, 1.0 / 44, 1.0 / 45, 1.0 / 46,
    1.0 / 47};
constexpr int TAYLOR_MAX = 47;
#ifndef HARVEST_THETA
#define HARVEST_THETA 2.0
#endif

__device__ __forceinline__ int q_exp2i(double x) { return ((__double2hiint(x) >> 20) & 0x7ff) - 1023; }
__device__ __forceinline__ double q_pow2(int k) { return __hiloint2double((k + 1023) << 20, 0); }
template <int LPI>
__device__ __forceinline__ double q_sum(double v, unsigned m)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v += __shfl_xor_sync(m, v, o);
    return v;
}
template <int LPI>
__device__ __forceinline__ double q_max(double v, unsigned m)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v = fmax(v, __shfl_xor_sync(m, v, o));
    return v;
}

template <int D, int LPI>
__global__ void __launch_bounds__(128) harvest_quad_kernel(const HarvestParams P)
{
    constexpr int R = (D + LPI - 1) / LPI;    // rows per lane
    constexpr int SH = LPI == 4 ? 2 : 3;
    const int lane = threadIdx.x & 31;
    const int q = lane & (LPI - 1), qb = lane & ~(LPI - 1);
    const unsigned qm = ((1u << LPI) - 1u) << qb;
    const int64_t braw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> SH;
    const bool live = braw < P.B;
    const int64_t b = live ? braw : P.B - 1;   // idle quads mirror the last item, never store
    const int n = P.n, sd = P.s;
    const int row = P.rows ? P.rows[b] : P.row_default;
    const uint64_t fz = P.frozen ? P.frozen[b] : P.frozen_default;
    const double dt = P.delta_t;

    // ---- own rows of A = [[dt L'^T, dt e_row, 0], [0, 0, dt J]] -------------
    // A table shared by every item (table_idx == null) is staged once per CTA
    // in shared memory; per-item coefficients go to registers.
    extern __shared__ double stab[];
    const double *tab = nullptr;
    double cfr[4] = {0.0, 0.0, 0.0, 0.0};
    double cz = 0.0;
    const bool shared_tab = P.mode == 1 && P.table_idx == nullptr;
    if (shared_tab) {
        const int tn = P.nterms * n * n;
        for (int i = threadIdx.x; i < tn; i += blockDim.x) stab[i] = P.tables[i];
        __syncthreads();
        tab = stab;
    }
    if (P.mode == 1) {
        if (!shared_tab) tab = P.tables + (size_t)P.table_idx[b] * P.nterms * n * n;
        const double *cf = P.coef + b * P.coef_stride;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (t < P.nterms) cfr[t] = cf[t];
        cz = P.c0 ? P.c0[b * P.c0_stride] : 0.0;
    }
    double a[R][D];
    bool fin = true;
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int j = q + LPI * m;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double v = 0.0;
            if (j < D) {
                if (j < n && c < n) {
                    double l;
                    if (P.mode == 1 && P.map_on) {
                        // row-scaled: local row c takes node m_c's coefficients
                        const int64_t mc = coef_node(P, b, row, c);
                        const double *cfc = P.coef + mc * P.coef_stride;
                        l = 0.0;
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            if (t < P.nterms) l = xadd(l, xmul(cfc[t], tab[(t * n + c) * n + j]));
                        const double czc = P.c0 ? P.c0[mc * P.c0_stride] : 0.0;
                        if (c == j && czc != 0.0) l = xadd(l, czc);
                    } else if (P.mode == 1) {
                        // localop.py:120-127: term order, then the reaction on the diagonal
                        l = 0.0;
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            if (t < P.nterms) l = xadd(l, xmul(cfr[t], tab[(t * n + c) * n + j]));
                        if (c == j && cz != 0.0) l = xadd(l, cz);
                    } else {
                        l = P.L[(b * n + c) * n + j];
                    }
                    if ((fz >> c) & 1ull) l = 0.0;                      // harvest.py:116-117
                    v = xmul(dt, l);
                } else if (c == n && j == row) {
                    v = dt;
                } else if (j >= n && c == j + 1) {
                    v = dt;
                }
            }
            fin &= (bool)isfinite(v);
            a[m][c] = v;
        }
    }
    int status = __all_sync(qm, fin) ? LMEP_OK : LMEP_NONFINITE;

    // ---- balancing: Osborne sweeps in parallel (see harvest.cu balance) --------
    int e[R];
#pragma unroll
    for (int m = 0; m < R; ++m) e[m] = 0;
    for (int sweep = 0; sweep < 12 && status == LMEP_OK; ++sweep) {
        double myc2[R];
#pragma unroll
        for (int m = 0; m < R; ++m) myc2[m] = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double p = 0.0;
#pragma unroll
            for (int m = 0; m < R; ++m) p = fma(a[m][c], a[m][c], p);
            p = q_sum<LPI>(p, qm);
            if ((c & (LPI - 1)) == q) myc2[c >> SH] = p;
        }
        int k[R];
        bool chg = false;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            k[m] = 0;
            double r2 = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) r2 = fma(a[m][c], a[m][c], r2);
            const double c2 = myc2[m];
            if (q + LPI * m < D && c2 > 1e-280 && r2 > 1e-280 && c2 < 1e280 && r2 < 1e280) {
                const double cn = sqrt(c2), rn = sqrt(r2);
                int kk = (q_exp2i(rn) - q_exp2i(cn)) / 2;
                while (cn * q_pow2(2 * kk + 1) < rn) ++kk;
                while (kk > 0 && !(cn * q_pow2(2 * kk - 1) < rn)) --kk;
                if (kk <= 0) {
                    kk = 0;
                    while (cn * q_pow2(-(2 * (-kk) + 1)) >= rn) --kk;
                }
                const double f = q_pow2(kk);
                if (kk != 0 && cn * f + rn / f < 0.95 * (cn + rn)) k[m] = kk;
            }
            chg |= k[m] != 0;
        }
        if (!__any_sync(qm, chg)) break;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const int kc = __shfl_sync(qm, k[c >> SH], qb + (c & (LPI - 1)));
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (kc != k[m]) a[m][c] *= q_pow2(kc - k[m]);
        }
#pragma unroll
        for (int m = 0; m < R; ++m) e[m] += k[m];
    }

    // ---- scaling: ||B / reps||_1 <= THETA ---------------------------------------
    double nrm = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
        double p = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) p += fabs(a[m][c]);
        nrm = fmax(nrm, q_sum<LPI>(p, qm));
    }
    // THETA = 2: Taylor terms of a norm-2 step peak at 2 (loss < 4 bits
    // against the decay of the exponential) and fewer steps beat shorter series
    constexpr double THETA = HARVEST_THETA;
    int s = 0;                                  // number of steps `reps`
    if (!(nrm <= 1e9)) status = LMEP_NONFINITE; // also NaN: not a stencil operator
    else s = nrm > THETA ? (int)ceil(nrm / THETA) : 1;
    if (s > 1) {
        const double sc = 1.0 / (double)s;
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int c = 0; c < D; ++c) a[m][c] *= sc;
    }

    // ---- exp(A) e_idx for every wanted column -----------------------------------
    int nmv = 0;
    const int reps = status == LMEP_OK ? s : 0;
    for (int qo = 0; qo < sd; ++qo) {
        const int idx = qo == 0 ? row : n + qo - 1;
        double t[D], acc[R];
#pragma unroll
        for (int c = 0; c < D; ++c) t[c] = (c == idx) ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) acc[m] = (q + LPI * m == idx) ? 1.0 : 0.0;
        for (int rep = 0; rep < reps; ++rep) {
            double wprev = INFINITY;
            for (int kt = 1; kt <= TAYLOR_MAX; ++kt) {
                double w[R];
                double wn = 0.0, an = 0.0;
                const double ik = kInvK[kt];
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int c = 0; c < D; c += 2) {
                        s0 = fma(a[m][c], t[c], s0);
                        if (c + 1 < D) s1 = fma(a[m][c + 1], t[c + 1], s1);
                    }
                    w[m] = (s0 + s1) * ik;
                    acc[m] += w[m];
                    // convergence is judged on the extracted rows only: the
                    // augmentation chain (rows >= n) is O(1) while dt^j phi_j is tiny
                    if (q + LPI * m < n) {
                        wn = fmax(wn, fabs(w[m]));
                        an = fmax(an, fabs(acc[m]));
                    }
                }
                ++nmv;
                wn = q_max<LPI>(wn, qm);
                an = q_max<LPI>(an, qm);
#pragma unroll
                for (int c = 0; c < D; ++c) t[c] = __shfl_sync(qm, w[c >> SH], qb + (c & (LPI - 1)));
                // the chain needs qo products to reach the extracted rows
                if (kt > qo && an > 0.0 && wn + wprev <= 0x1p-53 * an) break;
                wprev = wn;
            }
#pragma unroll
            for (int c = 0; c < D; ++c) t[c] = __shfl_sync(qm, acc[c >> SH], qb + (c & (LPI - 1)));
        }
        // back to A's coordinates: exp(A) e_idx = 2^-e_idx D exp(B) e_idx
        int eo = 0;
#pragma unroll
        for (int m = 0; m < R; ++m)
            if ((idx >> SH) == m) eo = e[m];
        const int eidx = __shfl_sync(qm, eo, qb + (idx & (LPI - 1)));
        bool okv = true;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int j = q + LPI * m;
            double w = acc[m] * q_pow2(e[m] - eidx);
            okv &= (bool)isfinite(w);
            if (qo > 0 && ((fz >> j) & 1ull)) w = 0.0;
            if (live && j < n) {
                if (P.layout == 0) P.out[(b * sd + qo) * n + j] = w;
                else P.out[((int64_t)qo * n + j) * P.out_ld + b] = w;
            }
        }
        if (!__all_sync(qm, okv)) status = LMEP_NONFINITE;
    }
    if (live && q == 0) {
        if (P.status) P.status[b] = status;
        if (P.ms) P.ms[b] = nmv | (min(s, 255) << 24);
    }
}

static int g_lanes_per_item = 8;     // d > 8: 8 lanes per item (lower registers, 2x warps)

template <int D>
static int launch_quad(const HarvestParams &P, cudaStream_t st)
{
    const int lpi = (D > 8 && g_lanes_per_item == 8) ? 8 : 4;
    const int64_t threads = P.B * lpi;
    const int64_t blocks = (threads + 127) / 128;
    if (blocks > 0x7fffffffLL) return LMEP_INVALID_CONFIG;
    const size_t shm = (P.mode == 1 && P.table_idx == nullptr) ? (size_t)P.nterms * P.n * P.n * 8 : 0;
    if (lpi == 8) harvest_quad_kernel<D, 8><<<(unsigned)blocks, 128, shm, st>>>(P);
    else harvest_quad_kernel<D, 4><<<(unsigned)blocks, 128, shm, st>>>(P);
    return launch_status("harvest_quad_kernel");
}

void set_lanes_per_item(int lpi) { g_lanes_per_item = lpi; }

int launch_harvest_quad(const HarvestParams &P, cudaStream_t st)
{
    if (P.mode == 1 && P.nterms > 4) return LMEP_INVALID_CONFIG;   // caller falls back to Pade
    switch (P.d) {
    case 2: return launch_quad<2>(P, st);
    case 3: return launch_quad<3>(P, st);
    case 4: return launch_quad<4>(P, st);
    case 5: return launch_quad<5>(P, st);
    case 6: return launch_quad<6>(P, st);
    case 7: return launch_quad<7>(P, st);
    case 8: return launch_quad<8>(P, st);
    case 9: return launch_quad<9>(P, st);
    case 10: return launch_quad<10>(P, st);
    case 11: return launch_quad<11>(P, st);
    case 12: return launch_quad<12>(P, st);
    case 13: return launch_quad<13>(P, st);
    case 14: return launch_quad<14>(P, st);
    case 15: return launch_quad<15>(P, st);
    case 16: return launch_quad<16>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
