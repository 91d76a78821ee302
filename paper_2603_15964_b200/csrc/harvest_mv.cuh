// harvest_mv.cuh -- K1 for d <= 16: warp-uniform expm-multiply harvest.
//
// Same mathematics as harvest_quad.cu: each wanted column of exp(A) (A the
// transposed reduced augmentation, harvest.cu) is computed as the action
// exp(A) e_c after power-of-two balancing, with A/reps stepped reps times by
// a Taylor series truncated when two consecutive terms fall below 2^-53 of
// the partial sum (Al-Mohy & Higham 2011; harvest.py:97-121 semantics).
//
// What changes is the mapping to the SM, driven by the ncu profile of the
// quad kernel (profiles/r1_harvest_quad_kernel.md: 9% of the instructions
// were DFMA, 32% were spent assembling A through generic loads, and each
// Taylor term paid 38 shuffles plus divergence checks for 26 DFMAs):
//
//   * LPI lanes own one item (rows q, q+LPI, ... of A in registers); a warp
//     holds G = 32/LPI items.  The Taylor iteration is flattened into one
//     warp-uniform loop: every group carries its own (column, rep, term)
//     state and the loop runs until all groups of the warp are done, so
//     every shuffle and vote uses the full mask (no MATCH/REDUX divergence
//     handling) and neighbouring nodes -- similar operators -- share trips.
//   * the Taylor iterate is replicated through shared memory instead of
//     shuffles: R stores plus D/2 conflict-free LDS.128 per term (group
//     vectors are padded so the G groups of a warp hit disjoint banks),
//     double buffered so one __syncwarp per term orders them.
//   * the convergence test reduces the high words of |w| and |acc| (upper and
//     lower bounds of the doubles) with 32-bit shuffles.
//   * with a CTA-shared derivative table (periodic grids: one window
//     geometry) A is assembled from a transposed, zero-padded shared copy of
//     the table with compile-time offsets (LDS only, NT terms unrolled).
#pragma once
#include <math.h>

#include "harvest.cuh"

namespace lmep {

constexpr unsigned MV_FULL = 0xffffffffu;
constexpr int MV_TMAX = 47;

__device__ __forceinline__ int mv_exp2i(double x) { return ((__double2hiint(x) >> 20) & 0x7ff) - 1023; }
__device__ __forceinline__ double mv_pow2(int k) { return __hiloint2double((k + 1023) << 20, 0); }
__device__ __forceinline__ unsigned mv_hiabs(double x) { return (unsigned)__double2hiint(x) & 0x7fffffffu; }

template <int LPI>
__device__ __forceinline__ double mv_gsum(double v)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v += __shfl_xor_sync(MV_FULL, v, o);
    return v;
}
template <int LPI>
__device__ __forceinline__ unsigned mv_gmax(unsigned v)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v = max(v, __shfl_xor_sync(MV_FULL, v, o));
    return v;
}
template <int LPI>
__device__ __forceinline__ unsigned mv_gor(unsigned v)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v |= __shfl_xor_sync(MV_FULL, v, o);
    return v;
}
template <int LPI>
__device__ __forceinline__ double mv_gfmax(double v)
{
#pragma unroll
    for (int o = 1; o < LPI; o <<= 1) v = fmax(v, __shfl_xor_sync(MV_FULL, v, o));
    return v;
}

template <int D, int LPI>
struct MvCfg {
    static constexpr int R = (D + LPI - 1) / LPI;       // rows per lane
    static constexpr int SH = LPI == 2 ? 1 : (LPI == 4 ? 2 : 3);
    static constexpr int G = 32 / LPI;                  // items per warp
    static constexpr int TS = (LPI == 8 || D > 8) ? 18 : 10;   // doubles per item vector (bank-spread pad)
    static constexpr int BUF = G * TS;                  // one buffer of a warp
    static constexpr int WARP_T = 2 * BUF;              // double buffered
    static constexpr int THREADS = 128;
    static constexpr int INV = 48;                      // 1/k! table
    static constexpr int EXPW = (THREADS / LPI) * 16 / 2;   // per-group balancing exponents (int)
    static_assert(TS >= D + (D & 1), "item vector too short");
};

template <int D, int LPI>
constexpr size_t mv_smem_bytes(int nt)
{
    using C = MvCfg<D, LPI>;
    return (size_t)(C::INV + C::EXPW + (C::THREADS / 32) * C::WARP_T + nt * D * D) * sizeof(double);
}

// A's rows owned by this lane from a CTA-shared table sT[t][j][c] = D_t[c][j]
// (zero outside n x n): a[m][c] = dt * L'[c][j], L' = L with frozen rows zeroed.
template <int D, int LPI, int NT>
__device__ __forceinline__ void mv_build_shared(double (&a)[MvCfg<D, LPI>::R][D],
                                                const double *sTab, const double (&cf)[NT],
                                                double cz, uint64_t fz, double dt, int n, int row,
                                                int q)
{
    constexpr int R = MvCfg<D, LPI>::R;
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int j = q + LPI * m;
        const int jj = j < D ? j : 0;
        const double *tr = sTab + jj * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            // localop.py:120-127: term order, then the reaction on the diagonal
            double l = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) l = xadd(l, xmul(cf[t], tr[t * D * D + c]));
            if (c == j && c < n && cz != 0.0) l = xadd(l, cz);
            if ((fz >> c) & 1ull) l = 0.0;                               // harvest.py:116-117
            double v = (j < n && c < n) ? xmul(dt, l) : 0.0;
            if (c == n && j == row) v = dt;
            else if (j >= n && c == j + 1) v = dt;
            a[m][c] = j < D ? v : 0.0;
        }
    }
}

// Generic assembly: per-item tables (table_idx), row-scaled coefficients
// (coef map) or explicit L (mode 2).
template <int D, int LPI>
__device__ __forceinline__ void mv_build_generic(double (&a)[MvCfg<D, LPI>::R][D],
                                                 const HarvestParams &P, int64_t b, uint64_t fz,
                                                 int row, int q)
{
    constexpr int R = MvCfg<D, LPI>::R;
    const int n = P.n;
    const double dt = P.delta_t;
    const double *tab = nullptr, *cf = nullptr;
    double cz = 0.0;
    if (P.mode == 1) {
        tab = P.tables + (size_t)(P.table_idx ? P.table_idx[b] : 0) * P.nterms * n * n;
        cf = P.coef + b * P.coef_stride;
        cz = P.c0 ? P.c0[b * P.c0_stride] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int j = q + LPI * m;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double v = 0.0;
            if (j < n && c < n) {
                double l;
                if (P.mode == 1) {
                    const double *cfc = cf;
                    double czc = cz;
                    if (P.map_on) {              // row-scaled: L row c reads node m_c
                        const int64_t mc = coef_node(P, b, row, c);
                        cfc = P.coef + mc * P.coef_stride;
                        czc = P.c0 ? P.c0[mc * P.c0_stride] : 0.0;
                    }
                    l = 0.0;
                    for (int t = 0; t < P.nterms; ++t)
                        l = xadd(l, xmul(cfc[t], tab[(t * n + c) * n + j]));
                    if (c == j && czc != 0.0) l = xadd(l, czc);
                } else {
                    l = P.L[(b * n + c) * n + j];
                }
                if ((fz >> c) & 1ull) l = 0.0;
                v = xmul(dt, l);
            } else if (j < D) {
                if (c == n && j == row) v = dt;
                else if (j >= n && c == j + 1) v = dt;
            }
            a[m][c] = v;
        }
    }
}

template <int D, int LPI, int NT>
__global__ void __launch_bounds__(128) harvest_mv_kernel(const HarvestParams P)
{
    using C = MvCfg<D, LPI>;
    constexpr int R = C::R, SH = C::SH;
    extern __shared__ __align__(16) double mv_sm[];
    double *sFact = mv_sm;                                     // 1/k!
    int *sE = reinterpret_cast<int *>(mv_sm + C::INV);        // [group][16] exponents
    double *sT = mv_sm + C::INV + C::EXPW + (threadIdx.x >> 5) * C::WARP_T;
    double *sTab = mv_sm + C::INV + C::EXPW + (C::THREADS / 32) * C::WARP_T;
    const int lane = threadIdx.x & 31;
    const int q = lane & (LPI - 1), qb = lane & ~(LPI - 1), grp = lane >> SH;
    const int n = P.n, sd = P.s;

    for (int i = threadIdx.x; i < C::INV; i += blockDim.x) {
        double f = 1.0;
        for (int j = 2; j <= i; ++j) f *= (double)j;
        sFact[i] = 1.0 / f;
    }
    if (NT > 0) {
        for (int i = threadIdx.x; i < NT * D * D; i += blockDim.x) {
            const int t = i / (D * D), r = i - t * D * D, j = r / D, c = r - j * D;
            sTab[i] = (j < n && c < n) ? P.tables[(t * n + c) * n + j] : 0.0;
        }
    }
    __syncthreads();

    const int64_t braw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> SH;
    const bool live = braw < P.B;
    const int64_t b = live ? braw : P.B - 1;   // idle groups mirror the last item, never store
    const int row = P.rows ? P.rows[b] : P.row_default;
    const uint64_t fz = P.frozen ? P.frozen[b] : P.frozen_default;

    double a[R][D];
    if constexpr (NT > 0) {
        double cf[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) cf[t] = P.coef[b * P.coef_stride + t];
        const double cz = P.c0 ? P.c0[b * P.c0_stride] : 0.0;
        mv_build_shared<D, LPI, NT>(a, sTab, cf, cz, fz, P.delta_t, n, row, q);
    } else {
        mv_build_generic<D, LPI>(a, P, b, fz, row, q);
    }
    unsigned finite = 1u;
#pragma unroll
    for (int m = 0; m < R; ++m)
#pragma unroll
        for (int c = 0; c < D; ++c) finite &= (unsigned)isfinite(a[m][c]);
    int status = (mv_gmax<LPI>(finite ^ 1u) == 0u) ? LMEP_OK : LMEP_NONFINITE;

    // ---- balancing: parallel Osborne sweeps with exact powers of two --------
    // Any power-of-two diagonal similarity leaves exp(A) unchanged up to
    // rounding (expm.py:27-30 balances for the norm and for overflow); the
    // step per row comes straight from the exponents of the squared row and
    // column 2-norms, which avoids the square roots and search loops of
    // dgebal's acceptance test.
    int e[R];
#pragma unroll
    for (int m = 0; m < R; ++m) e[m] = 0;
    for (int sweep = 0; sweep < 12; ++sweep) {
        double myc2[R];
#pragma unroll
        for (int m = 0; m < R; ++m) myc2[m] = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double p = 0.0;
#pragma unroll
            for (int m = 0; m < R; ++m) p = fma(a[m][c], a[m][c], p);
            p = mv_gsum<LPI>(p);
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
            if (status == LMEP_OK && q + LPI * m < D && c2 > 1e-280 && r2 > 1e-280 &&
                c2 < 1e280 && r2 < 1e280) {
                // 2^kk ~ sqrt(rn / cn) minimises cn 2^kk + rn 2^-kk; ex = log2(r2 / c2)
                // to +-1, so |ex| >= 4 (rn / cn >= 2^1.5) guarantees kk = +-1 or
                // more strictly reduces the row + column norm (no oscillation)
                const int ex = mv_exp2i(r2) - mv_exp2i(c2);
                if (ex >= 4) k[m] = (ex + 2) >> 2;
                else if (ex <= -4) k[m] = -((2 - ex) >> 2);
            }
            chg |= k[m] != 0;
        }
        if (!__any_sync(MV_FULL, chg)) break;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const int kc = __shfl_sync(MV_FULL, k[c >> SH], qb + (c & (LPI - 1)));
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (kc != k[m]) a[m][c] *= mv_pow2(kc - k[m]);
        }
#pragma unroll
        for (int m = 0; m < R; ++m) e[m] += k[m];
    }

    // ---- scaling: ||B / reps||_1 <= THETA ------------------------------------
    double nrm = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
        double p = 0.0;
#pragma unroll
        for (int m = 0; m < R; ++m) p += fabs(a[m][c]);
        nrm = fmax(nrm, mv_gsum<LPI>(p));
    }
    constexpr double THETA = 2.0;
    int s = 0;
    if (!(nrm <= 1e9)) status = LMEP_NONFINITE;
    else s = nrm > THETA ? (int)ceil(nrm / THETA) : 1;
    // half-step set: exp(B) = exp(B / reps)^reps, so after reps / 2 of the reps
    // the iterate is exp(B / 2) e_c -- the same columns at delta_t / 2 (the
    // augmentation scales with delta_t: (dt/2)^j phi_j(dt/2 L))
    const bool want_half = P.half_out != nullptr;
    if (want_half && status == LMEP_OK) s = s < 2 ? 2 : s + (s & 1);
    if (s > 1) {
        const double sc = 1.0 / (double)s;
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
            for (int c = 0; c < D; ++c) a[m][c] *= sc;
    }
    const int reps = status == LMEP_OK ? s : 0;

    // ---- flattened Taylor iteration: state (column qo, rep, term kt) per group
    // The iterate is the unscaled power u_k = B^k v (||B|| <= THETA keeps it
    // bounded) and the partial sum takes u_k / k! with one FMA per row.
    int *eg = sE + (threadIdx.x >> SH) * 16;                  // this group's exponents
#pragma unroll
    for (int m = 0; m < R; ++m)
        if (q + LPI * m < D) eg[q + LPI * m] = e[m];
    int qo = 0, rep = 0, kt = 1, nmv = 0, idx = row;
    bool done = reps == 0;
    unsigned bad = 0u;
    double acc[R];
#pragma unroll
    for (int m = 0; m < R; ++m) acc[m] = (q + LPI * m == idx) ? 1.0 : 0.0;
    double wprev = INFINITY;
    double *tg = sT + grp * C::TS;
    int buf = 0;
#pragma unroll
    for (int m = 0; m < R; ++m)
        if (q + LPI * m < D) tg[q + LPI * m] = acc[m];
    __syncwarp();
    while (__any_sync(MV_FULL, !done)) {
        const double *tv = tg + buf * C::BUF;
        double u[R];
        if constexpr (R >= 4) {                  // R independent chains already
#pragma unroll
            for (int m = 0; m < R; ++m) u[m] = 0.0;
#pragma unroll
            for (int c = 0; c < D; c += 2) {
                if (c + 1 < D) {
                    const double2 tt = *reinterpret_cast<const double2 *>(tv + c);
#pragma unroll
                    for (int m = 0; m < R; ++m) u[m] = fma(a[m][c + 1], tt.y, fma(a[m][c], tt.x, u[m]));
                } else {
                    const double t0 = tv[c];
#pragma unroll
                    for (int m = 0; m < R; ++m) u[m] = fma(a[m][c], t0, u[m]);
                }
            }
        } else {
            double s0[R], s1[R];
#pragma unroll
            for (int m = 0; m < R; ++m) s0[m] = s1[m] = 0.0;
#pragma unroll
            for (int c = 0; c < D; c += 2) {
                if (c + 1 < D) {
                    const double2 tt = *reinterpret_cast<const double2 *>(tv + c);
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        s0[m] = fma(a[m][c], tt.x, s0[m]);
                        s1[m] = fma(a[m][c + 1], tt.y, s1[m]);
                    }
                } else {
                    const double t0 = tv[c];
#pragma unroll
                    for (int m = 0; m < R; ++m) s0[m] = fma(a[m][c], t0, s0[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < R; ++m) u[m] = s0[m] + s1[m];
        }
        const double fk = sFact[kt];
        const double fa = done ? 0.0 : fk;
        unsigned wh = 0u, ah = 0u;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            acc[m] = fma(u[m], fa, acc[m]);
            // convergence is judged on the extracted rows only: the augmentation
            // chain (rows >= n) is O(1) while dt^j phi_j is tiny
            if (q + LPI * m < n) {
                wh = max(wh, mv_hiabs(u[m]));
                ah = max(ah, mv_hiabs(acc[m]));
            }
        }
        wh = mv_gmax<LPI>(wh);
        ah = mv_gmax<LPI>(ah);
        const double wn = __hiloint2double((int)wh, -1) * fk;  // >= max |u_k / k!| (to rounding)
        const double an = __hiloint2double((int)ah, 0);         // <= max |acc|
        // the chain needs qo products to reach the extracted rows
        const bool conv = (kt > qo && an > 0.0 && wn + wprev <= 0x1p-53 * an) || kt >= MV_TMAX;
        if (!done) {
            ++nmv;
            double nt[R];
            if (conv) {
                ++rep;
                kt = 1;
                wprev = INFINITY;
                if (want_half && qo < 2 && 2 * rep == reps) {
                    const int eidx = eg[idx];
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        const int j = q + LPI * m;
                        double o = acc[m] * mv_pow2(e[m] - eidx);
                        bad |= (unsigned)!isfinite(o);
                        if (qo > 0 && ((fz >> j) & 1ull)) o = 0.0;
                        if (live && j < n) {
                            if (P.layout == 0) P.half_out[(b * 2 + qo) * n + j] = o;
                            else P.half_out[((int64_t)qo * n + j) * P.out_ld + b] = o;
                        }
                    }
                }
                if (rep >= reps) {
                    // back to A's coordinates: exp(A) e_idx = 2^-e_idx D exp(B) e_idx
                    const int eidx = eg[idx];
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        const int j = q + LPI * m;
                        double o = acc[m] * mv_pow2(e[m] - eidx);
                        bad |= (unsigned)!isfinite(o);
                        if (qo > 0 && ((fz >> j) & 1ull)) o = 0.0;
                        if (live && j < n) {
                            if (P.layout == 0) P.out[(b * sd + qo) * n + j] = o;
                            else P.out[((int64_t)qo * n + j) * P.out_ld + b] = o;
                        }
                    }
                    ++qo;
                    rep = 0;
                    if (qo >= sd) {
                        done = true;
                    } else {
                        idx = n + qo - 1;
#pragma unroll
                        for (int m = 0; m < R; ++m) acc[m] = (q + LPI * m == idx) ? 1.0 : 0.0;
                    }
                }
#pragma unroll
                for (int m = 0; m < R; ++m) nt[m] = acc[m];
            } else {
                ++kt;
                wprev = wn;
#pragma unroll
                for (int m = 0; m < R; ++m) nt[m] = u[m];
            }
            buf ^= 1;
            double *to = tg + buf * C::BUF;
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (q + LPI * m < D) to[q + LPI * m] = nt[m];
        }
        __syncwarp();
    }
    if (mv_gor<LPI>(bad)) status = LMEP_NONFINITE;
    if (reps == 0 && live) {
        // failed before the iteration: outputs are NaN, the status says why
        const double qnan = __longlong_as_double(0x7ff8000000000000LL);
        for (int qq = 0; qq < sd; ++qq)
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const int j = q + LPI * m;
                if (j < n) {
                    if (P.layout == 0) P.out[(b * sd + qq) * n + j] = qnan;
                    else P.out[((int64_t)qq * n + j) * P.out_ld + b] = qnan;
                    if (want_half && qq < 2) {
                        if (P.layout == 0) P.half_out[(b * 2 + qq) * n + j] = qnan;
                        else P.half_out[((int64_t)qq * n + j) * P.out_ld + b] = qnan;
                    }
                }
            }
    }
    if (live && q == 0) {
        if (P.status) P.status[b] = status;
        if (P.ms) P.ms[b] = nmv | (min(s, 255) << 24);
    }
}

int mv_lanes_override();   // 0: default (4 lanes per item), 8: 8 lanes for d > 8

template <int D, int LPI>
int launch_mv_l(const HarvestParams &P, cudaStream_t st)
{
    using C = MvCfg<D, LPI>;
    const int64_t threads = P.B * LPI;
    const int64_t blocks = (threads + C::THREADS - 1) / C::THREADS;
    if (blocks > 0x7fffffffLL) return LMEP_INVALID_CONFIG;
    const bool shared_tab = P.mode == 1 && P.table_idx == nullptr && !P.map_on && P.nterms >= 1 &&
                            P.nterms <= 4;
    const int nt = shared_tab ? P.nterms : 0;
    const size_t shm = mv_smem_bytes<D, LPI>(nt);
    const dim3 g((unsigned)blocks), t(C::THREADS);
    switch (nt) {
    case 1: harvest_mv_kernel<D, LPI, 1><<<g, t, shm, st>>>(P); break;
    case 2: harvest_mv_kernel<D, LPI, 2><<<g, t, shm, st>>>(P); break;
    case 3: harvest_mv_kernel<D, LPI, 3><<<g, t, shm, st>>>(P); break;
    case 4: harvest_mv_kernel<D, LPI, 4><<<g, t, shm, st>>>(P); break;
    default: harvest_mv_kernel<D, LPI, 0><<<g, t, shm, st>>>(P); break;
    }
    return launch_status("harvest_mv_kernel");
}

template <int D>
int launch_mv(const HarvestParams &P, cudaStream_t st)
{
    if constexpr (D > 8) {
        if (mv_lanes_override() == 8) return launch_mv_l<D, 8>(P, st);
        return launch_mv_l<D, 4>(P, st);
    } else {
        return launch_mv_l<D, 4>(P, st);
    }
}

}  // namespace lmep
