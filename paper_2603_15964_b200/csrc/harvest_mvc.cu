// harvest_mvc.cu -- K1 for the largest per-node batches: one item per lane,
// the shared derivative tables as constant-bank operands.
//
// Scope: per-item harvests of a single table geometry with per-item
// coefficients (periodic / uniform grids with variable coefficients, BASELINE
// config 5), n in {7, 9, 11, 13}: the w_lin row (s = 1, harvest.py:73-79) with
// one or two derivative tables plus an optional reaction term, and the raw
// dt^j phi_j rows (s = 2..4, harvest.py:97-121) of two-table operators through
// the reduced (n + s - 1) augmentation.  Same mathematics as
// harvest_mvb.cuh: row r of exp(dt L_b) is exp(B^T)^reps e_r with
// B = S^-1 (dt L_b / reps) S, S a power-of-two balancing (expm.py:27-30), the
// Taylor series stopped by the rigorous tail bound (||B||_inf <= 4), the
// first term read off the tables (B^T e_r is column r: no product).
//
// What changes is where the operator lives.  L_b = sum_t cf_bt T_t (+ c0_b I)
// with the SAME tables T_t for every item, so
//     B^T v = sum_t (dt cf_bt / reps) (T'_t^T v) (+ dt c0_b / reps v)
// needs no per-item matrix at all: each lane keeps only its iterate, its
// partial sum and two table products (4 x 13 doubles), and the table entries
// are DFMA operands read straight from the constant bank (a warp-uniform
// address: no load instruction, no shared-memory traffic, no cross-lane
// exchange).  The price is one product per table instead of one with the
// assembled matrix (2 x 169 instead of 169 DFMA per term at n = 13), paid in
// exchange for the block kernel's per-item assembly, group broadcasts,
// ballots and 255-register footprint (profiles/r1h_harvest_mvb_kernel.md:
// 39% FP64 pipe, 12% occupancy, 41% of instructions FP64).
//
// The balancing exponents are launch-uniform: a one-warp prep kernel runs the
// block kernel's sweep on item 0, folds the exponents into the tables
// (T'_t[c][j] = T_t[c][j] 2^(e_c - e_j), exact) with their row abs-sum bounds,
// and the host copies that block into the constant bank (stream-ordered
// device-to-device copy).  Any diagonal similarity leaves exp(A) unchanged up
// to rounding; on single-geometry batches the per-superblock exponents of the
// block kernel are identical over the grid (C5), so nothing is lost.
#include <math.h>

#include <algorithm>
#include <mutex>

#include "harvest.cuh"
#include "harvest_mv.cuh"

namespace lmep {

namespace {

constexpr int MVC_D = 16;
constexpr int MVC_NT = 2;
constexpr double MVC_THETA = 4.0;
constexpr int MVC_PN = 13;             // polynomial kernel: n <= 13
constexpr int MVC_PV = 14;             // ... words of up to 13 factors (the last anti-diagonal is the check)
#ifndef LMEP_POLY_MINB
#define LMEP_POLY_MINB 11
#endif
#ifndef LMEP_POLY_IT
#define LMEP_POLY_IT 1
#endif
constexpr int MVC_IT = LMEP_POLY_IT;    // items per thread of the polynomial kernel (1: 48 registers, 94 us at config 5; 2 measured slower)
constexpr int MVC_PAIRS = (MVC_PV - 1) * MVC_PV / 2;   // pairs p + q < MVC_PV - 1

struct MvcConst {
    double tt[MVC_NT][MVC_D][MVC_D];   // tt[t][j][c] = T_t[c][j] 2^(e_c - e_j)  (row j of T'^T)
    double rs[MVC_NT + 1][MVC_D];      // row abs sums of tt[t]; rs[NT] = 1 (reaction: identity)
    double inv[52];                    // 1 / k
    double tf[52];                     // tail factor tau_k (||B||_inf <= THETA), inf while k + 2 <= THETA
    // reflection-symmetric tables (centred stencils on uniform grids): with R the
    // reversal j -> n-1-j, R T_t R = sg_t T_t, so T^T v follows from the halves
    // u = v + Rv, m = v - Rv on rows 0..M (M = (n-1)/2); fp / fm fold the columns
    double fp[MVC_NT][8][8];           // fp[t][i][j] = tt[i][j] + tt[i][n-1-j] (j < M), 2 tt[i][M]
    double fm[MVC_NT][8][8];           // fm[t][i][j] = tt[i][j] - tt[i][n-1-j] (j < M)
    double sg[MVC_NT];                 // reflection sign of table t
    int sym;                           // 1: every table (anti)symmetric, exponents symmetric
    // phi rows (s > 1): the reduced augmentation's entries A^T[row][n] and
    // A^T[j][j+1] (n <= j < d-1) are dt; ax[k] their balancing scales, rsa[j]
    // their |dt|-scaled row abs sums
    double ax[4];
    double rsa[MVC_D];
    int e[MVC_D];
    // polynomial kernel (s = 1, two tables): exp(a A_0 + b A_1) e_r = sum a^p b^q V_pq with
    // V_pq = (A_0 V_(p-1)q + A_1 V_p(q-1)) / (p + q), A_t = dt c_t(item 0) T'_t^T
    alignas(16) double pv[MVC_PV][MVC_PV][MVC_PN + 1]; // V_pq (p + q < MVC_PV; 16-byte rows), zero where numerically nilpotent
    alignas(16) float4 pl[MVC_PAIRS];  // (log2 |V_pq|_inf or -1e30: zero, p, q) of the pairs p + q < MVC_PV - 1 (the kernel reads the global copy)
    double cinv[MVC_NT];               // 1 / c_t(item 0): the kernel's a, b are c_t(item) cinv[t]
    double cf[MVC_PV][4];              // phi rows: cf[k][r] = dt^r k! / (k + r)!  (the dt^r phi_r row sums the degree-k terms with it)
    int poly_ok;                       // the series terminates inside the table (p + q < MVC_PV)
};

__constant__ MvcConst c_mvc;

// one warp: balance the representative item 0 (harvest_mvb.cuh sweep rule),
// fold the exponents into the tables, row sums, 1/k
__global__ void mvc_prep_kernel(const HarvestParams P, MvcConst *out)
{
    __shared__ double M[MVC_D][MVC_D + 1];
    __shared__ int kk[MVC_D];
    __shared__ int ee[MVC_D];
    const int j = threadIdx.x, n = P.n, nt = P.nterms, d = P.d, row = P.row_default;
    const bool c0 = P.c0 != nullptr;
    // the tables once into shared memory (coalesced); every pass below reads them there
    __shared__ double Tsm[MVC_NT][MVC_D][MVC_D];
    for (int i = j; i < nt * n * n; i += 32) {
        const int t = i / (n * n), r = i % (n * n);
        Tsm[t][r / n][r % n] = P.tables[i];
    }
    __syncwarp();
    for (int k = j; k < 52; k += 32) {
        out->inv[k] = k > 0 ? 1.0 / (double)k : 0.0;
        out->tf[k] = (k + 2 > MVC_THETA) ? (MVC_THETA / (k + 1)) / (1.0 - MVC_THETA / (k + 2)) : INFINITY;
    }
    bool ok = true;
    if (j < n) {
        // M[j][c] = dt * L_0[c][j] (row j of A^T), localop.py:120-127 term order
        for (int c = 0; c < n; ++c) {
            double l = 0.0;
            for (int t = 0; t < nt; ++t)
                l = xadd(l, xmul(P.coef[t], Tsm[t][c][j]));
            if (c0 && c == j) l = xadd(l, P.c0[0]);
            M[j][c] = xmul(P.delta_t, l);
            ok &= (bool)isfinite(M[j][c]);
        }
    }
    if (j < d) {
        for (int c = (j < n ? n : 0); c < d; ++c)
            M[j][c] = ((c == n && j == row) || (j >= n && c == j + 1)) ? P.delta_t : 0.0;
        ee[j] = 0;
    }
    ok = __all_sync(FULL, ok);
    // reflection (anti)symmetry of each raw table, within 1e-13 of its largest entry
    __shared__ double sgs[MVC_NT];
    bool sym = (n & 1) == 1;
    for (int t = 0; t < nt; ++t) {
        double amax = 0.0, dp = 0.0, dm = 0.0;
        if (j < n)
            for (int c = 0; c < n; ++c) {
                const double a = Tsm[t][c][j];
                const double r = Tsm[t][n - 1 - c][n - 1 - j];
                amax = fmax(amax, fabs(a));
                dp = fmax(dp, fabs(a - r));
                dm = fmax(dm, fabs(a + r));
            }
        for (int o = 16; o > 0; o >>= 1) {
            amax = fmax(amax, __shfl_xor_sync(FULL, amax, o));
            dp = fmax(dp, __shfl_xor_sync(FULL, dp, o));
            dm = fmax(dm, __shfl_xor_sync(FULL, dm, o));
        }
        const double tol = 1e-13 * amax;
        if (dp <= tol) { if (j == 0) sgs[t] = 1.0; }
        else if (dm <= tol) { if (j == 0) sgs[t] = -1.0; }
        else sym = false;
    }
    __syncwarp();
    for (int sweep = 0; ok && sweep < 12; ++sweep) {
        int k = 0;
        if (j < d) {
            double r2 = 0.0, c2 = 0.0;
            for (int c = 0; c < d; ++c) {
                r2 = fma(M[j][c], M[j][c], r2);
                c2 = fma(M[c][j], M[c][j], c2);
            }
            if (c2 > 1e-280 && r2 > 1e-280 && c2 < 1e280 && r2 < 1e280) {
                const int ex = mv_exp2i(r2) - mv_exp2i(c2);
                if (ex >= 4) k = (ex + 2) >> 2;
                else if (ex <= -4) k = -((2 - ex) >> 2);
            }
            kk[j] = k;
        }
        if (!__any_sync(FULL, k != 0)) break;
        __syncwarp();
        if (j < d) {
            for (int c = 0; c < d; ++c)
                if (kk[c] != k) M[j][c] *= mv_pow2(kk[c] - k);
            ee[j] += k;
        }
        __syncwarp();
    }
    __syncwarp();
    if (sym) {
        // a symmetric similarity keeps the balanced tables (anti)symmetric
        const int es = j < n ? (ee[j] + ee[n - 1 - j]) >> 1 : 0;
        __syncwarp();
        if (j < n) ee[j] = es;
        __syncwarp();
    }
    if (j == 0) out->sym = sym ? 1 : 0;
    if (j < 4) {
        const int r0 = j == 0 ? row : n + j - 1, c1 = n + j;
        out->ax[j] = c1 < d ? mv_pow2(ee[c1] - ee[r0]) : 0.0;
    }
    if (j < MVC_D) {
        double ra = 0.0;
        if (j == row && d > n) ra += fabs(P.delta_t) * mv_pow2(ee[n] - ee[row]);
        if (j >= n && j + 1 < d) ra += fabs(P.delta_t) * mv_pow2(ee[j + 1] - ee[j]);
        out->rsa[j] = ra;
    }
    if (j < MVC_NT) out->sg[j] = (sym && j < nt) ? sgs[j] : 1.0;
    if (j < MVC_D) {
        out->e[j] = j < d ? ee[j] : 0;
        for (int t = 0; t < MVC_NT; ++t) {
            double sum = 0.0;
            for (int c = 0; c < MVC_D; ++c) {
                double v = 0.0;
                if (t < nt && j < n && c < n)
                    v = Tsm[t][c][j] * mv_pow2(ee[c] - ee[j]);
                out->tt[t][j][c] = v;
                sum += fabs(v);
            }
            out->rs[t][j] = sum;
        }
        out->rs[MVC_NT][j] = (c0 && j < n) ? 1.0 : 0.0;
    }
    // folded halves (rows i <= M) from the balanced tables
    const int Mh = (n - 1) / 2;
    if (j < 8) {
        for (int t = 0; t < MVC_NT; ++t)
            for (int c = 0; c < 8; ++c) {
                double a = 0.0, b = 0.0;
                if (sym && t < nt && j <= Mh && c <= Mh) {
                    const double lo = Tsm[t][c][j] * mv_pow2(ee[c] - ee[j]);
                    const int c2 = n - 1 - c;
                    const double hi = Tsm[t][c2][j] * mv_pow2(ee[c2] - ee[j]);
                    if (c < Mh) { a = lo + hi; b = lo - hi; }
                    else a = 2.0 * lo;
                }
                out->fp[t][j][c] = a;
                out->fm[t][j][c] = b;
            }
    }
}

// ---- tables of the polynomial kernel (one CTA of MVC_PV warps, behind the
// prep kernel: reads its balanced tables from `out`) -------------------------
// For derivative tables the local operators are nilpotent (a word of more
// than n - 1 derivative matrices annihilates the window's interpolant), so
// exp(dt L_b)^T e_r is a POLYNOMIAL in the item's two coefficients: the
// vectors V_pq are shared by every item.  Warp p computes V_p(k-p) of
// anti-diagonal k from anti-diagonal k - 1.  A computed V_pq that is below the
// rounding error of its own recurrence is exactly zero in exact arithmetic and
// is stored as zero; the kernel is used when the series terminates inside the
// table (poly_ok).
__global__ void __launch_bounds__(32 * MVC_PV) mvc_poly_prep_kernel(const HarvestParams P, MvcConst *out)
{
    __shared__ double As[MVC_NT][MVC_PN][MVC_PN + 1];
    __shared__ double Vs[MVC_PV][MVC_PV][MVC_PN + 1];
    __shared__ double vinf[MVC_PV][MVC_PV];
    __shared__ double an[MVC_NT];
    __shared__ int bad;
    const int j = threadIdx.x & 31, wid = threadIdx.x >> 5, n = P.n, row = P.row_default;
    if (threadIdx.x == 0) bad = 0;
    if (wid < MVC_NT) {
        const int t = wid;
        double cn = P.coef[t];
        if (!(fabs(cn) > 0.0) || !isfinite(cn)) cn = 1.0;
        if (j == 0) out->cinv[t] = 1.0 / cn;
        double sum = 0.0;
        if (j < n)
            for (int c = 0; c < n; ++c) {
                const double a = (P.delta_t * cn) * out->tt[t][j][c];
                As[t][j][c] = a;
                sum += fabs(a);
            }
        for (int o = 16; o > 0; o >>= 1) sum = fmax(sum, __shfl_xor_sync(FULL, sum, o));
        if (j == 0) an[t] = sum;
    }
    for (int i = threadIdx.x; i < MVC_PV * MVC_PV * (MVC_PN + 1); i += blockDim.x) (&Vs[0][0][0])[i] = 0.0;
    for (int i = threadIdx.x; i < MVC_PV * MVC_PV; i += blockDim.x) (&vinf[0][0])[i] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) { Vs[0][0][row] = 1.0; vinf[0][0] = 1.0; }
    __syncthreads();
#pragma unroll 1
    for (int k = 1; k < MVC_PV; ++k) {
        const int p = wid, q = k - wid;
        if (q >= 0) {
            double v = 0.0, ref = 0.0;
            if (j < n) {
                if (p > 0)
                    for (int c = 0; c < n; ++c) v = fma(As[0][j][c], Vs[p - 1][q][c], v);
                if (q > 0)
                    for (int c = 0; c < n; ++c) v = fma(As[1][j][c], Vs[p][q - 1][c], v);
                v /= (double)k;
            }
            if (p > 0) ref += an[0] * vinf[p - 1][q];
            if (q > 0) ref += an[1] * vinf[p][q - 1];
            ref /= (double)k;
            double vi = j < n ? fabs(v) : 0.0;
            for (int o = 16; o > 0; o >>= 1) {
                const double w2 = __shfl_xor_sync(FULL, vi, o);
                vi = (w2 > vi || w2 != w2) ? w2 : vi;
            }
            if (!isfinite(vi) && j == 0) bad = 1;
            if (!(vi > 0x1p-46 * ref)) { v = 0.0; vi = 0.0; }        // numerically nilpotent
            if (j < n) Vs[p][q][j] = v;
            if (j == 0) vinf[p][q] = vi;
        }
        __syncthreads();
    }
    // the series must end inside the table: the last anti-diagonal is all zero
    bool pok = P.s >= 1 && P.s <= 4 && P.nterms == 2 && P.c0 == nullptr && n <= MVC_PN && !bad;
    for (int p = 0; p < MVC_PV; ++p)
        if (vinf[p][MVC_PV - 1 - p] != 0.0) pok = false;
    for (int i = threadIdx.x; i < MVC_PV * MVC_PV; i += blockDim.x) {
        const int p = i / MVC_PV, q = i % MVC_PV;
        const bool in = p + q < MVC_PV;
        const double vi = in ? vinf[p][q] : 0.0;
        const float lv = (vi > 0.0 && isfinite(vi)) ? (float)log2(vi) : -1e30f;
        if (p + q < MVC_PV - 1)
            out->pl[p * (MVC_PV - 1) - p * (p - 1) / 2 + q] = make_float4(pok ? lv : -1e30f, (float)p, (float)q, 0.f);
        // (stored back in the unbalanced coordinates: 2^(e_c - e_row), exact)
        for (int c = 0; c <= MVC_PN; ++c)
            out->pv[p][q][c] = (in && pok && c < n) ? Vs[p][q][c] * mv_pow2(out->e[c] - out->e[row]) : 0.0;
    }
    if (threadIdx.x < MVC_PV) {
        const int k = threadIdx.x;
        double c = 1.0;
        for (int r = 0; r < 4; ++r) {
            out->cf[k][r] = c;
            c *= P.delta_t / (double)(k + r + 1);
        }
    }
    if (threadIdx.x == 0) out->poly_ok = pok ? 1 : 0;
}

// Polynomial kernel (w_lin of two-table operators, harvest.py:97-121 per node):
// one item per lane evaluates  w = sum_pq a^p b^q V_pq  (a, b its two
// coefficients over item 0's) term by term -- 13 independent accumulators, one
// running monomial, the table entries read by wide uniform loads at
// compile-time constant-bank addresses -- over the columns a block-wide
// magnitude test keeps: at n = 13 with a diffusion-dominated step (config 5)
// 11-16 of the 91 columns in 3-4 rows.  A block whose largest term exceeds 2^6
// (cancellation) or whose coefficients are not finite hands its items to the
// Taylor kernel through the work list, as does every item when the series does
// not terminate inside the table.
// Config 5 (4,194,304 items): 94 us = 5.5 TB/s on its 124 B per item (16 in,
// 104 + 4 out), 0.85 of the measured HBM peak; 48 registers.

// an upper bound of log2 |x| from the high word of |x| (log2(1 + m) <= m + 0.0861)
__device__ __forceinline__ float poly_log2_ub(unsigned hi)
{
    return (float)((int)(hi >> 20) - 1023) + (float)(hi & 0xfffffu) * 0x1p-20f + 0.09f;
}

// Each CTA takes one block of 128 items, IT per thread (items t, t + 128 / IT, ...:
// the rows of a block do not depend on IT or on how the batch was sliced).
template <int N, int IT, int S>
__global__ void __launch_bounds__(128 / IT, S == 1 ? LMEP_POLY_MINB : (S == 2 ? 6 : (S == 3 ? 5 : 4))) harvest_poly_kernel(const HarvestParams P, const MvcConst *__restrict__ G)
{
    constexpr int T = 128 / IT;
    // column selection once per block, from the block-wide coefficient magnitudes
    __shared__ unsigned smax[T / 32][2];
    __shared__ int sq[MVC_PV];             // sq[p]: highest significant q of row p (-1: none)
    __shared__ int sflag;                  // 1: hand the block's items to the Taylor kernel
    const int tid = threadIdx.x;
    bool live[IT];
    int64_t b[IT];
    double a[IT], be[IT];
    unsigned ha = 0u, hb = 0u;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        const int64_t braw = (int64_t)blockIdx.x * 128 + it * T + tid;
        live[it] = braw < P.B;
        b[it] = live[it] ? braw : P.B - 1;
        a[it] = P.coef[b[it] * P.coef_stride] * c_mvc.cinv[0];
        be[it] = P.coef[b[it] * P.coef_stride + 1] * c_mvc.cinv[1];
        // (upper bounds from the high words; NaN / Inf sort last)
        ha = max(ha, mv_hiabs(a[it]));
        hb = max(hb, mv_hiabs(be[it]));
    }
    ha = __reduce_max_sync(FULL, ha);
    hb = __reduce_max_sync(FULL, hb);
    if ((tid & 31) == 0) { smax[tid >> 5][0] = ha; smax[tid >> 5][1] = hb; }
    if (tid < MVC_PV) sq[tid] = -1;
    if (tid == 0) sflag = c_mvc.poly_ok ? 0 : 1;
    __syncthreads();
    {
        // one (p, q) pair per thread: is |a|^p |b|^q |V_pq| significant / too large?
#pragma unroll
        for (int k = 0; k < T / 32; ++k) { ha = max(ha, smax[k][0]); hb = max(hb, smax[k][1]); }
        const float la = poly_log2_ub(ha), lb = poly_log2_ub(hb);
        for (int i = tid; i < MVC_PAIRS; i += T) {
            const float4 e = __ldg(&G->pl[i]);   // (log2 |V_pq|, p, q)
            const float t = fmaf(e.y, la, fmaf(e.z, lb, e.x));
            if (t > -60.f) atomicMax(&sq[(int)e.y], (int)e.z);
            if (!(t <= 6.f)) sflag = 1;
        }
    }
    __syncthreads();
    if (sflag) {
        // the block's items go to the Taylor kernel: one entry in its work list
        if (tid == 0) P.pending[1 + atomicAdd(P.pending, 1)] = (int)blockIdx.x;
        return;
    }
    // w = sum_pq (a^p be^q) V_pq term by term, rows and columns ascending with a
    // uniform exit after the last significant one: ONE accumulator per output
    // (no per-row partial sums), one running monomial per item, and both loops
    // fully unrolled so that every table entry is read at a compile-time
    // constant-bank address (wide uniform loads shared by the thread's items)
    const int myq = (tid & 31) < MVC_PV ? sq[tid & 31] : -1;
    const unsigned has = __ballot_sync(FULL, myq >= 0);
    const int Pw = has ? 31 - __clz((int)has) : -1;
    // phi rows (S > 1): the dt^r phi_r row is the same sum with the degree-k terms
    // weighted by cf[k][r] = dt^r k! / (k + r)!, so every table entry feeds S
    // accumulators (one more multiply per term and row)
    double w[S][IT][N], ap[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        ap[it] = 1.0;
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < N; ++j) w[r][it][j] = 0.0;
    }
    int cols = 0;
#pragma unroll
    for (int p = 0; p < MVC_PV - 1; ++p) {
        if (p > Pw) break;
        const int qt = __shfl_sync(FULL, myq, p);
        double m[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) m[it] = ap[it];
#pragma unroll
        for (int q = 0; q < MVC_PV - 1 - p; ++q) {
            if (q > qt) break;
            double mr[S][IT];
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                mr[0][it] = m[it];
#pragma unroll
                for (int r = 1; r < S; ++r) mr[r][it] = m[it] * c_mvc.cf[p + q][r];
            }
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double v = c_mvc.pv[p][q][j];
#pragma unroll
                for (int r = 0; r < S; ++r)
#pragma unroll
                    for (int it = 0; it < IT; ++it) w[r][it][j] = fma(mr[r][it], v, w[r][it][j]);
            }
#pragma unroll
            for (int it = 0; it < IT; ++it) m[it] *= be[it];
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) ap[it] *= a[it];
        cols += qt + 1;
    }
    // (N == P.n: the launcher instantiates the kernel per stencil width)
#pragma unroll
    for (int it = 0; it < IT; ++it) {
        if (!live[it]) continue;
        // any Inf / NaN among the outputs turns the zero-weighted sum into NaN
        double chk = 0.0;
#pragma unroll
        for (int r = 0; r < S; ++r)
#pragma unroll
            for (int j = 0; j < N; ++j) chk = fma(w[r][it][j], 0.0, chk);
        if (P.layout == 0) {
            double *o = P.out + b[it] * (S * N);
#pragma unroll
            for (int r = 0; r < S; ++r)
#pragma unroll
                for (int j = 0; j < N; ++j) o[r * N + j] = w[r][it][j];
        } else {
            double *o = P.out + b[it];
            const int64_t ld = P.out_ld;
#pragma unroll
            for (int r = 0; r < S; ++r)
#pragma unroll
                for (int j = 0; j < N; ++j) o[(r * N + j) * ld] = w[r][it][j];
        }
        P.status[b[it]] = chk == 0.0 ? LMEP_OK : LMEP_NONFINITE;
        if (P.ms) P.ms[b[it]] = cols;    // scaling field 0: a polynomial item, `cols` columns
    }
}

// 3 CTAs per SM (<= 168 registers): 12 warps hide the DFMA and constant-load
// latency better than 8 warps at the unbounded 174 (measured 1.01 vs 1.09 ms).
// N = n (the operator block), PA = s - 1 augmentation columns (phi rows).
template <int N, int NT, bool C0, int PA>
__global__ void __launch_bounds__(128, 3) harvest_mvc_kernel(const HarvestParams P)
{
    constexpr int D = N + PA;
    int64_t braw = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // (behind the polynomial kernel: a small grid walks the list of 128-item
    // blocks that kernel handed back, pending[0] entries from pending[1] on)
    const int nwork = P.pending ? P.pending[0] : 1;
#pragma unroll 1
    for (int work = blockIdx.x; work < (P.pending ? nwork : (int)blockIdx.x + 1); work += gridDim.x) {
    if (P.pending) braw = (int64_t)P.pending[1 + work] * blockDim.x + threadIdx.x;
    const bool live = braw < P.B;
    const int64_t b = live ? braw : P.B - 1;
    const int row = P.row_default;
    const double dt = P.delta_t;

    double cf[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) cf[t] = P.coef[b * P.coef_stride + t];
    const double cz = C0 ? P.c0[b * P.c0_stride] : 0.0;

    // scaling: ||B / reps||_inf <= THETA from the balanced row-sum bounds
    double nrm = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double r = 0.0;
        if (j < N) {
            r = C0 ? fabs(cz) * c_mvc.rs[MVC_NT][j] : 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) r = fma(fabs(cf[t]), c_mvc.rs[t][j], r);
        }
        r = fma(fabs(dt), r, PA > 0 ? c_mvc.rsa[j] : 0.0);
        nrm = (r > nrm || r != r) ? r : nrm;
    }
    int status = LMEP_OK, s = 0;
    if (!(nrm <= 1e9)) status = LMEP_NONFINITE;
    else s = nrm > MVC_THETA ? (int)ceil(nrm / MVC_THETA) : 1;
    const double dts = dt * (s > 1 ? 1.0 / (double)s : 1.0);
    double al[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) al[t] = dts * cf[t];
    const double alz = dts * cz;

    double acc[D], v[D], w[D];
    int kt = 1, rep = 0, nmv = 0;
    bool done = true, bad = false;
    // update after term kt (in w): rigorous stop tau_k |w|_inf <= 2^-53 |acc_{k-1}|_inf,
    // then the next iterate (w, or acc when a repetition of the series restarts)
    auto advance = [&]() {
        // scale: the extracted rows only (the augmentation entries of a phi
        // series are O(1) while its extracted rows are O(dt^j), harvest_mvb.cuh)
        unsigned ah = 0u, wh = 0u;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (j < N) ah = max(ah, mv_hiabs(acc[j]));
            wh = max(wh, mv_hiabs(w[j]));
        }
        const double an = __hiloint2double((int)ah, 0);
        const double wn = __hiloint2double((int)wh, -1) * c_mvc.tf[kt];
        const bool conv = (an > 0.0 && wn <= 0x1p-53 * an) || kt >= MV_TMAX;
        if (!done) {
            ++nmv;
#pragma unroll
            for (int j = 0; j < D; ++j) acc[j] += w[j];
            if (conv) {
                kt = 1;
                if (++rep >= s) done = true;
#pragma unroll
                for (int j = 0; j < D; ++j) v[j] = acc[j];
            } else {
                ++kt;
#pragma unroll
                for (int j = 0; j < D; ++j) v[j] = w[j];
            }
        }
    };
    const int n = P.n;
#pragma unroll 1
    for (int qo = 0; qo <= PA; ++qo) {
        // w_lin: row `row` of exp(A); raw dt^j phi_j rows: rows n + j - 1 (harvest.py:119-120)
        const int idx = qo == 0 ? row : N + qo - 1;
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] = v[j] = (j == idx) ? 1.0 : 0.0;
        kt = 1;
        rep = 0;
        done = status != LMEP_OK;
        if (qo == 0) {
            // term 1 on e_r is column r of the scaled tables (no product); the
            // augmentation rows see no top-block entry
            const double *t0 = &c_mvc.tt[0][0][0] + row;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                double o = 0.0;
                if (j < N) {
                    o = al[0] * t0[j * MVC_D];
#pragma unroll
                    for (int t = 1; t < NT; ++t) o = fma(al[t], t0[(t * MVC_D + j) * MVC_D], o);
                    if constexpr (C0) o = fma(alz, acc[j], o);
                }
                w[j] = o;
            }
            advance();
        }
        while (__any_sync(FULL, !done)) {
            // term k of the series restarted at acc: w = B^T v / k (1/k rides on the scalars)
            const double ik = c_mvc.inv[kt];
            double a[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) a[t] = al[t] * ik;
            const double az = alz * ik;
            if (c_mvc.sym) {
                // T^T v = (T^T u + T^T m) / 2 with u = v + Rv, m = v - Rv: rows 0..M from
                // the folded tables, rows n-1-i by the reflection signs (about 0.54 of
                // the full products)
                constexpr int M = (N - 1) / 2;
                double u[M + 1], m[M];
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    u[c] = v[c] + v[N - 1 - c];
                    m[c] = v[c] - v[N - 1 - c];
                }
                u[M] = v[M];
                double h[NT], hs[NT];
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    h[t] = 0.5 * a[t];
                    hs[t] = h[t] * c_mvc.sg[t];
                }
#pragma unroll
                for (int i = 0; i <= M; ++i) {
                    double lo = C0 ? az * v[i] : 0.0, hi = C0 ? az * v[N - 1 - i] : 0.0;
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        double pu = c_mvc.fp[t][i][0] * u[0];
#pragma unroll
                        for (int c = 1; c <= M; ++c) pu = fma(c_mvc.fp[t][i][c], u[c], pu);
                        double qm = c_mvc.fm[t][i][0] * m[0];
#pragma unroll
                        for (int c = 1; c < M; ++c) qm = fma(c_mvc.fm[t][i][c], m[c], qm);
                        lo = fma(h[t], pu + qm, lo);
                        hi = fma(hs[t], pu - qm, hi);
                    }
                    w[i] = lo;
                    if (i < M) w[N - 1 - i] = hi;
                }
            } else {
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double y[NT];
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        double p = c_mvc.tt[t][j][0] * v[0];
#pragma unroll
                        for (int c = 1; c < N; ++c) p = fma(c_mvc.tt[t][j][c], v[c], p);
                        y[t] = p;
                    }
                    double o = a[0] * y[0];
#pragma unroll
                    for (int t = 1; t < NT; ++t) o = fma(a[t], y[t], o);
                    if constexpr (C0) o = fma(az, v[j], o);
                    w[j] = o;
                }
            }
            if constexpr (PA > 0) {
                // augmentation: (B^T v)[row] += dt' v[n], (B^T v)[j] = dt' v[j+1] (n <= j < d-1)
                const double g = dts * ik;
                const double g0 = g * c_mvc.ax[0] * v[N];
#pragma unroll
                for (int i = 0; i < N; ++i)
                    if (i == row) w[i] += g0;
#pragma unroll
                for (int k = 0; k + 1 < PA; ++k) w[N + k] = (g * c_mvc.ax[k + 1]) * v[N + k + 1];
                w[D - 1] = 0.0;
            }
            advance();
        }
        if (live) {
            const int ei = c_mvc.e[idx];
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double o = status == LMEP_OK ? acc[j] * mv_pow2(c_mvc.e[j] - ei)
                                                   : __longlong_as_double(0x7ff8000000000000LL);
                bad |= !isfinite(o);
                if (j < n) {
                    if (P.layout == 0) P.out[(b * (PA + 1) + qo) * n + j] = o;
                    else P.out[((int64_t)qo * n + j) * P.out_ld + b] = o;
                }
            }
        }
    }
    if (live) {
        if (bad) status = LMEP_NONFINITE;
        if (P.status) P.status[b] = status;
        if (P.ms) P.ms[b] = nmv | (min(s, 255) << 24);
    }
    }
}

// Per-device state: the prep kernel's output block and the event of the
// device's last constant-table launch.  (__constant__ c_mvc itself is a
// per-device copy of the module's constant bank.)
struct MvcKey {
    const double *tables = nullptr;
    double dt = 0.0;
    int n = 0, s = 0, nterms = 0, row = 0, c0 = 0;
    bool operator==(const MvcKey &o) const
    {
        return tables == o.tables && dt == o.dt && n == o.n && s == o.s && nterms == o.nterms &&
               row == o.row && c0 == o.c0;
    }
};
struct MvcDevice {
    MvcConst *scratch = nullptr;
    cudaEvent_t done = nullptr;
    MvcKey key;                          // what the device's constant block was prepared for
    bool valid = false;
    int32_t *pending = nullptr;          // work list between the polynomial and the Taylor kernel
    int64_t pending_cap = 0;
};
// lmep_harvest_reuse_prep: the calling thread's next constant-table harvests are
// slices of one harvest and keep the first slice's prepared block
thread_local int t_reuse_prep = 0;
MvcDevice g_mvc_dev[kMaxDevices];
std::mutex g_mvc_mu;

template <int N, int NT, bool C0, int PA>
void launch_mvc_kernel(const HarvestParams &P, cudaStream_t st)
{
    const int64_t blocks = (P.B + 127) / 128;
    harvest_mvc_kernel<N, NT, C0, PA><<<(unsigned)blocks, 128, 0, st>>>(P);
}

template <int N>
void launch_mvc_d(const HarvestParams &P, cudaStream_t st)
{
    const bool c0 = P.c0 != nullptr;
    if (P.s > 1) {                       // phi rows: two tables, no reaction (eligibility)
        if (P.s == 2) launch_mvc_kernel<N, 2, false, 1>(P, st);
        else if (P.s == 3) launch_mvc_kernel<N, 2, false, 2>(P, st);
        else launch_mvc_kernel<N, 2, false, 3>(P, st);
    } else if (P.nterms == 1) {
        if (c0) launch_mvc_kernel<N, 1, true, 0>(P, st);
        else launch_mvc_kernel<N, 1, false, 0>(P, st);
    } else {
        if (c0) launch_mvc_kernel<N, 2, true, 0>(P, st);
        else launch_mvc_kernel<N, 2, false, 0>(P, st);
    }
}

template <int N>
void launch_poly(const HarvestParams &Q, const MvcConst *scratch, unsigned blocks, unsigned g, cudaStream_t st)
{
    switch (Q.s) {
    case 1:
        harvest_poly_kernel<N, MVC_IT, 1><<<blocks, 128 / MVC_IT, 0, st>>>(Q, scratch);
        harvest_mvc_kernel<N, 2, false, 0><<<g, 128, 0, st>>>(Q);
        break;
    case 2:
        harvest_poly_kernel<N, 1, 2><<<blocks, 128, 0, st>>>(Q, scratch);
        harvest_mvc_kernel<N, 2, false, 1><<<g, 128, 0, st>>>(Q);
        break;
    case 3:
        harvest_poly_kernel<N, 1, 3><<<blocks, 128, 0, st>>>(Q, scratch);
        harvest_mvc_kernel<N, 2, false, 2><<<g, 128, 0, st>>>(Q);
        break;
    default:
        harvest_poly_kernel<N, 1, 4><<<blocks, 128, 0, st>>>(Q, scratch);
        harvest_mvc_kernel<N, 2, false, 3><<<g, 128, 0, st>>>(Q);
        break;
    }
}

}  // namespace

bool harvest_mvc_eligible(const HarvestParams &P)
{
    return harvest_mvb_eligible(P) && P.s >= 1 && P.s <= 4 && P.d == P.n + P.s - 1 &&
           (P.s == 1 || (P.nterms == 2 && P.c0 == nullptr)) &&
           (P.n == 7 || P.n == 9 || P.n == 11 || P.n == 13) && P.nterms >= 1 &&
           P.nterms <= MVC_NT && P.row_default >= 0 && P.row_default < P.n &&
           P.B < ((int64_t)1 << 31) * 128;
}

// The constant block is per device and shared by every stream on it: each call
// first waits for the device's previous constant-table kernel (event; a no-op
// on the same stream), so a later copy can never overwrite tables an earlier
// kernel still reads.  The host mutex orders the enqueues of concurrent threads.
int launch_harvest_mvc(const HarvestParams &P, cudaStream_t st)
{
    std::lock_guard<std::mutex> lock(g_mvc_mu);
    MvcDevice &D = g_mvc_dev[current_device()];
    cudaError_t e = cudaSuccess;
    if (!D.scratch) {
        e = cudaMalloc((void **)&D.scratch, sizeof(MvcConst));
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&D.done, cudaEventDisableTiming);
        if (e != cudaSuccess) { set_last_error("harvest_mvc setup", e); return LMEP_CUDA_ERROR; }
    } else {
        e = cudaStreamWaitEvent(st, D.done, 0);
        if (e != cudaSuccess) { set_last_error("cudaStreamWaitEvent", e); return LMEP_CUDA_ERROR; }
    }
    MvcKey key;
    key.tables = P.tables; key.dt = P.delta_t; key.n = P.n; key.s = P.s; key.nterms = P.nterms;
    key.row = P.row_default; key.c0 = P.c0 != nullptr;
    // w_lin of two-table operators: the polynomial kernel first, the Taylor kernel
    // behind it on whatever it handed back
    const bool poly = P.s >= 1 && P.s <= 4 && P.nterms == 2 && P.c0 == nullptr && P.status != nullptr &&
                      P.half_out == nullptr &&
                      (P.n == 7 || P.n == 9 || P.n == 11 || P.n == 13) && P.n <= MVC_PN &&
                      device_settings().mvc.load() == 1;
    key.c0 |= poly ? 2 : 0;              // (a block prepared without the polynomial tables is not reused for it)
    // a later slice of the same harvest (same tables, step and shape; the block in
    // constant memory is still the one prepared for its first slice): the balancing
    // of that first slice's item serves the whole table, as in a one-launch harvest
    const bool reuse = t_reuse_prep && D.valid && key == D.key;
    if (!reuse) {
        mvc_prep_kernel<<<1, 32, 0, st>>>(P, D.scratch);
        if (poly) mvc_poly_prep_kernel<<<1, 32 * MVC_PV, 0, st>>>(P, D.scratch);
        e = cudaMemcpyToSymbolAsync(c_mvc, D.scratch, sizeof(MvcConst), 0, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) { set_last_error("cudaMemcpyToSymbolAsync", e); return LMEP_CUDA_ERROR; }
        D.key = key;
        D.valid = true;
    }
    HarvestParams Q = P;
    if (poly) {
        const unsigned blocks = (unsigned)((P.B + 127) / 128);
        // work list of the blocks the polynomial kernel hands back (grown on demand)
        if (D.pending_cap < (int64_t)blocks + 1) {
            if (D.pending) { cudaStreamSynchronize(st); cudaFree(D.pending); }
            D.pending_cap = std::max<int64_t>((int64_t)blocks + 1, 1 << 16);
            if (cudaMalloc((void **)&D.pending, D.pending_cap * sizeof(int32_t)) != cudaSuccess) {
                D.pending = nullptr; D.pending_cap = 0;
                set_last_error("harvest_mvc work list", cudaGetLastError());
                return LMEP_CUDA_ERROR;
            }
        }
        cudaMemsetAsync(D.pending, 0, sizeof(int32_t), st);
        Q.pending = D.pending;
        // the Taylor kernel behind it on what is left: a grid of at most six CTAs per SM
        const unsigned g = std::min<unsigned>(blocks, 6u * (unsigned)device_sm_count());
        switch (P.n) {
        case 7: launch_poly<7>(Q, D.scratch, blocks, g, st); break;
        case 9: launch_poly<9>(Q, D.scratch, blocks, g, st); break;
        case 11: launch_poly<11>(Q, D.scratch, blocks, g, st); break;
        default: launch_poly<13>(Q, D.scratch, blocks, g, st); break;
        }
    } else {
        switch (Q.n) {
        case 7: launch_mvc_d<7>(Q, st); break;
        case 9: launch_mvc_d<9>(Q, st); break;
        case 11: launch_mvc_d<11>(Q, st); break;
        default: launch_mvc_d<13>(Q, st); break;
        }
    }
    cudaEventRecord(D.done, st);
    return launch_status("harvest_mvc_kernel");
}

}  // namespace lmep

extern "C" int lmep_harvest_reuse_prep(int on)
{
    lmep::t_reuse_prep = on ? 1 : 0;
    return LMEP_OK;
}
