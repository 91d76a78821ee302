// harvest.cu -- K1/K2: batched fp64 local-operator assembly, matrix exponential
// and weight-row extraction (sm_100a).
//
// Reference path being replaced (per node, in Python):
//   localop.fornberg_weights      localop.py:61-96
//   localop.local_operator        localop.py:111-128
//   harvest.build_augmented       harvest.py:82-94
//   expm.expm                     expm.py:24-42  -> scipy.linalg.matrix_balance
//                                                   + scipy.linalg.expm (AMH 2009)
//   harvest.harvest_phi_weights   harvest.py:97-121
//
// Design: one warp owns one matrix.  The d x d (d <= 32) operands live in
// shared memory padded to DP x (DP+1) doubles (odd leading dimension: the
// column-parallel reads of a matrix product hit distinct banks).  Lane
// (c, g) = (lane % DP, lane / DP) owns column c of rows g, g+G, g+2G, ...
// (G = 32/DP), so a product C = A B costs per k one conflict-free read of
// B[k][c] plus E = DP/G broadcast reads of A[r][k] for E FMAs.  Reductions
// (norms, pivots, balancing sums) are warp shuffles; there are no block-level
// barriers, every warp runs independently.
#include <math.h>

#include <algorithm>

#include "harvest.cuh"

namespace lmep {

// --------------------------------------------------------------------------
// Fornberg weights (localop.py:61-96), bit-identical: separate IEEE roundings
// in the reference's evaluation order.  One thread per item.
// --------------------------------------------------------------------------
__global__ void fornberg_kernel(const double *__restrict__ z, const double *__restrict__ x,
                                int64_t xs, int n, int m, int64_t B, double *__restrict__ out)
{
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double *xb = x + b * xs;
    // the table lives in shared memory while the recursion reads back what it
    // just wrote; global stores would send every such read to L2 (47 us for one
    // 13-node table before this change)
    extern __shared__ double fb_sm[];
    double *c = fb_sm + threadIdx.x * (m + 1) * n;   // c[k*n + j]
    const double zz = z[b];
    for (int i = 0; i < (m + 1) * n; ++i) c[i] = 0.0;
    c[0] = 1.0;
    double c1 = 1.0;
    double c4 = xsub(xb[0], zz);
    for (int i = 1; i < n; ++i) {
        const int mn = i < m ? i : m;
        double c2 = 1.0;
        const double c5 = c4;
        c4 = xsub(xb[i], zz);
        for (int j = 0; j < i; ++j) {
            const double c3 = xsub(xb[i], xb[j]);
            c2 = xmul(c2, c3);
            if (j == i - 1) {
                for (int k = mn; k > 0; --k)
                    c[k * n + i] = xdiv(xmul(c1, xsub(xmul((double)k, c[(k - 1) * n + i - 1]),
                                                      xmul(c5, c[k * n + i - 1]))), c2);
                c[i] = xdiv(xmul(xmul(-c1, c5), c[i - 1]), c2);
            }
            for (int k = mn; k > 0; --k)
                c[k * n + j] = xdiv(xsub(xmul(c4, c[k * n + j]), xmul((double)k, c[(k - 1) * n + j])), c3);
            c[j] = xdiv(xmul(c4, c[j]), c3);
        }
        c1 = c2;
    }
    double *o = out + b * (int64_t)(m + 1) * n;
    for (int i = 0; i < (m + 1) * n; ++i) o[i] = c[i];
}

// The same recursion with one warp per item, lane j owning column j of the
// table (small batches: a single stencil geometry's n tables).  The column
// updates of one i are independent across j, and the new column i reads
// column i-1 before lane i-1 updates it, exactly as the serial loop does, so
// every value sees the same operations in the same order (bit-identical to
// fornberg_kernel); the division chain shrinks from O(n^2 m) to O(n m).
__global__ void fornberg_warp_kernel(const double *__restrict__ z, const double *__restrict__ x,
                                     int64_t xs, int n, int m, int64_t B, double *__restrict__ out)
{
    extern __shared__ double fw_sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    if (b >= B) return;
    double *c = fw_sm + (size_t)wib * (m + 1) * 32;          // c[k*32 + j]
    const double *xb = x + b * xs;
    const double zz = z[b];
    for (int k = 0; k <= m; ++k) c[k * 32 + lane] = (k == 0 && lane == 0) ? 1.0 : 0.0;
    const double xl = lane < n ? xb[lane] : 0.0;
    double c1 = 1.0;
    double c4 = xsub(xb[0], zz);
    __syncwarp();
    for (int i = 1; i < n; ++i) {
        const int mn = i < m ? i : m;
        const double xi = xb[i];
        const double c5 = c4;
        c4 = xsub(xi, zz);
        double c2 = 1.0;
        for (int j = 0; j < i; ++j) c2 = xmul(c2, xsub(xi, xb[j]));
        // lane i: the new column from the old column i-1
        double nc[LMEP_MAX_N];
        if (lane == i) {
            for (int k = mn; k > 0; --k)
                nc[k] = xdiv(xmul(c1, xsub(xmul((double)k, c[(k - 1) * 32 + i - 1]),
                                         xmul(c5, c[k * 32 + i - 1]))), c2);
            nc[0] = xdiv(xmul(xmul(-c1, c5), c[i - 1]), c2);
        }
        __syncwarp();
        if (lane < i) {
            const double c3 = xsub(xi, xl);
            for (int k = mn; k > 0; --k)
                c[k * 32 + lane] = xdiv(xsub(xmul(c4, c[k * 32 + lane]), xmul((double)k, c[(k - 1) * 32 + lane])), c3);
            c[lane] = xdiv(xmul(c4, c[lane]), c3);
        } else if (lane == i) {
            for (int k = mn; k >= 0; --k) c[k * 32 + i] = nc[k];
        }
        __syncwarp();
        c1 = c2;
    }
    double *o = out + b * (int64_t)(m + 1) * n;
    if (lane < n)
        for (int k = 0; k <= m; ++k) o[k * n + lane] = c[k * 32 + lane];
}

// --------------------------------------------------------------------------
// Warp-level dense matrix kernels on padded shared-memory tiles.
// --------------------------------------------------------------------------
template <int DP>
struct Tile {
    static constexpr int LD = DP + 1;
    static constexpr int G = 32 / DP;     // row groups
    static constexpr int E = DP / G;      // owned entries per lane
    static constexpr int SZ = DP * LD;    // doubles per matrix
    static constexpr int NBUF = 8;        // matrices per warp
    static constexpr int NVEC = 2;        // DP-vectors per warp (balance scale, scratch)
    static constexpr int WARP_DOUBLES = NBUF * SZ + NVEC * DP;
};

template <int DP>
__device__ __forceinline__ void mat_mul(const double *__restrict__ A, const double *__restrict__ B,
                                        double *__restrict__ C, int d, int lane)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    double acc[T::E];
#pragma unroll
    for (int j = 0; j < T::E; ++j) acc[j] = 0.0;
#pragma unroll 4
    for (int k = 0; k < d; ++k) {
        const double b = B[k * T::LD + c];
#pragma unroll
        for (int j = 0; j < T::E; ++j) acc[j] = fma(A[(g + T::G * j) * T::LD + k], b, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < T::E; ++j) C[(g + T::G * j) * T::LD + c] = acc[j];
    __syncwarp();
}

// max_j sum_i |M[i][j]|  (exact 1-norm, scipy _onenorm for small matrices)
template <int DP>
__device__ __forceinline__ double one_norm(const double *M, int d, int lane)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < T::E; ++j) {
        const int r = g + T::G * j;
        if (r < d && c < d) s += fabs(M[r * T::LD + c]);
    }
#pragma unroll
    for (int o = DP; o < 32; o <<= 1) s += __shfl_xor_sync(FULL, s, o);
#pragma unroll
    for (int o = 1; o < DP; o <<= 1) s = fmax(s, __shfl_xor_sync(FULL, s, o));
    return s;
}

// || (|scale*M|)^p ||_1 by p products v <- |scale*M|^T v from v = 1
// (scipy _onenorm_matrix_power_nnm).  v_i lives in lane i (i < DP).
template <int DP>
__device__ double abs_power_norm(const double *M, int d, int p, double scale, int lane)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    double v = (c < d) ? 1.0 : 0.0;
    for (int it = 0; it < p; ++it) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const double vr = __shfl_sync(FULL, v, r);
            if (r < d && c < d) s += fabs(M[r * T::LD + c] * scale) * vr;
        }
#pragma unroll
        for (int o = DP; o < 32; o <<= 1) s += __shfl_xor_sync(FULL, s, o);
        v = s;
    }
    double mx = (c < d) ? v : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    return mx;
}

// Incremental v_p = (|A|^T)^p 1 (v lives in lane c): ||(|A|)^p||_1 = max_c v_p[c].
// The ell(m) tests for m = 3, 5, 7, 9 need p = 7, 11, 15, 19 and share one
// iteration instead of restarting (scipy _onenorm_matrix_power_nnm each time).
template <int DP>
struct AbsPowerIter {
    double v;
    int p;
    __device__ void init(int d, int lane) { v = (lane % DP < d) ? 1.0 : 0.0; p = 0; }
    __device__ double norm(const double *M, int d, int target, int lane)
    {
        using T = Tile<DP>;
        const int c = lane % DP, g = lane / DP;
        for (; p < target; ++p) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < T::E; ++j) {
                const int r = g + T::G * j;
                const double vr = __shfl_sync(FULL, v, r);
                if (r < d && c < d) s += fabs(M[r * T::LD + c]) * vr;
            }
#pragma unroll
            for (int o = DP; o < 32; o <<= 1) s += __shfl_xor_sync(FULL, s, o);
            v = s;
        }
        double mx = (c < d) ? v : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        return mx;
    }
};

__device__ __forceinline__ int ell_from(double nrm, double onenorm_A, double scale, int m)
{
    double cm;
    switch (m) {
    case 3: cm = 100800.; break;
    case 5: cm = 10059033600.; break;
    case 7: cm = 4487938430976000.; break;
    case 9: cm = 5914384781877411840000.; break;
    default: cm = 113250775606021113483283660800000000.; break;
    }
    if (nrm == 0.0) return 0;
    const double alpha = nrm / (onenorm_A * scale * cm);
    const double v = ceil(log2(alpha / 0x1p-53) / (2 * m));
    return v > 0.0 ? (int)v : 0;
}

// scipy _ell: extra squarings demanded by the backward-error bound of degree m.
template <int DP>
__device__ int ell(const double *A, int d, int m, double scale, double onenorm_A, int lane)
{
    double cm;
    switch (m) {
    case 3: cm = 100800.; break;
    case 5: cm = 10059033600.; break;
    case 7: cm = 4487938430976000.; break;
    case 9: cm = 5914384781877411840000.; break;
    default: cm = 113250775606021113483283660800000000.; break;
    }
    const double u = 0x1p-53;
    const double nrm = abs_power_norm<DP>(A, d, 2 * m + 1, scale, lane);
    if (nrm == 0.0) return 0;
    const double alpha = nrm / (onenorm_A * scale * cm);
    const double v = ceil(log2(alpha / u) / (2 * m));
    return v > 0.0 ? (int)v : 0;
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// Diagonal balancing before the exponential (expm.py:27-39 balances with
// LAPACK dgebal, job 'S').  Any diagonal similarity by powers of two is exact,
// so the balancing only has to shrink the norm; the result of the exponential
// does not depend on which balancing is chosen beyond rounding.  dgebal sweeps
// the columns one after another (Gauss-Seidel order), which costs d dependent
// warp reductions per sweep; here every lane i evaluates dgebal's acceptance
// test for its own row/column pair simultaneously (Jacobi order, Osborne's
// iteration), with the power-of-two factor from integer exponent arithmetic:
//   f = 2^k with k chosen as dgebal's loops would, from ||col i||, ||row i||
//   accept if ||col i|| f + ||row i|| / f < 0.95 (||col i|| + ||row i||).
// Sweeps stop when no lane changes (at most 12).  Returns false on NaN.
__device__ __forceinline__ int exp2i(double x)      // floor(log2 x) for normal x > 0
{
    return ((__double2hiint(x) >> 20) & 0x7ff) - 1023;
}
__device__ __forceinline__ double pow2(int k)       // 2^k, |k| < 1000
{
    return __hiloint2double((k + 1023) << 20, 0);
}

template <int DP>
__device__ bool balance(double *A, double *scale, int d, int lane)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    double my_scale = 1.0;          // scale of row/column `lane`
    for (int sweep = 0; sweep < 12; ++sweep) {
        double c2 = 0.0, r2 = 0.0;
        if (lane < d) {
            for (int k = 0; k < d; ++k) {
                const double ce = A[k * T::LD + lane], re = A[lane * T::LD + k];
                c2 = fma(ce, ce, c2);
                r2 = fma(re, re, r2);
            }
        }
        if (isnan(c2 + r2)) return false;
        int k = 0;
        if (lane < d && c2 > 1e-280 && r2 > 1e-280 && c2 < 1e280 && r2 < 1e280) {
            const double cn = sqrt(c2), rn = sqrt(r2);
            // dgebal: while (c < r/2) {c*=2; r/=2}  /  while (c/2 >= r) {c/=2; r*=2}
            int kk = (exp2i(rn) - exp2i(cn)) / 2;
            while (cn * pow2(2 * kk + 1) < rn) ++kk;
            while (kk > 0 && !(cn * pow2(2 * kk - 1) < rn)) --kk;
            if (kk <= 0) {
                kk = 0;
                while (cn * pow2(-(2 * (-kk) + 1)) >= rn) --kk;
                while (kk < 0 && !(cn * pow2(-(2 * (-kk) - 1)) >= rn)) ++kk;
            }
            const double f = pow2(kk);
            if (kk != 0 && cn * f + rn / f < 0.95 * (cn + rn)) k = kk;
        }
        if (!__any_sync(FULL, k != 0)) break;
        // A[r][c] <- A[r][c] * f_c / f_r  (row r divided by f_r, column c times f_c)
        my_scale *= pow2(k);
        const int kc = __shfl_sync(FULL, k, c);
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const int kr = __shfl_sync(FULL, k, r);
            if (r < d && c < d && kc != kr) A[r * T::LD + c] *= pow2(kc - kr);
        }
        __syncwarp();
    }
    if (lane < DP) scale[lane] = my_scale;
    __syncwarp();
    return true;
}

// Solve Q X = P in place (X overwrites P) by Gaussian elimination with partial
// pivoting (first maximal pivot, LAPACK idamax).  Returns false if singular.
template <int DP>
__device__ bool lu_solve(double *Q, double *P, double *inv_piv, int d, int lane)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    for (int k = 0; k < d; ++k) {
        // pivot: first maximal |Q[i][k]|, i >= k (LAPACK idamax), exact comparison
        double val = (lane >= k && lane < d) ? fabs(Q[lane * T::LD + k]) : -1.0;
        int idx = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, val, o);
            const int oi = __shfl_xor_sync(FULL, idx, o);
            if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
        }
        if (!(val > 0.0)) return false;
        if (idx != k) {
            if (lane < d) {
                double t = Q[k * T::LD + lane];
                Q[k * T::LD + lane] = Q[idx * T::LD + lane];
                Q[idx * T::LD + lane] = t;
                t = P[k * T::LD + lane];
                P[k * T::LD + lane] = P[idx * T::LD + lane];
                P[idx * T::LD + lane] = t;
            }
            __syncwarp();
        }
        const double inv = 1.0 / Q[k * T::LD + k];
        if (lane == 0) inv_piv[k] = inv;
        const double qk = (c < d) ? Q[k * T::LD + c] : 0.0;
        const double pk = (c < d) ? P[k * T::LD + c] : 0.0;
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            if (r > k && r < d && c < d) {
                const double l = Q[r * T::LD + k] * inv;
                if (c > k) Q[r * T::LD + c] -= l * qk;
                P[r * T::LD + c] -= l * pk;
            }
        }
        __syncwarp();
    }
    for (int k = d - 1; k >= 0; --k) {
        const double x = (c < d) ? P[k * T::LD + c] / Q[k * T::LD + k] : 0.0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            if (c < d) {
                if (r < k) P[r * T::LD + c] -= Q[r * T::LD + k] * x;
                else if (r == k) P[r * T::LD + c] = x;
            }
        }
        __syncwarp();
    }
    return true;
}

// Pade coefficients b_0..b_m (AMH 2009 / scipy).
__constant__ double kB3[4] = {120., 60., 12., 1.};
__constant__ double kB5[6] = {30240., 15120., 3360., 420., 30., 1.};
__constant__ double kB7[8] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.};
__constant__ double kB9[10] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                               2162160., 110880., 3960., 90., 1.};
__constant__ double kB13[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                                1187353796428800., 129060195264000., 10559470521600.,
                                670442572800., 33522128640., 1323241920., 40840800., 960960.,
                                16380., 182., 1.};

// exp(A) for the d x d matrix in buf[0] (padded with zeros).  Returns the
// buffer index holding the result (-1 on non-finite / singular).  *mo, *so get
// the Pade degree and the number of squarings.  Follows oracle/lmep_oracle.c
// orc_expm (balance -> AMH 2009 Algorithm 6.1 with exact norms -> unbalance).
template <int DP>
__device__ int warp_expm(double *buf, double *scale, int d, int lane, int *mo, int *so)
{
    using T = Tile<DP>;
    const int c = lane % DP, g = lane / DP;
    double *M[T::NBUF];
#pragma unroll
    for (int q = 0; q < T::NBUF; ++q) M[q] = buf + q * T::SZ;
    double *A = M[0];

    // finiteness guard (expm.py:35-36)
    bool fin = true;
#pragma unroll
    for (int j = 0; j < T::E; ++j) {
        const int r = g + T::G * j;
        if (r < d && c < d) fin &= (bool)isfinite(A[r * T::LD + c]);
    }
    if (!__all_sync(FULL, fin)) return -1;
    if (!balance<DP>(A, scale, d, lane)) return -1;

    double *A2 = M[1], *A4 = M[2], *A6 = M[3], *A8 = M[4];
    double *U = M[5], *V = M[6], *W = M[7];
    mat_mul<DP>(A, A, A2, d, lane);
    mat_mul<DP>(A2, A2, A4, d, lane);
    mat_mul<DP>(A4, A2, A6, d, lane);
    // Degree selection (AMH 2009 Alg. 6.1 as scipy implements it).  The tests
    // eta < theta_m on d_k = ||A^k||^(1/k) are evaluated as ||A^k|| < theta_m^k
    // (no fractional powers); roots are taken only on the degree-13 branch.
    const double n4 = one_norm<DP>(A4, d, lane);
    const double n6 = one_norm<DP>(A6, d, lane);
    const double nA = one_norm<DP>(A, d, lane);
    constexpr double t3 = 1.495585217958292e-002, t5 = 2.539398330063230e-001;
    constexpr double t7 = 9.504178996162932e-001, t9 = 2.097847961257068e+000;
    constexpr double t3_4 = t3 * t3 * t3 * t3, t3_6 = t3_4 * t3 * t3;
    constexpr double t5_4 = t5 * t5 * t5 * t5, t5_6 = t5_4 * t5 * t5;
    constexpr double t7_6 = t7 * t7 * t7 * t7 * t7 * t7, t7_8 = t7_6 * t7 * t7;
    constexpr double t9_6 = t9 * t9 * t9 * t9 * t9 * t9, t9_8 = t9_6 * t9 * t9;
    AbsPowerIter<DP> pw;
    pw.init(d, lane);
    int m = 13, s = 0;
    if (n4 < t3_4 && n6 < t3_6 && ell_from(pw.norm(A, d, 7, lane), nA, 1.0, 3) == 0) {
        m = 3;
    } else if (n4 < t5_4 && n6 < t5_6 && ell_from(pw.norm(A, d, 11, lane), nA, 1.0, 5) == 0) {
        m = 5;
    } else {
        mat_mul<DP>(A6, A2, A8, d, lane);
        const double n8 = one_norm<DP>(A8, d, lane);
        if (n6 < t7_6 && n8 < t7_8 && ell_from(pw.norm(A, d, 15, lane), nA, 1.0, 7) == 0) {
            m = 7;
        } else if (n6 < t9_6 && n8 < t9_8 && ell_from(pw.norm(A, d, 19, lane), nA, 1.0, 9) == 0) {
            m = 9;
        } else {
            const double d6 = pow(n6, 1.0 / 6.0), d8 = pow(n8, 0.125);
            const double eta3 = fmax(d6, d8);
            mat_mul<DP>(A4, A6, W, d, lane);  // A10, only for its norm
            const double d10 = pow(one_norm<DP>(W, d, lane), 0.1);
            const double eta4 = fmax(d8, d10);
            const double eta5 = fmin(eta3, eta4);
            if (eta5 == 0.0) s = 0;
            else {
                const double v = ceil(log2(eta5 / 4.25));
                s = v > 0.0 ? (int)v : 0;
            }
            s += ell<DP>(A, d, 13, ldexp(1.0, -s), nA, lane);
            m = 13;
        }
    }

    if (m != 13) {
        const double *b = m == 3 ? kB3 : m == 5 ? kB5 : m == 7 ? kB7 : kB9;
        const double *P2[4] = {A2, A4, A6, A8};
        const int np = (m - 1) / 2;
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            double w = 0.0, v = 0.0;
            if (r < d && c < d) {
                for (int q = np; q >= 1; --q) {
                    const double pe = P2[q - 1][r * T::LD + c];
                    w = w + b[2 * q + 1] * pe;
                    v = v + b[2 * q] * pe;
                }
                if (r == c) { w += b[1]; v += b[0]; }
            }
            W[r * T::LD + c] = w;
            V[r * T::LD + c] = v;
        }
        __syncwarp();
        mat_mul<DP>(A, W, U, d, lane);
    } else {
        const double s1 = ldexp(1.0, -s), s2 = ldexp(1.0, -2 * s), s4 = ldexp(1.0, -4 * s),
                     s6 = ldexp(1.0, -6 * s);
        double *Bm = A8;
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const int e = r * T::LD + c;
            Bm[e] = A[e] * s1;
            A2[e] *= s2;
            A4[e] *= s4;
            A6[e] *= s6;
            W[e] = kB13[13] * A6[e] + kB13[11] * A4[e] + kB13[9] * A2[e];
        }
        __syncwarp();
        mat_mul<DP>(A6, W, U, d, lane);
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const int e = r * T::LD + c;
            double u = U[e] + kB13[7] * A6[e] + kB13[5] * A4[e] + kB13[3] * A2[e];
            if (r == c && r < d) u += kB13[1];
            U[e] = (r < d && c < d) ? u : 0.0;
        }
        __syncwarp();
        mat_mul<DP>(Bm, U, W, d, lane);   // U <- Bm * U  (result in W)
        double *t = U; U = W; W = t;
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const int e = r * T::LD + c;
            W[e] = kB13[12] * A6[e] + kB13[10] * A4[e] + kB13[8] * A2[e];
        }
        __syncwarp();
        mat_mul<DP>(A6, W, V, d, lane);
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            const int e = r * T::LD + c;
            double v = V[e] + kB13[6] * A6[e] + kB13[4] * A4[e] + kB13[2] * A2[e];
            if (r == c && r < d) v += kB13[0];
            V[e] = (r < d && c < d) ? v : 0.0;
        }
        __syncwarp();
    }
    // P = U + V (into U), Q = V - U (into V); solve Q X = P.
#pragma unroll
    for (int j = 0; j < T::E; ++j) {
        const int r = g + T::G * j;
        const int e = r * T::LD + c;
        const double u = U[e], v = V[e];
        U[e] = u + v;
        V[e] = -u + v;
    }
    __syncwarp();
    if (!lu_solve<DP>(V, U, scale + DP, d, lane)) return -1;
    double *X = U, *Y = V;
    for (int q = 0; q < s; ++q) {
        mat_mul<DP>(X, X, Y, d, lane);
        double *t = X; X = Y; Y = t;
    }
    // undo balancing: E = D^-1 ... scipy form E * (d_i / d_j)  (expm.py:39)
    bool ok = true;
    const double inv_sc = 1.0 / scale[c];          // scales are powers of two: exact
#pragma unroll
    for (int j = 0; j < T::E; ++j) {
        const int r = g + T::G * j;
        if (r < d && c < d) {
            const double e = X[r * T::LD + c] * (scale[r] * inv_sc);
            X[r * T::LD + c] = e;
            ok &= (bool)isfinite(e);
        }
    }
    __syncwarp();
    *mo = m;
    *so = s;
    if (!__all_sync(FULL, ok)) return -1;
    return (int)((X - buf) / T::SZ);
}



template <int DP, int WPB>
__global__ void __launch_bounds__(32 * WPB) harvest_kernel(const HarvestParams P)
{
    using T = Tile<DP>;
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * WPB + warp;
    if (b >= P.B) return;  // warp-uniform; the kernel has no block barriers
    double *buf = smem + (size_t)warp * T::WARP_DOUBLES;
    double *scale = buf + T::NBUF * T::SZ;
    double *A = buf;
    const int d = P.d;
    const int c = lane % DP, g = lane / DP;

    int row = 0;
    uint64_t fz = 0;
    if (P.mode == 0) {
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            A[r * T::LD + c] = (r < d && c < d) ? P.Ain[(b * d + r) * d + c] : 0.0;
        }
    } else {
        const int n = P.n;
        row = P.rows ? P.rows[b] : P.row_default;
        fz = P.frozen ? P.frozen[b] : P.frozen_default;
        const double dt = P.delta_t;
        // A[j][i] = dt * L'[i][j] for i, j < n (transposed operator block);
        // lane (g, c) builds entries (r, c) of A, i.e. L[c][r].
        const double *tab = nullptr, *cf = nullptr;
        double cz = 0.0;
        if (P.mode == 1) {
            const int ti = P.table_idx ? P.table_idx[b] : 0;
            tab = P.tables + (size_t)ti * P.nterms * n * n;
            cf = P.coef + b * P.coef_stride;
            cz = P.c0 ? P.c0[b * P.c0_stride] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            double a = 0.0;
            if (r < n && c < n) {
                const int i = c, jj = r;  // L[i][jj]
                double l;
                if (P.mode == 1) {
                    // localop.py:120-127: L[i] += c_k * table[k] in term order, then c0*I
                    const double *cfi = cf;
                    double czi = cz;
                    if (P.map_on) {          // row-scaled: row i reads node m_i
                        const int64_t mi = coef_node(P, b, row, i);
                        cfi = P.coef + mi * P.coef_stride;
                        czi = P.c0 ? P.c0[mi * P.c0_stride] : 0.0;
                    }
                    l = 0.0;
                    for (int t = 0; t < P.nterms; ++t)
                        l = xadd(l, xmul(cfi[t], tab[(t * n + i) * n + jj]));
                    if (i == jj && czi != 0.0) l = xadd(l, czi);
                } else {
                    l = P.L[(b * n + i) * n + jj];
                }
                if ((fz >> i) & 1ull) l = 0.0;   // harvest.py:116-117
                a = xmul(dt, l);
            } else if (r < d && c < d) {
                // augmentation: column n carries dt*e_row, then the dt-shift chain
                if (c == n && r == row) a = dt;
                else if (r >= n && c == r + 1) a = dt;
            }
            A[r * T::LD + c] = a;
        }
    }
    __syncwarp();

    int st = LMEP_OK, m = 0, s = 0, res = 0;
    if (d == 1) {
        if (lane == 0) {
            const double e = exp(A[0]);
            A[0] = e;
        }
        __syncwarp();
        if (!isfinite(A[0])) st = LMEP_NONFINITE;
    } else {
        res = warp_expm<DP>(buf, scale, d, lane, &m, &s);
        if (res < 0) { st = LMEP_NONFINITE; res = 0; }
    }
    const double *E = buf + res * T::SZ;
    if (P.status && lane == 0) P.status[b] = st;
    if (P.ms && lane == 0) P.ms[b] = m | (s << 8);

    if (P.mode == 0) {
#pragma unroll
        for (int j = 0; j < T::E; ++j) {
            const int r = g + T::G * j;
            if (r < d && c < d) P.out[(b * d + r) * d + c] = E[r * T::LD + c];
        }
        return;
    }
    // Row extraction (harvest.py:119-120) in the transposed reduced form:
    // w_lin[i] = E[i][row]; w_phi_q[i] = E[i][n+q-1] (zero on frozen rows).
    const int n = P.n, sd = P.s;
    for (int e = lane; e < sd * n; e += 32) {
        const int q = e / n, i = e % n;
        double w;
        if (q == 0) w = E[i * T::LD + row];
        else w = ((fz >> i) & 1ull) ? 0.0 : E[i * T::LD + n + q - 1];
        if (P.layout == 0) P.out[(b * sd + q) * n + i] = w;
        else P.out[((int64_t)q * n + i) * P.out_ld + b] = w;
    }
}

template <int DP, int WPB>
static int launch_harvest(const HarvestParams &P, cudaStream_t st)
{
    using T = Tile<DP>;
    const size_t shm = (size_t)WPB * T::WARP_DOUBLES * sizeof(double);
    auto kern = harvest_kernel<DP, WPB>;
    static std::atomic<uint64_t> attr{0};
    const int dev = current_device();
    if (!done_on_device(attr, dev)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        mark_device(attr, dev);
    }
    const int64_t blocks = (P.B + WPB - 1) / WPB;
    if (blocks > 0x7fffffffLL) return LMEP_INVALID_CONFIG;
    kern<<<(unsigned)blocks, 32 * WPB, shm, st>>>(P);
    return launch_status("harvest_kernel");
}

int mv_lanes_override() { return device_settings().mv_lanes.load(); }

// *half_done (nullable) reports whether the launched kernel also wrote the
// half-step set P.half_out (only the per-item expm-multiply kernel does)
static int dispatch_harvest(const HarvestParams &Pin, cudaStream_t st, bool *half_done = nullptr)
{
    if (half_done) *half_done = false;
    if (Pin.B == 0) {
        if (half_done) *half_done = true;
        return LMEP_OK;
    }
    HarvestParams P = Pin;
    P.half_out = nullptr;
    const DeviceSettings &ds = device_settings();
    const int method = ds.harvest_method.load();
    if (P.mode != 0 && method != 1 && P.d >= 2 && P.d <= 16 && (P.mode == 2 || P.nterms <= 4)) {
        if (method == 0 && ds.mv_lanes.load() == 0 && ds.mvc.load() && harvest_mvc_eligible(P))
            return launch_harvest_mvc(P, st);
        if (method == 0 && harvest_mvb_eligible(P)) return launch_harvest_mvb(P, st);
        if (Pin.half_out && Pin.s >= 2) {
            P.half_out = Pin.half_out;
            if (half_done) *half_done = true;
        }
        return launch_harvest_mv(P, st);
    }
    if (P.d <= 8) return launch_harvest<8, 8>(P, st);
    if (P.d <= 16) return launch_harvest<16, 4>(P, st);
    if (P.d <= 32) return launch_harvest<32, 2>(P, st);
    return LMEP_DIMENSION;
}

}  // namespace lmep

using namespace lmep;

extern "C" int lmep_fornberg(const double *z, const double *x, int64_t x_stride, int n, int m,
                             int64_t B, double *out, void *stream)
{
    if (n < 1 || n > LMEP_MAX_N) return LMEP_DIMENSION;
    if (m < 0 || m > n - 1) return LMEP_ORDER_TOO_HIGH;
    if (B == 0) return LMEP_OK;
    if (B <= 4096) {
        // few tables (one stencil geometry): a warp per item, columns across lanes
        const int wpb = 4;
        const size_t shm = (size_t)wpb * (m + 1) * 32 * sizeof(double);
        fornberg_warp_kernel<<<(unsigned)((B + wpb - 1) / wpb), 32 * wpb, shm, (cudaStream_t)stream>>>(
            z, x, x_stride, n, m, B, out);
        return launch_status("fornberg_warp_kernel");
    }
    const size_t per = (size_t)(m + 1) * n * sizeof(double);
    const int tpb = (int)std::max<size_t>(1, std::min<size_t>(64, (32 * 1024) / per));
    fornberg_kernel<<<(unsigned)((B + tpb - 1) / tpb), tpb, tpb * per, (cudaStream_t)stream>>>(
        z, x, x_stride, n, m, B, out);
    return launch_status("fornberg_kernel");
}

extern "C" int lmep_expm(const double *A, int d, int64_t B, double *E, int32_t *status,
                         int32_t *ms, void *stream)
{
    if (d < 1 || d > LMEP_MAX_DIM) return LMEP_DIMENSION;
    HarvestParams P{};
    P.mode = 0;
    P.d = d;
    P.Ain = A;
    P.B = B;
    P.out_ld = B;
    P.out = E;
    P.status = status;
    P.ms = ms;
    return dispatch_harvest(P, (cudaStream_t)stream);
}

static int harvest_params(HarvestParams &P, int n, int s, int nterms, const double *tables,
                          const int32_t *table_idx, const double *coef, int64_t coef_stride,
                          const double *c0, int64_t c0_stride, const double *L, double delta_t,
                          const int32_t *target_row, int row_default, const uint64_t *frozen,
                          uint64_t frozen_default, int64_t B, int layout, double *w_out,
                          int32_t *status, int32_t *ms, const lmep_coef_map *map, int64_t out_ld);

extern "C" int lmep_harvest_chunk(int n, int s, int nterms, const double *tables,
                                  const int32_t *table_idx, const double *coef,
                                  int64_t coef_stride, const double *c0, int64_t c0_stride,
                                  const double *L, double delta_t, const int32_t *target_row,
                                  int row_default, const uint64_t *frozen,
                                  uint64_t frozen_default, int64_t B, int layout, double *w_out,
                                  int32_t *status, int32_t *ms, const lmep_coef_map *map,
                                  int64_t out_ld, void *stream)
{
    HarvestParams P{};
    const int rc = harvest_params(P, n, s, nterms, tables, table_idx, coef, coef_stride, c0,
                                  c0_stride, L, delta_t, target_row, row_default, frozen,
                                  frozen_default, B, layout, w_out, status, ms, map, out_ld);
    if (rc) return rc;
    return dispatch_harvest(P, (cudaStream_t)stream);
}

// lmep_harvest_ex: the chunk call plus the half-step set and the device flag
extern "C" int lmep_harvest_ex(const lmep_harvest_args *a, void *stream)
{
    if (!a) return LMEP_INVALID_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    HarvestParams P{};
    int rc = harvest_params(P, a->n, a->s, a->nterms, a->tables, a->table_idx, a->coef,
                            a->coef_stride, a->c0, a->c0_stride, a->L, a->delta_t,
                            a->target_row, (int)a->row_default, a->frozen, a->frozen_default, a->B,
                            a->layout, a->w_out, a->status, a->ms, a->map,
                            a->layout == 1 ? a->out_ld : a->B);
    if (rc) return rc;
    if (a->half_out && a->s < 2) return LMEP_INVALID_CONFIG;
    if (a->status_any && !a->status) return LMEP_INVALID_CONFIG;
    P.half_out = a->half_out;
    bool half_done = false;
    rc = dispatch_harvest(P, st, &half_done);
    if (rc) return rc;
    if (a->status_any && (rc = launch_status_or(a->status, a->B, a->status_any, st))) return rc;
    if (a->half_out && !half_done) {
        // the selected kernel emits one set: a second launch at delta_t / 2, s = 2
        HarvestParams H{};
        int32_t *hs = nullptr;
        if (a->status) {
            cudaError_t e = cudaMallocAsync((void **)&hs, sizeof(int32_t) * (a->B > 0 ? a->B : 1), st);
            if (e != cudaSuccess) { set_last_error("cudaMallocAsync", e); return LMEP_CUDA_ERROR; }
        }
        rc = harvest_params(H, a->n, 2, a->nterms, a->tables, a->table_idx, a->coef,
                            a->coef_stride, a->c0, a->c0_stride, a->L, 0.5 * a->delta_t,
                            a->target_row, (int)a->row_default, a->frozen, a->frozen_default, a->B,
                            a->layout, a->half_out, hs, nullptr, a->map,
                            a->layout == 1 ? a->out_ld : a->B);
        if (!rc) rc = dispatch_harvest(H, st);
        if (!rc && hs) {
            rc = launch_status_merge(a->status, hs, a->B, st);
            if (!rc && a->status_any) rc = launch_status_or(hs, a->B, a->status_any, st);
        }
        if (hs) cudaFreeAsync(hs, st);
        if (rc) return rc;
    }
    return LMEP_OK;
}

static int harvest_params(HarvestParams &P, int n, int s, int nterms, const double *tables,
                          const int32_t *table_idx, const double *coef, int64_t coef_stride,
                          const double *c0, int64_t c0_stride, const double *L, double delta_t,
                          const int32_t *target_row, int row_default, const uint64_t *frozen,
                          uint64_t frozen_default, int64_t B, int layout, double *w_out,
                          int32_t *status, int32_t *ms, const lmep_coef_map *map, int64_t out_ld)
{
    if (layout == 1 && out_ld < B) return LMEP_DIMENSION;
    if (s < 1 || s > 6) return LMEP_INVALID_CONFIG;                 // harvest.py:85-86
    if (n < 1 || n > LMEP_MAX_N || n + s - 1 > LMEP_MAX_DIM) return LMEP_DIMENSION;
    if (!target_row && (row_default < 0 || row_default >= n)) return LMEP_DIMENSION;
    if (layout != 0 && layout != 1) return LMEP_INVALID_CONFIG;
    if (!L && nterms > 0 && (!tables || !coef)) return LMEP_INVALID_CONFIG;
    if (nterms < 0 || nterms > 8) return LMEP_INVALID_CONFIG;
    P = HarvestParams{};
    P.mode = L ? 2 : 1;
    P.n = n;
    P.s = s;
    P.d = n + s - 1;
    P.nterms = nterms;
    P.tables = tables;
    P.table_idx = table_idx;
    P.coef = coef;
    P.coef_stride = coef_stride;
    P.c0 = c0;
    P.c0_stride = c0_stride;
    P.L = L;
    P.delta_t = delta_t;
    P.rows = target_row;
    P.row_default = row_default;
    P.frozen = frozen;
    P.frozen_default = frozen_default;
    P.B = B;
    P.out_ld = layout == 1 ? out_ld : B;
    P.layout = layout;
    P.out = w_out;
    P.status = status;
    P.ms = ms;
    if (map) {
        if (L || !coef || map->nnodes < 1) return LMEP_INVALID_CONFIG;
        P.map_on = 1;
        P.map_periodic = map->periodic ? 1 : 0;
        P.map_node0 = map->node0;
        P.map_nnodes = map->nnodes;
    }
    return LMEP_OK;
}

extern "C" int lmep_harvest_mapped(int n, int s, int nterms, const double *tables,
                                   const int32_t *table_idx, const double *coef,
                                   int64_t coef_stride, const double *c0, int64_t c0_stride,
                                   const double *L, double delta_t, const int32_t *target_row,
                                   int row_default, const uint64_t *frozen,
                                   uint64_t frozen_default, int64_t B, int layout, double *w_out,
                                   int32_t *status, int32_t *ms, const lmep_coef_map *map,
                                   void *stream)
{
    return lmep_harvest_chunk(n, s, nterms, tables, table_idx, coef, coef_stride, c0, c0_stride,
                              L, delta_t, target_row, row_default, frozen, frozen_default, B,
                              layout, w_out, status, ms, map, B, stream);
}

extern "C" int lmep_harvest(int n, int s, int nterms, const double *tables,
                            const int32_t *table_idx, const double *coef, int64_t coef_stride,
                            const double *c0, int64_t c0_stride, const double *L, double delta_t,
                            const int32_t *target_row, int row_default, const uint64_t *frozen,
                            uint64_t frozen_default, int64_t B, int layout, double *w_out,
                            int32_t *status, int32_t *ms, void *stream)
{
    return lmep_harvest_mapped(n, s, nterms, tables, table_idx, coef, coef_stride, c0, c0_stride,
                               L, delta_t, target_row, row_default, frozen, frozen_default, B,
                               layout, w_out, status, ms, nullptr, stream);
}

extern "C" int lmep_set_harvest_method(int method)
{
    // 0 auto: constant-table kernel (harvest_mvc.cu) / block-balanced mv
    // (harvest_mvb.cuh) for large single-geometry batches, else the per-item mv
    // (4 lanes per item); 1 pade; 4 per-item mv with 8 lanes for d > 8; 5
    // per-item mv only; 6 / 7 / 8 auto with the block-balanced kernel forced to
    // 8 / 2 / 4 lanes per item (tuning); 9 auto without the constant-table
    // kernel.  (2 / 3 named the retired first-generation kernel.)  Applies to
    // the calling thread's current device.
    // 10 = auto with the constant-table kernel's Taylor series only (no polynomial kernel)
    if (method < 0 || method > 10 || method == 2 || method == 3) return LMEP_INVALID_CONFIG;
    lmep::DeviceSettings &ds = lmep::device_settings();
    ds.mvc.store(method == 0 ? 1 : (method == 10 ? 2 : 0));
    ds.mv_lanes.store((method == 4 || method == 6) ? 8 : (method == 7 ? 2 : (method == 8 ? 4 : 0)));
    if (method == 4) method = 5;
    if (method >= 6) method = 0;   // 6..10
    ds.harvest_method.store(method);
    return LMEP_OK;
}
