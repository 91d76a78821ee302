/*
 * lmep_oracle.c -- CPU restatement of the reference LMEP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2603_15964_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links, imports or executes anything under oracle/.
 *
 * Reference: /root/reference/pkg/src/localexp (Python + numba + scipy).
 * Each function cites the reference file:line it restates.  The matrix
 * exponential lives in third-party scipy (>=1.10 per pyproject.toml:12,
 * 1.18.1 in the build container): scipy.linalg.matrix_balance (LAPACK dgebal,
 * job='S') and scipy.linalg.expm (Al-Mohy & Higham 2009, "A New Scaling and
 * Squaring Algorithm for the Matrix Exponential", Algorithm 6.1 with exact
 * 1-norms for small matrices, theta_13 = 4.25 as in scipy's _expm).  Those
 * published algorithms are restated here from their descriptions; parity is
 * pinned against golden vectors produced by the live reference
 * (tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp (see oracle/Makefile).  FMA
 * contraction is OFF so the stepping loops reproduce numba's (no fastmath,
 * kernels.py:8-9) separate multiply / add roundings bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* status codes shared with include/lmep.h */
#define ORC_OK 0
#define ORC_NONFINITE 1
#define ORC_DIM 2
#define ORC_INVALID 3
#define ORC_ORDER 5
#define ORC_DUPLICATE 6

#define ORC_MAXD 64

/* ------------------------------------------------------------------ */
/* Fornberg weights: localop.py:61-96                                  */
/* c is (m+1) x n row-major: c[k*n + j]                                */
/* ------------------------------------------------------------------ */
int orc_fornberg(double z, const double *x, int n, int m, double *c)
{
    if (m < 0 || m > n - 1) return ORC_ORDER;                 /* localop.py:69-70 */
    if (n > 1) {                                               /* localop.py:71-74 */
        double mx = x[0], mnx = x[0];
        for (int i = 1; i < n; ++i) { if (x[i] > mx) mx = x[i]; if (x[i] < mnx) mnx = x[i]; }
        double spread = mx - mnx;
        /* min gap of the sorted nodes */
        double *s = (double *)malloc(sizeof(double) * n);
        memcpy(s, x, sizeof(double) * n);
        for (int i = 1; i < n; ++i) { double v = s[i]; int j = i - 1; while (j >= 0 && s[j] > v) { s[j + 1] = s[j]; --j; } s[j + 1] = v; }
        double gap = INFINITY;
        for (int i = 1; i < n; ++i) { double g = s[i] - s[i - 1]; if (g < gap) gap = g; }
        free(s);
        if (gap <= 1e-14 * spread) return ORC_DUPLICATE;
    }
    for (int i = 0; i < (m + 1) * n; ++i) c[i] = 0.0;
    c[0] = 1.0;
    double c1 = 1.0;
    double c4 = x[0] - z;
    for (int i = 1; i < n; ++i) {
        int mn = i < m ? i : m;
        double c2 = 1.0;
        double c5 = c4;
        c4 = x[i] - z;
        for (int j = 0; j < i; ++j) {
            double c3 = x[i] - x[j];
            c2 *= c3;
            if (j == i - 1) {
                for (int k = mn; k > 0; --k)
                    c[k * n + i] = c1 * ((double)k * c[(k - 1) * n + i - 1] - c5 * c[k * n + i - 1]) / c2;
                c[i] = -c1 * c5 * c[i - 1] / c2;
            }
            for (int k = mn; k > 0; --k)
                c[k * n + j] = (c4 * c[k * n + j] - (double)k * c[(k - 1) * n + j]) / c3;
            c[j] = c4 * c[j] / c3;
        }
        c1 = c2;
    }
    return ORC_OK;
}

/* local_operator: localop.py:111-128.  terms are (order, coefficient) in the
 * spec's order; L is n x n row-major. */
int orc_local_operator(const double *x, int n, const int *korder, const double *kcoef,
                       int nterms, double *L)
{
    int kmax = 0;
    double c0 = 0.0;
    for (int t = 0; t < nterms; ++t) if (korder[t] > kmax) kmax = korder[t];
    for (int t = 0; t < nterms; ++t) if (korder[t] == 0) { c0 = kcoef[t]; break; }
    if (kmax > n - 1) return ORC_ORDER;
    for (int i = 0; i < n * n; ++i) L[i] = 0.0;
    if (kmax > 0) {
        double *tab = (double *)malloc(sizeof(double) * (kmax + 1) * n);
        for (int i = 0; i < n; ++i) {
            int st = orc_fornberg(x[i], x, n, kmax, tab);
            if (st) { free(tab); return st; }
            for (int t = 0; t < nterms; ++t) {
                int k = korder[t];
                if (k > 0)
                    for (int j = 0; j < n; ++j) L[i * n + j] = L[i * n + j] + kcoef[t] * tab[k * n + j];
            }
        }
        free(tab);
    }
    if (c0 != 0.0)
        for (int i = 0; i < n; ++i) L[i * n + i] = L[i * n + i] + c0;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Balancing: scipy.linalg.matrix_balance(A, permute=False) = LAPACK   */
/* dgebal job 'S' (LAPACK >= 3.5: 2-norms incl. diagonal).  Restated.  */
/* A is d x d row-major, modified in place to D^-1 A D; scale = diag D */
/* ------------------------------------------------------------------ */
static double nrm2_col(const double *A, int d, int j)
{
    double ssq = 0.0, scale = 0.0; /* classic scaled sum of squares */
    for (int i = 0; i < d; ++i) {
        double v = fabs(A[i * d + j]);
        if (v != 0.0) {
            if (scale < v) { ssq = 1.0 + ssq * (scale / v) * (scale / v); scale = v; }
            else ssq += (v / scale) * (v / scale);
        }
    }
    return scale * sqrt(ssq);
}
static double nrm2_row(const double *A, int d, int i)
{
    double ssq = 0.0, scale = 0.0;
    for (int j = 0; j < d; ++j) {
        double v = fabs(A[i * d + j]);
        if (v != 0.0) {
            if (scale < v) { ssq = 1.0 + ssq * (scale / v) * (scale / v); scale = v; }
            else ssq += (v / scale) * (v / scale);
        }
    }
    return scale * sqrt(ssq);
}

int orc_matrix_balance(double *A, int d, double *scale)
{
    const double sclfac = 2.0, factor = 0.95;
    const double sfmin1 = DBL_MIN / (DBL_EPSILON);   /* dlamch('S')/dlamch('P') */
    const double sfmax1 = 1.0 / sfmin1;
    const double sfmin2 = sfmin1 * sclfac;
    const double sfmax2 = 1.0 / sfmin2;
    for (int i = 0; i < d; ++i) scale[i] = 1.0;
    int noconv = 1, sweeps = 0;
    while (noconv) {
        noconv = 0;
        if (++sweeps > 1000) break;
        for (int i = 0; i < d; ++i) {
            double c = nrm2_col(A, d, i);
            double r = nrm2_row(A, d, i);
            double ca = 0.0, ra = 0.0;
            for (int k = 0; k < d; ++k) { double v = fabs(A[k * d + i]); if (v > ca) ca = v; }
            for (int k = 0; k < d; ++k) { double v = fabs(A[i * d + k]); if (v > ra) ra = v; }
            if (c == 0.0 || r == 0.0) continue;
            if (isnan(c + ca + r + ra)) return ORC_NONFINITE;
            double g = r / sclfac, f = 1.0, s = c + r;
            while (c < g && fmax(f, fmax(c, ca)) < sfmax2 && fmin(r, fmin(g, ra)) > sfmin2) {
                f *= sclfac; c *= sclfac; ca *= sclfac; r /= sclfac; g /= sclfac; ra /= sclfac;
            }
            g = c / sclfac;
            while (g >= r && fmax(r, ra) < sfmax2 && fmin(fmin(f, c), fmin(g, ca)) > sfmin2) {
                f /= sclfac; c /= sclfac; g /= sclfac; ca /= sclfac; r *= sclfac; ra *= sclfac;
            }
            if ((c + r) >= factor * s) continue;
            if (f < 1.0 && scale[i] < 1.0) { if (f * scale[i] <= sfmin1) continue; }
            if (f > 1.0 && scale[i] > 1.0) { if (scale[i] >= sfmax1 / f) continue; }
            g = 1.0 / f;
            scale[i] *= f;
            noconv = 1;
            for (int k = 0; k < d; ++k) A[i * d + k] *= g;   /* row i  / f */
            for (int k = 0; k < d; ++k) A[k * d + i] *= f;   /* col i  * f */
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Matrix exponential: AMH 2009 Algorithm 6.1 as scipy implements it   */
/* (exact 1-norms for small orders, theta_13 = 4.25).                  */
/* ------------------------------------------------------------------ */
static void mm(const double *A, const double *B, double *C, int d)
{
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            double acc = 0.0;
            for (int k = 0; k < d; ++k) acc += A[i * d + k] * B[k * d + j];
            C[i * d + j] = acc;
        }
}
static double onenorm(const double *A, int d)
{
    double best = 0.0;
    for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int i = 0; i < d; ++i) s += fabs(A[i * d + j]);
        if (s > best) best = s;
    }
    return best;
}
/* ||(|sA|)^p||_1 via v <- |sA|^T v from ones (scipy _onenorm_matrix_power_nnm);
 * s is an exact power of two applied to every entry. */
static double onenorm_abs_power(const double *A, int d, int p, double scale)
{
    double v[ORC_MAXD], w[ORC_MAXD];
    for (int i = 0; i < d; ++i) v[i] = 1.0;
    for (int it = 0; it < p; ++it) {
        for (int j = 0; j < d; ++j) {
            double s = 0.0;
            for (int i = 0; i < d; ++i) s += fabs(A[i * d + j] * scale) * v[i];
            w[j] = s;
        }
        for (int j = 0; j < d; ++j) v[j] = w[j];
    }
    double mx = 0.0;
    for (int i = 0; i < d; ++i) if (v[i] > mx) mx = v[i];
    return mx;
}
/* scipy _ell: backward-error based extra squarings */
static int ell(const double *A, int d, int m, double scale)
{
    double c;
    switch (m) {
    case 3: c = 100800.; break;
    case 5: c = 10059033600.; break;
    case 7: c = 4487938430976000.; break;
    case 9: c = 5914384781877411840000.; break;
    default: c = 113250775606021113483283660800000000.; break;
    }
    const double u = ldexp(1.0, -53);
    double nrm = onenorm_abs_power(A, d, 2 * m + 1, scale);
    if (nrm == 0.0) return 0;
    double alpha = nrm / (onenorm(A, d) * scale * c);
    double v = ceil(log2(alpha / u) / (2 * m));
    int iv = (int)v;
    return iv > 0 ? iv : 0;
}

/* Solve Q X = P with LU partial pivoting (LAPACK gesv restated). */
static int solve_pq(double *Q, double *P, int d)
{
    int piv[ORC_MAXD];
    for (int k = 0; k < d; ++k) {
        int p = k;
        double best = fabs(Q[k * d + k]);
        for (int i = k + 1; i < d; ++i) { double v = fabs(Q[i * d + k]); if (v > best) { best = v; p = i; } }
        piv[k] = p;
        if (best == 0.0) return ORC_NONFINITE;
        if (p != k)
            for (int j = 0; j < d; ++j) { double t = Q[k * d + j]; Q[k * d + j] = Q[p * d + j]; Q[p * d + j] = t; }
        double inv = 1.0 / Q[k * d + k];
        for (int i = k + 1; i < d; ++i) Q[i * d + k] *= inv;
        for (int i = k + 1; i < d; ++i) {
            double l = Q[i * d + k];
            if (l != 0.0) for (int j = k + 1; j < d; ++j) Q[i * d + j] -= l * Q[k * d + j];
        }
    }
    for (int k = 0; k < d; ++k) if (piv[k] != k)
        for (int j = 0; j < d; ++j) { double t = P[k * d + j]; P[k * d + j] = P[piv[k] * d + j]; P[piv[k] * d + j] = t; }
    for (int j = 0; j < d; ++j) {
        for (int i = 0; i < d; ++i) {          /* forward, unit lower */
            double s = P[i * d + j];
            for (int k = 0; k < i; ++k) s -= Q[i * d + k] * P[k * d + j];
            P[i * d + j] = s;
        }
        for (int i = d - 1; i >= 0; --i) {     /* backward */
            double s = P[i * d + j];
            for (int k = i + 1; k < d; ++k) s -= Q[i * d + k] * P[k * d + j];
            P[i * d + j] = s / Q[i * d + i];
        }
    }
    return ORC_OK;
}

static const double B3[4] = {120., 60., 12., 1.};
static const double B5[6] = {30240., 15120., 3360., 420., 30., 1.};
static const double B7[8] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.};
static const double B9[10] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                              2162160., 110880., 3960., 90., 1.};
static const double B13[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                               1187353796428800., 129060195264000., 10559470521600.,
                               670442572800., 33522128640., 1323241920., 40840800., 960960.,
                               16380., 182., 1.};

/* E = exp(A) (no balancing).  Returns chosen Pade degree m and squarings s. */
int orc_expm_raw(const double *A, int d, double *E, int *m_out, int *s_out)
{
    if (d < 1 || d > ORC_MAXD) return ORC_DIM;
    if (d == 1) { E[0] = exp(A[0]); if (m_out) *m_out = 0; if (s_out) *s_out = 0; return ORC_OK; }
    size_t sz = (size_t)d * d;
    double *buf = (double *)malloc(sizeof(double) * sz * 10);
    double *A2 = buf, *A4 = buf + sz, *A6 = buf + 2 * sz, *A8 = buf + 3 * sz, *A10 = buf + 4 * sz;
    double *U = buf + 5 * sz, *V = buf + 6 * sz, *T = buf + 7 * sz, *W = buf + 8 * sz, *X = buf + 9 * sz;
    mm(A, A, A2, d);
    mm(A2, A2, A4, d);
    mm(A4, A2, A6, d);
    double d4 = pow(onenorm(A4, d), 0.25);
    double d6 = pow(onenorm(A6, d), 1.0 / 6.0);
    int m = 13, s = 0, have8 = 0;
    double d8 = 0.0, d10 = 0.0;
    double eta1 = fmax(d4, d6);
    if (eta1 < 1.495585217958292e-002 && ell(A, d, 3, 1.0) == 0) m = 3;
    else if (eta1 < 2.539398330063230e-001 && ell(A, d, 5, 1.0) == 0) m = 5;
    else {
        mm(A6, A2, A8, d); have8 = 1;
        d8 = pow(onenorm(A8, d), 0.125);
        double eta3 = fmax(d6, d8);
        if (eta3 < 9.504178996162932e-001 && ell(A, d, 7, 1.0) == 0) m = 7;
        else if (eta3 < 2.097847961257068e+000 && ell(A, d, 9, 1.0) == 0) m = 9;
        else {
            mm(A4, A6, A10, d);
            d10 = pow(onenorm(A10, d), 0.1);
            double eta4 = fmax(d8, d10);
            double eta5 = fmin(eta3, eta4);
            if (eta5 == 0.0) s = 0;
            else { double v = ceil(log2(eta5 / 4.25)); s = v > 0 ? (int)v : 0; }
            s += ell(A, d, 13, ldexp(1.0, -s));
            m = 13;
        }
    }
    (void)have8;
    /* U, V */
    if (m == 3 || m == 5 || m == 7 || m == 9) {
        const double *b = m == 3 ? B3 : m == 5 ? B5 : m == 7 ? B7 : B9;
        const double *P2[4] = {A2, A4, A6, A8};
        /* W = b[m] A_{m-1} + ... + b[3] A2 + b[1] I ; V = b[m-1] A_{m-1} + ... + b[2] A2 + b[0] I */
        int np = (m - 1) / 2;
        for (size_t i = 0; i < sz; ++i) { W[i] = 0.0; V[i] = 0.0; }
        for (int q = np; q >= 1; --q) {
            const double *Pw = P2[q - 1];
            for (size_t i = 0; i < sz; ++i) {
                W[i] = W[i] + b[2 * q + 1] * Pw[i];
                V[i] = V[i] + b[2 * q] * Pw[i];
            }
        }
        for (int i = 0; i < d; ++i) { W[i * d + i] += b[1]; V[i * d + i] += b[0]; }
        mm(A, W, U, d);
    } else {
        double s1 = ldexp(1.0, -s), s2 = ldexp(1.0, -2 * s), s4 = ldexp(1.0, -4 * s), s6 = ldexp(1.0, -6 * s);
        double *Bm = X;
        for (size_t i = 0; i < sz; ++i) { Bm[i] = A[i] * s1; A2[i] *= s2; A4[i] *= s4; A6[i] *= s6; }
        for (size_t i = 0; i < sz; ++i) W[i] = B13[13] * A6[i] + B13[11] * A4[i] + B13[9] * A2[i];
        mm(A6, W, U, d);                 /* U2 */
        for (size_t i = 0; i < sz; ++i) U[i] = U[i] + B13[7] * A6[i] + B13[5] * A4[i] + B13[3] * A2[i];
        for (int i = 0; i < d; ++i) U[i * d + i] += B13[1];
        mm(Bm, U, T, d);                 /* U */
        memcpy(U, T, sizeof(double) * sz);
        for (size_t i = 0; i < sz; ++i) W[i] = B13[12] * A6[i] + B13[10] * A4[i] + B13[8] * A2[i];
        mm(A6, W, V, d);                 /* V2 */
        for (size_t i = 0; i < sz; ++i) V[i] = V[i] + B13[6] * A6[i] + B13[4] * A4[i] + B13[2] * A2[i];
        for (int i = 0; i < d; ++i) V[i * d + i] += B13[0];
    }
    /* P = U + V, Q = -U + V ; solve Q X = P */
    for (size_t i = 0; i < sz; ++i) { T[i] = U[i] + V[i]; W[i] = -U[i] + V[i]; }
    int st = solve_pq(W, T, d);
    if (st) { free(buf); return st; }
    for (int q = 0; q < s; ++q) { mm(T, T, X, d); memcpy(T, X, sizeof(double) * sz); }
    memcpy(E, T, sizeof(double) * sz);
    free(buf);
    if (m_out) *m_out = m;
    if (s_out) *s_out = s;
    return ORC_OK;
}

static int all_finite(const double *a, size_t n)
{
    for (size_t i = 0; i < n; ++i) if (!isfinite(a[i])) return 0;
    return 1;
}

/* expm.py:24-42: finiteness guard, balance (permute=False), expm, unbalance */
int orc_expm(const double *A, int d, double *E, int *m_out, int *s_out)
{
    if (d < 1 || d > ORC_MAXD) return ORC_DIM;
    size_t sz = (size_t)d * d;
    if (!all_finite(A, sz)) return ORC_NONFINITE;
    double *B = (double *)malloc(sizeof(double) * sz);
    double scale[ORC_MAXD];
    memcpy(B, A, sizeof(double) * sz);
    int st = orc_matrix_balance(B, d, scale);
    if (!st) st = orc_expm_raw(B, d, E, m_out, s_out);
    free(B);
    if (st) return st;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) E[i * d + j] = E[i * d + j] * (scale[i] / scale[j]);
    if (!all_finite(E, sz)) return ORC_NONFINITE;
    return ORC_OK;
}

/* harvest.py:82-94 */
int orc_build_augmented(const double *L, int n, int s, double *A)
{
    if (s < 1 || s > 6) return ORC_INVALID;
    int D = s * n;
    for (int i = 0; i < D * D; ++i) A[i] = 0.0;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) A[i * D + j] = L[i * n + j];
    for (int b = 0; b < s - 1; ++b)
        for (int i = 0; i < n; ++i) A[(b * n + i) * D + (b + 1) * n + i] = 1.0;
    return ORC_OK;
}

/* harvest.py:97-121 (reference block form).  frozen: bitmask over rows.
 * w is s x n: w[0] = w_lin, w[j] = raw dt^j phi_j row. */
int orc_harvest_phi(const double *L, int n, double dt, int s, int row, uint64_t frozen,
                    double *w, int *m_out, int *s_out)
{
    if (row < 0 || row >= n) return ORC_DIM;
    if (s < 1 || s > 6) return ORC_INVALID;
    int D = s * n;
    if (D > ORC_MAXD) return ORC_DIM;
    double *A = (double *)malloc(sizeof(double) * D * D);
    double *E = (double *)malloc(sizeof(double) * D * D);
    orc_build_augmented(L, n, s, A);
    for (int j = 0; j < n; ++j) if ((frozen >> j) & 1ull)
        for (int k = 0; k < D; ++k) A[j * D + k] = 0.0;
    for (int i = 0; i < D * D; ++i) A[i] = dt * A[i];
    int st = orc_expm(A, D, E, m_out, s_out);
    if (!st)
        for (int b = 0; b < s; ++b)
            for (int j = 0; j < n; ++j) w[b * n + j] = E[row * D + b * n + j];
    free(A); free(E);
    return st;
}

/* Reduced transposed (n+p) augmentation (the CUDA kernel's algorithm, not
 * the reference's).  exp(dt*[[L'^T, e_r, 0],[0, 0, J]]): column r of the
 * top-left block is w_lin, column n+j-1 is the raw dt^j phi_j row; frozen
 * entries of the phi rows are zeroed (the reference zeroes the identity
 * block's frozen rows).  Kept for cross-checking the kernel's formulation. */
int orc_harvest_phi_reduced(const double *L, int n, double dt, int s, int row, uint64_t frozen,
                            double *w, int *m_out, int *s_out)
{
    if (row < 0 || row >= n) return ORC_DIM;
    if (s < 1 || s > 6) return ORC_INVALID;
    int p = s - 1, D = n + p;
    if (D > ORC_MAXD) return ORC_DIM;
    double *A = (double *)calloc((size_t)D * D, sizeof(double));
    double *E = (double *)malloc(sizeof(double) * D * D);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            A[j * D + i] = ((frozen >> i) & 1ull) ? 0.0 : dt * L[i * n + j];
    if (p >= 1) A[row * D + n] = dt;
    for (int q = 0; q + 1 < p; ++q) A[(n + q) * D + n + q + 1] = dt;
    int st = orc_expm(A, D, E, m_out, s_out);
    if (!st) {
        for (int j = 0; j < n; ++j) w[j] = E[j * D + row];
        for (int b = 1; b < s; ++b)
            for (int j = 0; j < n; ++j)
                w[b * n + j] = ((frozen >> j) & 1ull) ? 0.0 : E[j * D + n + b - 1];
    }
    free(A); free(E);
    return st;
}

/* Per-node variable-coefficient batch (config 5 oracle): L_i = c1_i*D1 +
 * c2_i*D2 from a shared Fornberg table (bit-identical to local_operator with
 * spec ((1,c1),(2,c2))), harvested per node; OpenMP over nodes. */
int orc_harvest_batch_vc(const double *D1, const double *D2, int n, const double *c1,
                         const double *c2, int64_t count, double dt, int s, int row,
                         int reduced, double *w /* [count][s][n] */, int nthreads)
{
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64) reduction(| : err)
#endif
    for (int64_t i = 0; i < count; ++i) {
        double L[ORC_MAXD * ORC_MAXD];
        for (int a = 0; a < n * n; ++a) L[a] = (0.0 + c1[i] * D1[a]) + c2[i] * D2[a];
        int st = reduced ? orc_harvest_phi_reduced(L, n, dt, s, row, 0, w + i * s * n, NULL, NULL)
                         : orc_harvest_phi(L, n, dt, s, row, 0, w + i * s * n, NULL, NULL);
        if (st) err |= 1;
    }
    return err ? ORC_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Stepping: kernels.py                                                */
/* ------------------------------------------------------------------ */
/* kernels.py:23-29 */
void orc_banded_matvec(const double *w, const int64_t *mem, const double *u, double *out,
                       int64_t N, int n)
{
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < N; ++i) {
        double acc = 0.0;
        const double *wi = w + i * n;
        const int64_t *mi = mem + i * n;
        for (int j = 0; j < n; ++j) acc += wi[j] * u[mi[j]];
        out[i] = acc;
    }
}

/* Boundary closure applied where the reference pins (kernels.py:39-41,
 * 93-95, 101-103, 112-114, 129-131).  bc: 0 none, 1 Dirichlet pin,
 * 2 zero-gradient (Neumann) closure u0 = -sum_{j>=1} dl_j u_j / dl_0 and
 * u_{N-1} = -sum_{j<n-1} dr_j u_{N-n+j} / dr_{n-1}. */
typedef struct {
    int bc;
    double lo, hi;
    const double *dl, *dr;
    int nb;
} orc_bc;

static void apply_bc(double *u, int64_t N, const orc_bc *b)
{
    if (b->bc == 1) { u[0] = b->lo; u[N - 1] = b->hi; }
    else if (b->bc == 2) {
        int n = b->nb;
        double acc = 0.0;
        for (int j = 1; j < n; ++j) acc += b->dl[j] * u[j];
        u[0] = -acc / b->dl[0];
        acc = 0.0;
        for (int j = 0; j < n - 1; ++j) acc += b->dr[j] * u[N - n + j];
        u[N - 1] = -acc / b->dr[n - 1];
    }
}

/* kernels.py:33-43 (+ Neumann closure extension) */
void orc_run_linear(const double *w, const int64_t *mem, const double *u0, int64_t N, int n,
                    int64_t steps, int bc, double lo, double hi, const double *dl,
                    const double *dr, double *out)
{
    orc_bc b = {bc, lo, hi, dl, dr, n};
    double *u = (double *)malloc(sizeof(double) * N);
    double *buf = (double *)malloc(sizeof(double) * N);
    memcpy(u, u0, sizeof(double) * N);
    for (int64_t s = 0; s < steps; ++s) {
        orc_banded_matvec(w, mem, u, buf, N, n);
        apply_bc(buf, N, &b);
        double *t = u; u = buf; buf = t;
    }
    memcpy(out, u, sizeof(double) * N);
    free(u); free(buf);
}

/* kernels.py:47-58 */
static void nonlinear(int kind, const double *d1w, const int64_t *mem, const double *u,
                      double *out, double *tmp, int64_t N, int n)
{
    if (kind == 0) {
        for (int64_t i = 0; i < N; ++i) out[i] = 0.0;
    } else if (kind == 1) {
        orc_banded_matvec(d1w, mem, u, tmp, N, n);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t i = 0; i < N; ++i) out[i] = -u[i] * tmp[i];
    } else {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t i = 0; i < N; ++i) out[i] = -u[i] * u[i] * u[i];
    }
}

/* kernels.py:62-132 (+ Neumann closure extension) */
void orc_run_etdrk4(const double *w_full, const double *w_alpha, const double *w_beta,
                    const double *w_gamma, const double *w_half, const double *w_p1h,
                    const double *d1w, const int64_t *mem, int kind, const double *u0,
                    int64_t N, int n, int64_t steps, int bc, double lo, double hi,
                    const double *dl, const double *dr, double *out)
{
    orc_bc b = {bc, lo, hi, dl, dr, n};
    double *pool = (double *)malloc(sizeof(double) * N * 12);
    double *u = pool, *n0 = pool + N, *n1 = pool + 2 * N, *n2 = pool + 3 * N, *n3 = pool + 4 * N;
    double *whu = pool + 5 * N, *a = pool + 6 * N, *bb = pool + 7 * N, *c = pool + 8 * N;
    double *t1 = pool + 9 * N, *t2 = pool + 10 * N, *tmp = pool + 11 * N;
    memcpy(u, u0, sizeof(double) * N);
    for (int64_t s = 0; s < steps; ++s) {
        nonlinear(kind, d1w, mem, u, n0, tmp, N, n);
        orc_banded_matvec(w_half, mem, u, whu, N, n);
        orc_banded_matvec(w_p1h, mem, n0, t1, N, n);
        for (int64_t i = 0; i < N; ++i) a[i] = whu[i] + t1[i];
        apply_bc(a, N, &b);
        nonlinear(kind, d1w, mem, a, n1, tmp, N, n);
        orc_banded_matvec(w_p1h, mem, n1, t1, N, n);
        for (int64_t i = 0; i < N; ++i) bb[i] = whu[i] + t1[i];
        apply_bc(bb, N, &b);
        nonlinear(kind, d1w, mem, bb, n2, tmp, N, n);
        orc_banded_matvec(w_half, mem, a, t1, N, n);
        for (int64_t i = 0; i < N; ++i) t2[i] = 2.0 * n2[i] - n0[i];
        orc_banded_matvec(w_p1h, mem, t2, tmp, N, n);
        for (int64_t i = 0; i < N; ++i) c[i] = t1[i] + tmp[i];
        apply_bc(c, N, &b);
        nonlinear(kind, d1w, mem, c, n3, tmp, N, n);
        orc_banded_matvec(w_full, mem, u, t1, N, n);
        orc_banded_matvec(w_alpha, mem, n0, t2, N, n);
        for (int64_t i = 0; i < N; ++i) t1[i] += t2[i];
        for (int64_t i = 0; i < N; ++i) tmp[i] = n1[i] + n2[i];
        orc_banded_matvec(w_beta, mem, tmp, t2, N, n);
        for (int64_t i = 0; i < N; ++i) t1[i] += t2[i];
        orc_banded_matvec(w_gamma, mem, n3, t2, N, n);
        for (int64_t i = 0; i < N; ++i) u[i] = t1[i] + t2[i];
        apply_bc(u, N, &b);
    }
    memcpy(out, u, sizeof(double) * N);
    free(pool);
}

/* ETD multistep order 2 with one ETDRK4 warm-up step: timestep.py:187-215
 * (update) and :364-380 (warm-up).  The reference evaluates this path with
 * numpy einsum; here the banded products run in ascending order.
 * ops0/ops1/ops2: exp, dt*phi1, dt^2*phi2 rows at dt (raw), warm set is the
 * etdrk4 operator set.  kind: nonlinearity (convective uses d1w). */
void orc_run_etd2(const double *ops0, const double *ops1, const double *ops2,
                  const double *w_full, const double *w_alpha, const double *w_beta,
                  const double *w_gamma, const double *w_half, const double *w_p1h,
                  const double *d1w, const int64_t *mem, int kind, const double *u0,
                  int64_t N, int n, int64_t steps, double dt, int bc, double lo, double hi,
                  const double *dl, const double *dr, double *out, double *nhist_out)
{
    orc_bc b = {bc, lo, hi, dl, dr, n};
    double *pool = (double *)malloc(sizeof(double) * N * 6);
    double *u = pool, *nk = pool + N, *np_ = pool + 2 * N, *t1 = pool + 3 * N, *t2 = pool + 4 * N,
           *tmp = pool + 5 * N;
    memcpy(u, u0, sizeof(double) * N);
    if (steps >= 1) {
        nonlinear(kind, d1w, mem, u, np_, tmp, N, n);   /* history = (N(u0),) */
        orc_run_etdrk4(w_full, w_alpha, w_beta, w_gamma, w_half, w_p1h, d1w, mem, kind, u, N, n,
                       1, bc, lo, hi, dl, dr, u);
    }
    for (int64_t s = 1; s < steps; ++s) {
        nonlinear(kind, d1w, mem, u, nk, tmp, N, n);
        orc_banded_matvec(ops0, mem, u, t1, N, n);
        orc_banded_matvec(ops1, mem, nk, t2, N, n);
        for (int64_t i = 0; i < N; ++i) t1[i] = t1[i] + t2[i] / 1.0;
        for (int64_t i = 0; i < N; ++i) tmp[i] = nk[i] - np_[i];
        orc_banded_matvec(ops2, mem, tmp, t2, N, n);
        for (int64_t i = 0; i < N; ++i) u[i] = t1[i] + t2[i] / dt;
        apply_bc(u, N, &b);
        double *t = np_; np_ = nk; nk = t;
    }
    memcpy(out, u, sizeof(double) * N);
    if (nhist_out) memcpy(nhist_out, np_, sizeof(double) * N);
    free(pool);
}

/* ------------------------------------------------------------------ */
/* Compact-operator stepping (full-size parity runs).                  */
/*                                                                     */
/* The same arithmetic as the member-array loops above -- every node's */
/* window sum runs j = 0..n-1 ascending from acc = 0.0 with separate   */
/* multiply / add roundings (kernels.py:23-29) and every pointwise     */
/* expression keeps the reference's operand order (kernels.py:62-132,  */
/* timestep.py:187-215) -- but the window of node i comes from the     */
/* select_stencils rule (grid.py:136-175) by index arithmetic instead  */
/* of an (N, n) int64 member array, and rows are stored compactly:     */
/*   mode 0  one shared row [n]          (periodic uniform grid)       */
/*   mode 1  classes [nleft + 1 + nright][n]: node i < nleft uses      */
/*           class i, i >= N - nright class nleft+1+(i-(N-nright)),    */
/*           every other node the interior class nleft                 */
/*   mode 2  per-node rows [N][n] (the reference's weights layout)     */
/*   mode 3  keyed rows [K][n] with a per-node key cls[N]: the rows of  */
/*           the reference's exact-match harvest cache (harvest.py:    */
/*           135-159), one per distinct (coordinates, row, frozen) key */
/* Results are bit-identical to the member-array loops on the dense    */
/* rows these expand to (tests/test_oracle_golden.py checks that); the */
/* pointwise stages are fused into the window loops and every loop is  */
/* OpenMP-parallel, so the BASELINE-size runs (C4: 2^24 x 1000 steps)  */
/* finish in minutes instead of hours.                                 */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t N;
    int32_t n, row, periodic, mode, nleft, nright;
    const int32_t *cls;        /* mode 3: key of node i */
} orc_geom;

static inline const double *crow(const orc_geom *g, const double *w, int64_t i)
{
    if (g->mode == 0) return w;
    if (g->mode == 2) return w + i * g->n;
    if (g->mode == 3) return w + (int64_t)g->cls[i] * g->n;
    if (i < g->nleft) return w + i * g->n;
    if (i >= g->N - g->nright) return w + (g->nleft + 1 + (i - (g->N - g->nright))) * g->n;
    return w + (int64_t)g->nleft * g->n;
}

/* sum_j w_i[j] * u[member(i, j)], ascending j (kernels.py:23-29) */
static inline double cdot(const orc_geom *g, const double *w, const double *u, int64_t i)
{
    const double *wr = crow(g, w, i);
    const int n = g->n;
    const int64_t N = g->N;
    int64_t s = i - g->row;
    double acc = 0.0;
    if (g->periodic) {
        if (s >= 0 && s + n <= N) {
            for (int j = 0; j < n; ++j) acc += wr[j] * u[s + j];
        } else {
            s = ((s % N) + N) % N;
            for (int j = 0; j < n; ++j) {
                int64_t m = s + j;
                if (m >= N) m -= N;
                acc += wr[j] * u[m];
            }
        }
    } else {
        if (s < 0) s = 0;
        if (s > N - n) s = N - n;
        for (int j = 0; j < n; ++j) acc += wr[j] * u[s + j];
    }
    return acc;
}

/* kernels.py:47-58 for node i (convective: -u * (D1 u), cubic: -u^3) */
static inline double cnl(int kind, const orc_geom *g, const double *d1w, const double *u,
                         int64_t i)
{
    if (kind == 0) return 0.0;
    if (kind == 1) return -u[i] * cdot(g, d1w, u, i);
    return -u[i] * u[i] * u[i];
}

#ifdef _OPENMP
#define ORC_PFOR _Pragma("omp parallel for schedule(static)")
#else
#define ORC_PFOR
#endif

/* kernels.py:33-43 on compact rows */
void orc_run_linear_c(const orc_geom *g, const double *w, const double *u0, int64_t steps,
                      int bc, double lo, double hi, const double *dl, const double *dr,
                      double *out)
{
    const int64_t N = g->N;
    orc_bc b = {bc, lo, hi, dl, dr, g->n};
    double *u = (double *)malloc(sizeof(double) * N);
    double *buf = (double *)malloc(sizeof(double) * N);
    memcpy(u, u0, sizeof(double) * N);
    for (int64_t s = 0; s < steps; ++s) {
        ORC_PFOR
        for (int64_t i = 0; i < N; ++i) buf[i] = cdot(g, w, u, i);
        apply_bc(buf, N, &b);
        double *t = u; u = buf; buf = t;
    }
    memcpy(out, u, sizeof(double) * N);
    free(u); free(buf);
}

/* kernels.py:62-132 on compact rows (+ the Neumann closure of Appendix B.2),
 * one step; rows: w, alpha, beta, gamma, w_half, p1_half, d1. */
static void etdrk4_step_c(const orc_geom *g, const double *const *R, int kind, double *u,
                          double *unew, double *pool, const orc_bc *b)
{
    const int64_t N = g->N;
    const double *w = R[0], *al = R[1], *be = R[2], *ga = R[3], *wh = R[4], *p1h = R[5],
                 *d1 = R[6];
    double *n0 = pool, *n1 = pool + N, *n2 = pool + 2 * N, *n3 = pool + 3 * N;
    double *whu = pool + 4 * N, *a = pool + 5 * N, *bb = pool + 6 * N, *c = pool + 7 * N;
    double *t2 = pool + 8 * N;
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) {
        n0[i] = cnl(kind, g, d1, u, i);
        whu[i] = cdot(g, wh, u, i);
    }
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) a[i] = whu[i] + cdot(g, p1h, n0, i);
    apply_bc(a, N, b);
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) n1[i] = cnl(kind, g, d1, a, i);
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) bb[i] = whu[i] + cdot(g, p1h, n1, i);
    apply_bc(bb, N, b);
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) {
        n2[i] = cnl(kind, g, d1, bb, i);
        t2[i] = 2.0 * n2[i] - n0[i];
    }
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) c[i] = cdot(g, wh, a, i) + cdot(g, p1h, t2, i);
    apply_bc(c, N, b);
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) {
        n3[i] = cnl(kind, g, d1, c, i);
        t2[i] = n1[i] + n2[i];
    }
    ORC_PFOR
    for (int64_t i = 0; i < N; ++i) {
        double t1 = cdot(g, w, u, i);
        t1 += cdot(g, al, n0, i);
        t1 += cdot(g, be, t2, i);
        unew[i] = t1 + cdot(g, ga, n3, i);
    }
    apply_bc(unew, N, b);
}

void orc_run_etdrk4_c(const orc_geom *g, const double *w, const double *al, const double *be,
                      const double *ga, const double *wh, const double *p1h, const double *d1,
                      int kind, const double *u0, int64_t steps, int bc, double lo, double hi,
                      const double *dl, const double *dr, double *out, double *nl0_out)
{
    const int64_t N = g->N;
    const double *R[7] = {w, al, be, ga, wh, p1h, d1};
    orc_bc b = {bc, lo, hi, dl, dr, g->n};
    double *pool = (double *)malloc(sizeof(double) * N * 11);
    double *u = pool + 9 * N, *un = pool + 10 * N;
    memcpy(u, u0, sizeof(double) * N);
    for (int64_t s = 0; s < steps; ++s) {
        etdrk4_step_c(g, R, kind, u, un, pool, &b);
        if (s == 0 && nl0_out) memcpy(nl0_out, pool, sizeof(double) * N);   /* N(u0) */
        double *t = u; u = un; un = t;
    }
    memcpy(out, u, sizeof(double) * N);
    free(pool);
}

/* ETD multistep, order 2 (timestep.py:187-215) after one ETDRK4 warm-up step
 * (timestep.py:364-380), on compact rows: ops0/ops1/ops2 = exp, dt*phi1,
 * dt^2*phi2 at dt; warm = the ETDRK4 rows (w, alpha, beta, gamma, w_half,
 * p1_half); d1 the (scaled) derivative row of the convective N(u). */
void orc_run_etd2_c(const orc_geom *g, const double *ops0, const double *ops1,
                    const double *ops2, const double *w, const double *al, const double *be,
                    const double *ga, const double *wh, const double *p1h, const double *d1,
                    int kind, const double *u0, int64_t steps, double dt, int bc, double lo,
                    double hi, const double *dl, const double *dr, double *out,
                    double *nhist_out)
{
    const int64_t N = g->N;
    const double *R[7] = {w, al, be, ga, wh, p1h, d1};
    orc_bc b = {bc, lo, hi, dl, dr, g->n};
    double *pool = (double *)malloc(sizeof(double) * N * 14);
    double *u = pool + 9 * N, *un = pool + 10 * N, *nk = pool + 11 * N, *np_ = pool + 12 * N,
           *gr = pool + 13 * N;
    memcpy(u, u0, sizeof(double) * N);
    if (steps >= 1) {
        etdrk4_step_c(g, R, kind, u, un, pool, &b);
        memcpy(np_, pool, sizeof(double) * N);              /* history = (N(u0),) */
        double *t = u; u = un; un = t;
    }
    for (int64_t s = 1; s < steps; ++s) {
        ORC_PFOR
        for (int64_t i = 0; i < N; ++i) {
            nk[i] = cnl(kind, g, d1, u, i);
            gr[i] = nk[i] - np_[i];
        }
        ORC_PFOR
        for (int64_t i = 0; i < N; ++i) {
            double t1 = cdot(g, ops0, u, i);
            t1 = t1 + cdot(g, ops1, nk, i) / 1.0;
            un[i] = t1 + cdot(g, ops2, gr, i) / dt;
        }
        apply_bc(un, N, &b);
        double *t = u; u = un; un = t;
        t = np_; np_ = nk; nk = t;
    }
    memcpy(out, u, sizeof(double) * N);
    if (nhist_out) memcpy(nhist_out, np_, sizeof(double) * N);
    free(pool);
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void orc_set_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
