// step.cuh -- K3/K4/K5: fused fp64 banded time steps (sm_100a).
//
// Reference loops being replaced (kernels.py, numba, one core):
//   banded_matvec  kernels.py:23-29     out[i] = sum_j w[i,j] u[m[i,j]] (ascending j)
//   run_linear     kernels.py:33-43     steps x (matvec, Dirichlet pin, swap)
//   _nonlinear     kernels.py:47-58     0 | -u*(D1 u) | -u^3
//   run_etdrk4     kernels.py:62-132    4-stage exponential RK, 9 (+4) matvecs/step
//   etd_multistep_step timestep.py:187-215 (s = 2): W u + P1 N_k + P2 (N_k - N_{k-1})/dt
//
// Design (one kernel template for all three schemes):
//   * A CTA owns `tile` consecutive nodes and stages them plus a halo of
//     ksteps * ext * (row | n-1-row) nodes in shared memory (coalesced loads;
//     periodic wrap or neighbour-shard ghost buffers).  It then advances the
//     tile `ksteps` time steps entirely on chip: each stage is computed on the
//     range its successors need, the range shrinking towards the owned nodes
//     (halo recompute instead of a grid-wide barrier per stage).  u is read
//     from and written to HBM once per launch.
//   * Ring mode: a periodic grid that fits one CTA stays resident for ALL
//     steps in one launch; ghost cells are refreshed from the ring after each
//     stage (C1: 1000 steps, one launch).
//   * Each thread evaluates P consecutive outputs from a register window of
//     P + n - 1 staged values (odd P: the lane stride P is bank-conflict free),
//     interior weights come from the kernel parameter (constant) bank.
//     Boundary-class nodes take a per-node slow path.
//   * EXACT instantiations use separate IEEE multiply/add roundings in the
//     reference's ascending order, reproducing numba bit for bit; the others
//     use FMA (measured gate impact ~1e-15).
//   * Pins / Neumann closures are applied after every stage exactly where the
//     reference pins (kernels.py:93-95,101-103,112-114,129-131), and the fused
//     pointwise quantities of the pinned node are recomputed.
#pragma once
#include <algorithm>

#include "common.cuh"

namespace lmep {

enum { SCH_LIN = 0, SCH_ETDRK4 = 1, SCH_ETD2 = 2 };
constexpr int STEP_THREADS = 256;
constexpr int SLOT_PAD = 24;

struct StepParams {
    int64_t N, off, nloc;
    int n, row, periodic, ring;
    int eL, eR;
    int wmode, nrows, nleft, nright;
    int64_t L_int, R_int;                       // fast-path interior [L_int, R_int)
    double wi[LMEP_MAX_ROWS][LMEP_MAX_N];       // interior / shared rows
    const double *wc;                           // class rows [C][nrows][n]
    const double *wp;                           // per-node SoA [nrows][n][nloc]
    int nl;
    int bc;
    double lo, hi;
    double dl[LMEP_MAX_N], dr[LMEP_MAX_N];
    const double *u_in;
    double *u_out;
    const double *q_in;                         // etd2 history N_{k-1}
    double *q_out;
    const double *hl, *hr, *qhl, *qhr;          // ghost buffers (sharded) or null
    int64_t G;
    double *nl0_out;
    double dt;
    int ksteps, ext;
    int64_t tile;
    int64_t slot_len;
    int *flag;
};

template <bool EX>
__device__ __forceinline__ double padd(double a, double b)
{
    if constexpr (EX) return xadd(a, b);
    else return a + b;
}

// kernels.py:47-58 (numba: out = -u*tmp and -u*u*u, unary minus first)
template <bool EX>
__device__ __forceinline__ double nlp(int kind, double u, double du)
{
    if (kind == LMEP_NL_CONVECTIVE) return EX ? xmul(-u, du) : (-u) * du;
    if (kind == LMEP_NL_CUBIC) return EX ? xmul(xmul(-u, u), u) : ((-u) * u) * u;
    return 0.0;
}

__device__ __forceinline__ int64_t wrap(int64_t g, int64_t N)
{
    g %= N;
    return g < 0 ? g + N : g;
}

__device__ __forceinline__ double load_node(const StepParams &p, const double *v, const double *gl,
                                            const double *gr, int64_t g)
{
    if (gl == nullptr && gr == nullptr) {
        if (p.periodic) return v[wrap(g, p.N)];
        return v[g - p.off];
    }
    const int64_t li = g - p.off;
    if (li < 0) return gl[p.G + li];
    if (li >= p.nloc) return gr[li - p.nloc];
    return v[li];
}

__device__ __forceinline__ int64_t class_of(const StepParams &p, int64_t i)
{
    if (i < p.nleft) return i;
    if (i >= p.N - p.nright) return p.nleft + 1 + (i - (p.N - p.nright));
    return -1;
}

// one banded product at node i (any position: clamped window, class rows)
template <bool EX>
__device__ double band_slow(const StepParams &p, int r, const double *X, int64_t i, int64_t base)
{
    const int n = p.n;
    int64_t st = i - p.row;
    if (!p.periodic) st = st < 0 ? 0 : (st > p.N - n ? p.N - n : st);
    const double *wr;
    int64_t ws = 1;
    if (p.wmode == LMEP_W_PERNODE) {
        // single shard: halo nodes of a periodic tile wrap onto their owners
        const int64_t li = (p.periodic && p.hl == nullptr) ? wrap(i, p.N) : i - p.off;
        wr = p.wp + (int64_t)r * n * p.nloc + li;
        ws = p.nloc;
    } else if (p.wmode == LMEP_W_CLASS) {
        const int64_t cl = class_of(p, i);
        wr = cl < 0 ? p.wi[r] : p.wc + (cl * p.nrows + r) * n;
    } else {
        wr = p.wi[r];
    }
    const double *x = X + (st - base);
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = macc<EX>(acc, wr[j * ws], x[j]);
    return acc;
}

// P banded products at the consecutive interior nodes c0..c0+P-1.
template <int NS, int P, bool EX>
__device__ __forceinline__ void band_fast(const StepParams &p, int r, const double *X, int64_t c0,
                                          int64_t base, double *out)
{
    const double *x = X + (c0 - p.row - base);
    if constexpr (NS > 0) {
        double win[P + NS - 1];
#pragma unroll
        for (int q = 0; q < P + NS - 1; ++q) win[q] = x[q];
        if (p.wmode != LMEP_W_PERNODE) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < NS; ++j) acc = macc<EX>(acc, p.wi[r][j], win[q + j]);
                out[q] = acc;
            }
        } else {
            const double *w = p.wp + (int64_t)r * NS * p.nloc + (c0 - p.off);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < NS; ++j) acc = macc<EX>(acc, __ldcs(w + (int64_t)j * p.nloc + q), win[q + j]);
                out[q] = acc;
            }
        }
    } else {
        const int n = p.n;
        for (int q = 0; q < P; ++q) {
            double acc = 0.0;
            if (p.wmode != LMEP_W_PERNODE) {
                for (int j = 0; j < n; ++j) acc = macc<EX>(acc, p.wi[r][j], x[q + j]);
            } else {
                const double *w = p.wp + (int64_t)r * n * p.nloc + (c0 - p.off) + q;
                for (int j = 0; j < n; ++j) acc = macc<EX>(acc, __ldcs(w + (int64_t)j * p.nloc), x[q + j]);
            }
            out[q] = acc;
        }
    }
}

template <int NS, int P, bool EX>
__device__ __forceinline__ void bands(const StepParams &p, int r, const double *X, int64_t c0,
                                      int cnt, bool fast, int64_t base, double *out)
{
    if (fast) band_fast<NS, P, EX>(p, r, X, c0, base, out);
    else
        for (int q = 0; q < cnt; ++q) out[q] = band_slow<EX>(p, r, X, c0 + q, base);
}

// Value of a pinned node gb computed from stage vector X (smem, base-relative).
template <bool EX>
__device__ double bc_value(const StepParams &p, const double *X, int64_t gb, int64_t base)
{
    if (p.bc == LMEP_BC_DIRICHLET) return gb == 0 ? p.lo : p.hi;
    const int n = p.n;
    double acc = 0.0;
    if (gb == 0) {
        for (int j = 1; j < n; ++j) acc = xadd(acc, xmul(p.dl[j], X[j - base]));
        return xdiv(-acc, p.dl[0]);
    }
    const int64_t s0 = p.N - n;
    for (int j = 0; j < n - 1; ++j) acc = xadd(acc, xmul(p.dr[j], X[s0 + j - base]));
    return xdiv(-acc, p.dr[n - 1]);
}

template <int SCH, int NS, bool EX, int P>
__global__ void __launch_bounds__(STEP_THREADS) step_kernel(const __grid_constant__ StepParams p)
{
    extern __shared__ double sm[];
    constexpr int NSLOT = SCH == SCH_LIN ? 2 : (SCH == SCH_ETD2 ? 5 : 7);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int eL = p.eL, eR = p.eR;
    const bool ring = p.ring != 0;
    const bool pins = !p.periodic && p.bc != LMEP_BC_NONE;

    int64_t O0, O1;
    if (ring) {
        O0 = 0;
        O1 = p.N;
    } else {
        const int64_t t0 = (int64_t)blockIdx.x * p.tile;
        O0 = p.off + t0;
        O1 = p.off + (t0 + p.tile < p.nloc ? t0 + p.tile : p.nloc);
    }
    auto expand = [&](int units, int64_t &lo, int64_t &hi) {
        if (ring) { lo = 0; hi = p.N; return; }
        lo = O0 - (int64_t)units * eL;
        hi = O1 + (int64_t)units * eR;
        if (!p.periodic) {
            if (lo < 0) lo = 0;
            if (hi > p.N) hi = p.N;
        }
    };
    const int K = p.ksteps;
    int64_t base, gend;
    if (ring) { base = -eL; gend = p.N + eR; }
    else expand(K * p.ext, base, gend);
    const int len = (int)(gend - base);

    double *S[NSLOT];
#pragma unroll
    for (int q = 0; q < NSLOT; ++q) S[q] = sm + (int64_t)q * p.slot_len;

    // ---- stage u (and the etd2 history) into shared memory -------------
    for (int idx = tid; idx < len; idx += nt) {
        const int64_t g = base + idx;
        S[0][idx] = load_node(p, p.u_in, p.hl, p.hr, g);
        if constexpr (SCH == SCH_ETD2) S[1][idx] = load_node(p, p.q_in, p.qhl, p.qhr, g);
    }
    __syncthreads();

    // ring: refresh ghost cells of slot X from the ring itself
    auto refresh = [&](double *X) {
        if (!ring) return;
        __syncthreads();
        for (int idx = tid; idx < eL + eR; idx += nt) {
            if (idx < eL) X[idx] = X[p.N + idx];
            else X[eL + p.N + (idx - eL)] = X[eL + (idx - eL)];
        }
    };
    // thread 0 applies the closure of stage vector X at the boundary nodes in
    // [lo, hi); fix(gb, value, si) recomputes dependent pointwise values.
    auto pin_pass = [&](double *X, int64_t lo, int64_t hi, auto &&fix) {
        if (!pins) return;
        __syncthreads();
        if (tid == 0) {
            const int64_t ends[2] = {0, p.N - 1};
            for (int e = 0; e < 2; ++e) {
                const int64_t gb = ends[e];
                if (gb < lo || gb >= hi) continue;
                const double v = bc_value<EX>(p, X, gb, base);
                X[gb - base] = v;
                fix(gb - base, v);
            }
        }
    };
    auto none = [](int64_t, double) {};

#define CHUNK_LOOP(LO, HI)                                                          \
    for (int64_t c0 = (LO) + (int64_t)tid * P; c0 < (HI); c0 += (int64_t)nt * P)
#define CHUNK_SETUP(HI)                                                             \
    const int cnt = (int)((HI) - c0 < P ? (HI) - c0 : P);                           \
    const bool fast = cnt == P && c0 >= p.L_int && c0 + P <= p.R_int &&                  \
                      (p.wmode != LMEP_W_PERNODE || (c0 >= p.off && c0 + P <= p.off + p.nloc));

    const int nlk = p.nl;
    const int cv = (SCH != SCH_LIN && nlk == LMEP_NL_CONVECTIVE) ? 1 : 0;

    if constexpr (SCH == SCH_LIN) {
        int iU = 0, iV = 1;
        for (int s = 0; s < K; ++s) {
            const int u0 = (K - 1 - s) * p.ext;
            int64_t lo, hi;
            expand(u0, lo, hi);
            double *XU = S[iU], *XV = S[iV];
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double b[P];
                bands<NS, P, EX>(p, LMEP_ROW_W, XU, c0, cnt, fast, base, b);
                for (int q = 0; q < cnt; ++q) XV[c0 + q - base] = b[q];
            }
            pin_pass(XV, lo, hi, none);
            refresh(XV);
            __syncthreads();
            int t = iU; iU = iV; iV = t;
        }
        for (int64_t i = O0 + tid; i < O1; i += nt) {
            const double v = S[iU][i - base];
            p.u_out[i - p.off] = v;
            if (!isfinite(v)) *p.flag = 1;
        }
    } else if constexpr (SCH == SCH_ETDRK4) {
        // role -> slot
        enum { U, N0, WH, A, N1, B, S12, C, N3, UN, NR };
        int sl[NR];
        if (cv) {
            sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[N3] = 3; sl[N1] = 4; sl[S12] = 4;
            sl[B] = 5; sl[C] = 5; sl[UN] = 6;
        } else {
            sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[UN] = 3; sl[N1] = 4; sl[C] = 4;
            sl[S12] = 5; sl[B] = 6; sl[N3] = 6;
        }
        for (int s = 0; s < K; ++s) {
            const int u0 = (K - 1 - s) * p.ext;
            double *XU = S[sl[U]], *XN0 = S[sl[N0]], *XWH = S[sl[WH]], *XA = S[sl[A]];
            double *XN1 = S[sl[N1]], *XB = S[sl[B]], *XS12 = S[sl[S12]], *XC = S[sl[C]];
            double *XN3 = S[sl[N3]], *XUN = S[sl[UN]];
            double *XT2 = XWH;
            int64_t lo, hi;
            // P1: n0 = N(u)
            expand(u0 + 4 + 3 * cv, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double du[P];
                if (cv) bands<NS, P, EX>(p, LMEP_ROW_D1, XU, c0, cnt, fast, base, du);
                for (int q = 0; q < cnt; ++q) {
                    const int64_t si = c0 + q - base;
                    XN0[si] = nlp<EX>(nlk, XU[si], cv ? du[q] : 0.0);
                }
            }
            refresh(XN0);
            __syncthreads();
            // P2: whu = wh.u ; a = whu + p1h.n0 [pin] ; (cubic) n1 = N(a)
            expand(u0 + 3 + 3 * cv, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double bw[P], bp[P];
                bands<NS, P, EX>(p, LMEP_ROW_WHALF, XU, c0, cnt, fast, base, bw);
                bands<NS, P, EX>(p, LMEP_ROW_P1HALF, XN0, c0, cnt, fast, base, bp);
                for (int q = 0; q < cnt; ++q) {
                    const int64_t si = c0 + q - base;
                    const double a = padd<EX>(bw[q], bp[q]);
                    XWH[si] = bw[q];
                    XA[si] = a;
                    if (!cv) XN1[si] = nlp<EX>(nlk, a, 0.0);
                }
            }
            pin_pass(XA, lo, hi, [&](int64_t si, double v) { if (!cv) XN1[si] = nlp<EX>(nlk, v, 0.0); });
            refresh(XWH);
            refresh(XA);
            if (!cv) refresh(XN1);
            __syncthreads();
            // P3 (convective): n1 = N(a)
            if (cv) {
                expand(u0 + 3 + 2 * cv, lo, hi);
                CHUNK_LOOP(lo, hi) {
                    CHUNK_SETUP(hi)
                    double da[P];
                    bands<NS, P, EX>(p, LMEP_ROW_D1, XA, c0, cnt, fast, base, da);
                    for (int q = 0; q < cnt; ++q) {
                        const int64_t si = c0 + q - base;
                        XN1[si] = nlp<EX>(nlk, XA[si], da[q]);
                    }
                }
                refresh(XN1);
                __syncthreads();
            }
            // P4: b = whu + p1h.n1 [pin] ; (cubic) n2 = N(b), t2 = 2 n2 - n0, s12 = n1 + n2
            expand(u0 + 2 + 2 * cv, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double bp[P];
                bands<NS, P, EX>(p, LMEP_ROW_P1HALF, XN1, c0, cnt, fast, base, bp);
                for (int q = 0; q < cnt; ++q) {
                    const int64_t si = c0 + q - base;
                    const double b = padd<EX>(XWH[si], bp[q]);
                    XB[si] = b;
                    if (!cv) {
                        const double n2 = nlp<EX>(nlk, b, 0.0);
                        XT2[si] = EX ? xsub(xmul(2.0, n2), XN0[si]) : 2.0 * n2 - XN0[si];
                        XS12[si] = padd<EX>(XN1[si], n2);
                    }
                }
            }
            pin_pass(XB, lo, hi, [&](int64_t si, double v) {
                if (!cv) {
                    const double n2 = nlp<EX>(nlk, v, 0.0);
                    XT2[si] = EX ? xsub(xmul(2.0, n2), XN0[si]) : 2.0 * n2 - XN0[si];
                    XS12[si] = padd<EX>(XN1[si], n2);
                }
            });
            refresh(XB);
            if (!cv) { refresh(XT2); refresh(XS12); }
            __syncthreads();
            // P5 (convective): n2 = N(b), t2 = 2 n2 - n0, s12 = n1 + n2
            if (cv) {
                expand(u0 + 2 + cv, lo, hi);
                CHUNK_LOOP(lo, hi) {
                    CHUNK_SETUP(hi)
                    double db[P];
                    bands<NS, P, EX>(p, LMEP_ROW_D1, XB, c0, cnt, fast, base, db);
                    for (int q = 0; q < cnt; ++q) {
                        const int64_t si = c0 + q - base;
                        const double n2 = nlp<EX>(nlk, XB[si], db[q]);
                        XT2[si] = EX ? xsub(xmul(2.0, n2), XN0[si]) : 2.0 * n2 - XN0[si];
                        XS12[si] = padd<EX>(XN1[si], n2);
                    }
                }
                refresh(XT2);
                refresh(XS12);
                __syncthreads();
            }
            // P6: c = wh.a + p1h.t2 [pin] ; (cubic) n3 = N(c)
            expand(u0 + 1 + cv, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double ba[P], bt[P];
                bands<NS, P, EX>(p, LMEP_ROW_WHALF, XA, c0, cnt, fast, base, ba);
                bands<NS, P, EX>(p, LMEP_ROW_P1HALF, XT2, c0, cnt, fast, base, bt);
                for (int q = 0; q < cnt; ++q) {
                    const int64_t si = c0 + q - base;
                    const double c = padd<EX>(ba[q], bt[q]);
                    XC[si] = c;
                    if (!cv) XN3[si] = nlp<EX>(nlk, c, 0.0);
                }
            }
            pin_pass(XC, lo, hi, [&](int64_t si, double v) { if (!cv) XN3[si] = nlp<EX>(nlk, v, 0.0); });
            refresh(XC);
            if (!cv) refresh(XN3);
            __syncthreads();
            // P7 (convective): n3 = N(c)
            if (cv) {
                expand(u0 + 1, lo, hi);
                CHUNK_LOOP(lo, hi) {
                    CHUNK_SETUP(hi)
                    double dc[P];
                    bands<NS, P, EX>(p, LMEP_ROW_D1, XC, c0, cnt, fast, base, dc);
                    for (int q = 0; q < cnt; ++q) {
                        const int64_t si = c0 + q - base;
                        XN3[si] = nlp<EX>(nlk, XC[si], dc[q]);
                    }
                }
                refresh(XN3);
                __syncthreads();
            }
            // P8: u' = ((w.u + alpha.n0) + beta.s12) + gamma.n3 [pin]
            expand(u0, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double b0[P], b1[P], b2[P], b3[P];
                bands<NS, P, EX>(p, LMEP_ROW_W, XU, c0, cnt, fast, base, b0);
                bands<NS, P, EX>(p, LMEP_ROW_ALPHA, XN0, c0, cnt, fast, base, b1);
                bands<NS, P, EX>(p, LMEP_ROW_BETA, XS12, c0, cnt, fast, base, b2);
                bands<NS, P, EX>(p, LMEP_ROW_GAMMA, XN3, c0, cnt, fast, base, b3);
                for (int q = 0; q < cnt; ++q)
                    XUN[c0 + q - base] = padd<EX>(padd<EX>(padd<EX>(b0[q], b1[q]), b2[q]), b3[q]);
            }
            pin_pass(XUN, lo, hi, none);
            refresh(XUN);
            __syncthreads();
            if (s == 0 && p.nl0_out)
                for (int64_t i = O0 + tid; i < O1; i += nt) p.nl0_out[i - p.off] = XN0[i - base];
            // rotate: u <- u'; roles sharing u''s slot move to the old u slot
            const int newU = sl[UN], oldU = sl[U];
            for (int r = 0; r < NR; ++r)
                if (sl[r] == newU) sl[r] = oldU;
            sl[U] = newU;
        }
        for (int64_t i = O0 + tid; i < O1; i += nt) {
            const double v = S[sl[U]][i - base];
            p.u_out[i - p.off] = v;
            if (!isfinite(v)) *p.flag = 1;
        }
    } else {  // SCH_ETD2
        int iU = 0, iQ = 1, iK = 2, iD = 3, iV = 4;
        for (int s = 0; s < K; ++s) {
            const int u0 = (K - 1 - s) * p.ext;
            double *XU = S[iU], *XQ = S[iQ], *XK = S[iK], *XD = S[iD], *XV = S[iV];
            int64_t lo, hi;
            // P1: nk = N(u), d = nk - n_{k-1}
            expand(u0 + 1, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double du[P];
                if (cv) bands<NS, P, EX>(p, LMEP_ROW_D1, XU, c0, cnt, fast, base, du);
                for (int q = 0; q < cnt; ++q) {
                    const int64_t si = c0 + q - base;
                    const double nk = nlp<EX>(nlk, XU[si], cv ? du[q] : 0.0);
                    XK[si] = nk;
                    XD[si] = EX ? xsub(nk, XQ[si]) : nk - XQ[si];
                }
            }
            refresh(XK);
            refresh(XD);
            __syncthreads();
            // P2: u' = (W u + P1 nk) + P2 d / dt   (timestep.py:206-210)
            expand(u0, lo, hi);
            CHUNK_LOOP(lo, hi) {
                CHUNK_SETUP(hi)
                double b0[P], b1[P], b2[P];
                bands<NS, P, EX>(p, LMEP_ROW_W, XU, c0, cnt, fast, base, b0);
                bands<NS, P, EX>(p, LMEP_ROW_ALPHA, XK, c0, cnt, fast, base, b1);
                bands<NS, P, EX>(p, LMEP_ROW_BETA, XD, c0, cnt, fast, base, b2);
                for (int q = 0; q < cnt; ++q) {
                    const double t = EX ? xdiv(b2[q], p.dt) : b2[q] * (1.0 / p.dt);
                    XV[c0 + q - base] = padd<EX>(padd<EX>(b0[q], b1[q]), t);
                }
            }
            pin_pass(XV, lo, hi, none);
            refresh(XV);
            __syncthreads();
            // history <- nk, u <- u'
            int t = iQ; iQ = iK; iK = t;
            t = iU; iU = iV; iV = t;
        }
        for (int64_t i = O0 + tid; i < O1; i += nt) {
            const double v = S[iU][i - base];
            p.u_out[i - p.off] = v;
            p.q_out[i - p.off] = S[iQ][i - base];
            if (!isfinite(v)) *p.flag = 1;
        }
    }
#undef CHUNK_LOOP
#undef CHUNK_SETUP
}

template <int SCH, bool EX, int P>
inline int launch_ns(int ns_case, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    void (*k)(StepParams) = nullptr;
    switch (ns_case) {
    case 7: k = step_kernel<SCH, 7, EX, P>; break;
    case 9: k = step_kernel<SCH, 9, EX, P>; break;
    case 11: k = step_kernel<SCH, 11, EX, P>; break;
    case 13: k = step_kernel<SCH, 13, EX, P>; break;
    default: k = step_kernel<SCH, 0, EX, P>; break;
    }
    if (shm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) { set_last_error("cudaFuncSetAttribute", e); return LMEP_CUDA_ERROR; }
    }
    k<<<grid, STEP_THREADS, shm, st>>>(p);
    return launch_status("step_kernel");
}

int launch_scheme_lin(bool pernode, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st);
int launch_scheme_etdrk4(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st);
int launch_scheme_etd2(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st);

}  // namespace lmep
