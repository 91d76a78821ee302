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

constexpr int STEP_THREADS = 256;
constexpr int SLOT_PAD = 24;
constexpr int STEP_P_ETDRK4 = 7;   // consecutive outputs per thread (odd: conflict-free)
constexpr int STEP_P_ETDRK4_CV = 5; // convective N: wider stencils, one more window per stage
// pointwise N: 7 nodes per thread at n = 7 (C4), 5 for wider stencils (7 spills at 128 registers)
constexpr int step_p_etdrk4(int nl, int n) { return (nl == LMEP_NL_CONVECTIVE || n != 7) ? STEP_P_ETDRK4_CV : STEP_P_ETDRK4; }
constexpr int STEP_P_ETD2 = 1;

struct StepParams {
    int64_t N, off, nloc;
    int n, row, periodic, ring;
    int eL, eR;
    int wmode, nrows, nleft, nright;
    int64_t L_int, R_int;                       // fast-path interior [L_int, R_int)
    double wi[LMEP_MAX_ROWS][LMEP_MAX_N];       // interior / shared rows
    const double *wc;                           // class rows [C][nrows][n]
    const double *wp;                           // per-node SoA [nrows][n][wld]
    int64_t wld, wpad;                          // per-node table: leading dim, local node 0 at wpad
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
    double *push_l, *push_r;                    // fused peer stores of the slab edges (or null)
    int64_t push_w;
    int64_t tile_lo, tile_hi;                   // persistent per-node kernels: tiles of this launch (hi = 0: all)
    int64_t tile_wrap;                          // ... > 0: tile indices >= tile_wrap continue at tile 0 (a range that wraps)
    int pdl;                                    // ... launched as a programmatic dependent of the launch before it on the
                                                // stream: 1 = only u_in is that launch's output (the rows may be fetched
                                                // before it has finished), 2 = the rows may be too
    int64_t ext_off;                            // ... on a slab: u_in / rows start ext_off nodes before the owned ones
    double *nl0_out;
    double dt;
    double dtj[6];                              // etd-s: dt**j as Python computes it
    int64_t qld;                                // etd-s: history vector stride (>= nloc)
    int ksteps, ext;
    int etds;                                   // etd-s order (1..5)
    int threads;                                // CTA size (multiple of 32, <= STEP_THREADS)
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

// result of owned local node li: u_out, plus the neighbours' mailboxes when the
// launch carries fused peer stores (lmep_halo.push_*: first / last push_w nodes)
__device__ __forceinline__ void store_out(const StepParams &p, int64_t li, double v)
{
    p.u_out[li] = v;
    if (p.push_w > 0) {
        if (p.push_l && li < p.push_w) p.push_l[li] = v;
        if (p.push_r && li >= p.nloc - p.push_w) p.push_r[li - (p.nloc - p.push_w)] = v;
    }
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
__device__ __noinline__ double band_slow(const StepParams &p, int r, const double *X, int64_t i, int64_t base)
{
    const int n = p.n;
    int64_t st = i - p.row;
    if (!p.periodic) st = st < 0 ? 0 : (st > p.N - n ? p.N - n : st);
    const double *wr;
    int64_t ws = 1;
    if (p.wmode == LMEP_W_PERNODE) {
        // single shard: halo nodes of a periodic tile wrap onto their owners
        const int64_t li = (p.periodic && p.hl == nullptr) ? wrap(i, p.N) : i - p.off;
        wr = p.wp + (int64_t)r * n * p.wld + li + p.wpad;
        ws = p.wld;
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
template <int NS, int P, bool EX, bool PN>
__device__ __forceinline__ void band_fast(const StepParams &p, int r, const double *X, int l,
                                          int64_t lbase, double *out)
{
    const double *x = X + (l - p.row);
    if constexpr (NS > 0) {
        double win[P + NS - 1];
#pragma unroll
        for (int q = 0; q < P + NS - 1; ++q) win[q] = x[q];
        if constexpr (!PN) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < NS; ++j) acc = macc<EX>(acc, p.wi[r][j], win[q + j]);
                out[q] = acc;
            }
        } else {
            const double *w = p.wp + (int64_t)r * NS * p.wld + (lbase + l + p.wpad);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int j = 0; j < NS; ++j) acc = macc<EX>(acc, __ldcs(w + (int64_t)j * p.wld + q), win[q + j]);
                out[q] = acc;
            }
        }
    } else {
        const int n = p.n;
        for (int q = 0; q < P; ++q) {
            double acc = 0.0;
            if constexpr (!PN) {
                for (int j = 0; j < n; ++j) acc = macc<EX>(acc, p.wi[r][j], x[q + j]);
            } else {
                const double *w = p.wp + (int64_t)r * n * p.wld + (lbase + l + p.wpad) + q;
                for (int j = 0; j < n; ++j) acc = macc<EX>(acc, __ldcs(w + (int64_t)j * p.wld), x[q + j]);
            }
            out[q] = acc;
        }
    }
}

// Value of a pinned node gb computed from stage vector X (smem, base-relative).
template <bool EX>
__device__ __noinline__ double bc_value(const StepParams &p, const double *X, int64_t gb, int64_t base)
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

// One stage pass over the tile-local range [lo, hi): NB banded products
// (rows[b] applied to X[b]) per node, then epi(l, v[NB]).  Full interior
// chunks of P nodes take the register-window fast path with no guards; the
// few remaining nodes (range ends, boundary classes) take a per-node path.
template <int NS, int P, bool EX, bool PN, int NB, class Epi>
__device__ __forceinline__ void run_pass(const StepParams &p, int lo, int hi, int fLo, int fHi,
                                         int64_t base, int64_t lbase, const int (&rows)[NB],
                                         const double *const (&X)[NB], Epi &&epi)
{
    const int tid = threadIdx.x, nt = blockDim.x;
    const int flo = lo > fLo ? lo : fLo;
    const int fhi = hi < fHi ? hi : fHi;
    // interior chunks, the last one possibly partial: the fast path computes
    // all P outputs (the window may run into the slot padding) and stores cnt
    const int nch = fhi > flo ? (fhi - flo + P - 1) / P : 0;
#pragma unroll 1
    for (int ch = tid; ch < nch; ch += nt) {
        const int l = flo + ch * P;
        const int cnt = fhi - l < P ? fhi - l : P;
        double v[NB > 0 ? NB : 1][P];
#pragma unroll
        for (int b = 0; b < NB; ++b) band_fast<NS, P, EX, PN>(p, rows[b], X[b], l, lbase, v[b]);
#pragma unroll
        for (int q = 0; q < P; ++q) {
            if (q < cnt) {
                double vq[NB > 0 ? NB : 1];
#pragma unroll
                for (int b = 0; b < NB; ++b) vq[b] = v[b][q];
                epi(l + q, vq);
            }
        }
    }
    // boundary-class nodes of non-periodic grids (or the whole range if it has
    // no interior part): per-node path, handed to the threads with fewest chunks
    const int a_end = nch > 0 ? flo : hi;
    const int b_beg = nch > 0 ? fhi : hi;
    const int na = a_end - lo, nb = hi - b_beg;
#pragma unroll 1
    for (int k = nt - 1 - tid; k < na + nb; k += nt) {
        const int l = k < na ? lo + k : b_beg + (k - na);
        double vq[NB > 0 ? NB : 1];
#pragma unroll
        for (int b = 0; b < NB; ++b) vq[b] = band_slow<EX>(p, rows[b], X[b], base + l, base);
        epi(l, vq);
    }
}

// pointwise pass (no banded product)
template <class Epi>
__device__ __forceinline__ void run_pointwise(int lo, int hi, Epi &&epi)
{
#pragma unroll 1
    for (int l = lo + (int)threadIdx.x; l < hi; l += blockDim.x) epi(l);
}

// Lean pass for CTAs whose whole staged range is interior (periodic grids, or
// tiles clear of the boundary classes and pins): every chunk of P nodes in
// [lo, hi) takes the register-window path, with no range clamping, boundary
// path or tail guard.  Nodes in the halo whose windows reach stale values are
// computed anyway (they are never stored; the staged halo covers exactly the
// ranges the generic passes would compute), and the last chunk's overhang
// lands in the slot padding (SLOT_PAD + P >= NS - 1 + P).
template <int NS, int P, bool EX, int NB, class Epi>
__device__ __forceinline__ void fast_pass(const StepParams &p, int lo, int hi, const int (&rows)[NB],
                                          const double *const (&X)[NB], Epi &&epi)
{
    const int nch = (hi - lo + P - 1) / P;
#pragma unroll 1
    for (int ch = threadIdx.x; ch < nch; ch += blockDim.x) {
        const int l = lo + ch * P;
        double v[NB][P];
#pragma unroll
        for (int b = 0; b < NB; ++b) band_fast<NS, P, EX, false>(p, rows[b], X[b], l, 0, v[b]);
#pragma unroll
        for (int q = 0; q < P; ++q) {
            double vq[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) vq[b] = v[b][q];
            epi(l + q, vq);
        }
    }
}

template <int P, class Epi>
__device__ __forceinline__ void fast_pointwise(int lo, int hi, Epi &&epi)
{
    const int nch = (hi - lo + P - 1) / P;
#pragma unroll 1
    for (int ch = threadIdx.x; ch < nch; ch += blockDim.x) {
        const int l = lo + ch * P;
#pragma unroll
        for (int q = 0; q < P; ++q) epi(l + q);
    }
}

}  // namespace lmep
#include "step_rk4.cuh"
namespace lmep {

template <int SCH, int NS, bool EX, int P, int NLK, bool PN, int ETDS = 2>
__global__ void __launch_bounds__(STEP_THREADS, SCH == SCH_LIN ? 1 : 2)
step_kernel(const __grid_constant__ StepParams p)
{
    extern __shared__ double sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int eL = p.eL, eR = p.eR;
    const bool ring = p.ring != 0;
    const bool pins = !p.periodic && p.bc != LMEP_BC_NONE;
    constexpr int nlk = NLK;
    constexpr bool cv = SCH != SCH_LIN && NLK == LMEP_NL_CONVECTIVE;

    int64_t O0, O1;
    if (ring) {
        O0 = 0;
        O1 = p.N;
    } else {
        const int64_t t0 = (int64_t)blockIdx.x * p.tile;
        O0 = p.off + t0;
        O1 = p.off + (t0 + p.tile < p.nloc ? t0 + p.tile : p.nloc);
    }
    auto expand_g = [&](int units, int64_t &lo, int64_t &hi) {
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
    else expand_g(K * p.ext, base, gend);
    const int len = (int)(gend - base);
    // pass ranges in tile-local (shared-memory) coordinates, 32-bit: the owned
    // range [o0, o1) grows by units*(eL, eR), clamped to the grid for
    // non-periodic grids (ring mode: the whole staged ring)
    const int64_t big = 1 << 30;
    auto clampi = [&](int64_t v) { return (int)(v < -big ? -big : (v > big ? big : v)); };
    const int o0 = ring ? 0 : clampi(O0 - base), o1 = ring ? (int)p.N : clampi(O1 - base);
    const int cLo = (ring || p.periodic) ? -(1 << 30) : clampi(-base);
    const int cHi = (ring || p.periodic) ? (1 << 30) : clampi(p.N - base);
    auto expand = [&](int units, int &lo, int &hi) {
        if (ring) { lo = eL; hi = eL + (int)p.N; return; }          // global [0, N)
        lo = o0 - units * eL;
        hi = o1 + units * eR;
        lo = lo > cLo ? lo : cLo;
        hi = hi < cHi ? hi : cHi;
    };
    // fast-path window: interior class and, for per-node rows, owned nodes
    const int64_t lbase = base - p.off;
    int fLo, fHi;
    {
        int64_t a = p.L_int - base, b = p.R_int - base;
        if (PN) {
            a = a > -lbase ? a : -lbase;
            b = b < p.nloc - lbase ? b : p.nloc - lbase;
        }
        fLo = clampi(a);
        fHi = clampi(b);
    }
    const int slen = (int)p.slot_len;
#define S(q) (sm + (q) * slen)

    // ---- stage u (and the etd2 history) into shared memory -------------
    // ETDRK4 tiles that lie inside one shard without wrapping: the loads of a
    // thread are issued back to back (one memory latency per tile, not one per
    // element; the dependent load -> store loop below cost 15% of the C4 kernel)
    bool staged = false;
    if constexpr (SCH == SCH_ETDRK4) {
        if (!ring && p.hl == nullptr && p.hr == nullptr && base >= p.off && gend <= p.off + p.nloc) {
            const double *src = p.u_in + (base - p.off);
            constexpr int UB = 8;
            for (int i0 = tid; i0 < len; i0 += UB * nt) {
                double v[UB];
#pragma unroll
                for (int j = 0; j < UB; ++j) v[j] = i0 + j * nt < len ? __ldg(src + i0 + j * nt) : 0.0;
#pragma unroll
                for (int j = 0; j < UB; ++j) {
                    if (i0 + j * nt < len) {
                        S(0)[i0 + j * nt] = v[j];
                        if constexpr (!cv) S(1)[i0 + j * nt] = nlp<EX>(nlk, v[j], 0.0);
                    }
                }
            }
            staged = true;
        }
    }
    for (int idx = tid; !staged && idx < len; idx += nt) {
        const int64_t g = base + idx;
        const double u = load_node(p, p.u_in, p.hl, p.hr, g);
        S(0)[idx] = u;
        if constexpr (SCH == SCH_ETD2) {
#pragma unroll
            for (int i = 1; i < ETDS; ++i)                       // history N_{k-i}, newest first
                S(i)[idx] = load_node(p, p.q_in + (int64_t)(i - 1) * p.qld,
                                      p.qhl ? p.qhl + (int64_t)(i - 1) * p.G : nullptr,
                                      p.qhr ? p.qhr + (int64_t)(i - 1) * p.G : nullptr, g);
        }
        if constexpr (SCH == SCH_ETDRK4 && !cv) S(1)[idx] = nlp<EX>(nlk, u, 0.0);  // n0 of step 0
    }
    __syncthreads();

    // end of a pass: barrier, then (ring) refresh the ghost cells of X
    auto refresh = [&](double *X) {
        if (!ring) return;
        __syncthreads();
        for (int idx = tid; idx < eL + eR; idx += nt) {
            if (idx < eL) X[idx] = X[p.N + idx];
            else X[eL + p.N + (idx - eL)] = X[eL + (idx - eL)];
        }
    };
    // thread 0 applies the closure of stage vector X at the boundary nodes in
    // [lo, hi); fix(l, value) recomputes the dependent pointwise values.
    const int pb0 = clampi(-base), pb1 = clampi(p.N - 1 - base);   // boundary nodes, tile-local
    auto pin_pass = [&](double *X, int lo, int hi, auto &&fix) {
        if (!pins) return;
        if (!((pb0 >= lo && pb0 < hi) || (pb1 >= lo && pb1 < hi))) return;   // CTA-uniform
        __syncthreads();
        if (tid == 0) {
            const int64_t ends[2] = {0, p.N - 1};
            for (int e = 0; e < 2; ++e) {
                const int64_t gb = ends[e];
                if (gb - base < lo || gb - base >= hi) continue;
                const double v = bc_value<EX>(p, X, gb, base);
                X[gb - base] = v;
                fix((int)(gb - base), v);
            }
        }
    };
    auto none = [](int, double) {};
    auto sub2 = [](double n2, double n0) { return EX ? xsub(xmul(2.0, n2), n0) : 2.0 * n2 - n0; };

    if constexpr (SCH == SCH_LIN) {
        int iU = 0, iV = 1;
        if constexpr (!PN && NS > 0) {
            // Ring mode (a periodic grid resident in one CTA, C1): one barrier per
            // step.  The threads that write nodes mirrored by the ghost cells also
            // write the mirror, so no separate ghost refresh (and its barrier) is
            // needed: staged position eL + i holds node i, ghosts [0, eL) mirror
            // nodes N - eL .. N - 1 and [eL + N, eL + N + eR) mirror nodes 0 .. eR - 1.
            if (ring) {
                const int NN = (int)p.N;
                for (int s = 0; s < K; ++s) {
                    double *XU = S(iU), *XV = S(iV);
                    const int rows[1] = {LMEP_ROW_W};
                    const double *const X[1] = {XU};
                    fast_pass<NS, P, EX, 1>(p, eL, eL + NN, rows, X, [&](int l, const double *v) {
                        if (l < eL + NN) {
                            XV[l] = v[0];
                            if (l >= NN) XV[l - NN] = v[0];
                            if (l < eL + eR) XV[l + NN] = v[0];
                        }
                    });
                    __syncthreads();
                    const int t = iU; iU = iV; iV = t;
                }
                bool bad = false;
                for (int64_t i = O0 + tid; i < O1; i += nt) {
                    const double v = S(iU)[i - base];
                    store_out(p, i - p.off, v);
                    bad |= !isfinite(v);
                }
                if (bad) *p.flag = 1;
                return;
            }
        }
        for (int s = 0; s < K; ++s) {
            int lo, hi;
            expand((K - 1 - s) * p.ext, lo, hi);
            double *XU = S(iU), *XV = S(iV);
            const int rows[1] = {LMEP_ROW_W};
            const double *const X[1] = {XU};
            run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                                       [&](int l, const double *v) { XV[l] = v[0]; });
            pin_pass(XV, lo, hi, none);
            refresh(XV);
            __syncthreads();
            const int t = iU; iU = iV; iV = t;
        }
        for (int64_t i = O0 + tid; i < O1; i += nt) {
            const double v = S(iU)[i - base];
            store_out(p, i - p.off, v);
            if (!isfinite(v)) *p.flag = 1;
        }
    } else if constexpr (SCH == SCH_ETDRK4) {
        // role -> slot; T2 shares WH's slot
        enum { U, N0, WH, A, N1, B, S12, C, N3, UN, NR };
        int sl[NR];
        // ---- interior fast path: same slot plan and arithmetic as below, every pass
        // over [eL, len) (the windows of node eL start at staged node 0)
        if constexpr (!PN && NS > 0) {
            // (a non-periodic tile clear of the boundary classes holds no pinned node)
            const bool fast = !ring && (p.periodic || (base >= p.L_int && gend <= p.R_int));
            // one chunk of P staged nodes per thread: the register-resident passes
            // (step_rk4.cuh); CTA-uniform
            if (fast && (len - eL + P - 1) / P <= nt) {
                if constexpr (cv) etdrk4_regs_convective<NS, P, EX>(p, sm, slen, len, K, O0, O1, base);
                else etdrk4_regs_pointwise<NS, P, EX, NLK>(p, sm, slen, len, K, O0, O1, base);
                return;
            }
            if (fast) {
                if constexpr (cv) {
                    sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[N3] = 3; sl[N1] = 4; sl[S12] = 4;
                    sl[B] = 5; sl[C] = 5; sl[UN] = 6;
                } else {
                    sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[UN] = 3; sl[N1] = 4; sl[C] = 4;
                    sl[S12] = 5; sl[B] = 6; sl[N3] = 6;
                }
                const int lo = eL, hi = len;
                for (int s = 0; s < K; ++s) {
                    double *XU = S(sl[U]), *XN0 = S(sl[N0]), *XWH = S(sl[WH]), *XA = S(sl[A]);
                    double *XN1 = S(sl[N1]), *XB = S(sl[B]), *XS12 = S(sl[S12]), *XC = S(sl[C]);
                    double *XN3 = S(sl[N3]), *XUN = S(sl[UN]);
                    double *XT2 = XWH;
                    if constexpr (cv) {
                        const int rows[1] = {LMEP_ROW_D1};
                        const double *const X[1] = {XU};
                        fast_pass<NS, P, EX, 1>(p, lo, hi, rows, X,
                            [&](int l, const double *v) { XN0[l] = nlp<EX>(nlk, XU[l], v[0]); });
                        __syncthreads();
                    } else if (s > 0) {
                        fast_pointwise<P>(0, hi, [&](int l) { XN0[l] = nlp<EX>(nlk, XU[l], 0.0); });
                        __syncthreads();
                    }
                    {
                        const int rows[2] = {LMEP_ROW_WHALF, LMEP_ROW_P1HALF};
                        const double *const X[2] = {XU, XN0};
                        fast_pass<NS, P, EX, 2>(p, lo, hi, rows, X, [&](int l, const double *v) {
                            const double a = padd<EX>(v[0], v[1]);
                            XWH[l] = v[0];
                            XA[l] = a;
                            if constexpr (!cv) XN1[l] = nlp<EX>(nlk, a, 0.0);
                        });
                    }
                    __syncthreads();
                    if constexpr (cv) {
                        const int rows[1] = {LMEP_ROW_D1};
                        const double *const X[1] = {XA};
                        fast_pass<NS, P, EX, 1>(p, lo, hi, rows, X,
                            [&](int l, const double *v) { XN1[l] = nlp<EX>(nlk, XA[l], v[0]); });
                        __syncthreads();
                    }
                    {
                        const int rows[1] = {LMEP_ROW_P1HALF};
                        const double *const X[1] = {XN1};
                        fast_pass<NS, P, EX, 1>(p, lo, hi, rows, X, [&](int l, const double *v) {
                            const double b = padd<EX>(XWH[l], v[0]);
                            XB[l] = b;
                            if constexpr (!cv) {
                                const double n2 = nlp<EX>(nlk, b, 0.0);
                                XT2[l] = sub2(n2, XN0[l]);
                                XS12[l] = padd<EX>(XN1[l], n2);
                            }
                        });
                    }
                    __syncthreads();
                    if constexpr (cv) {
                        const int rows[1] = {LMEP_ROW_D1};
                        const double *const X[1] = {XB};
                        fast_pass<NS, P, EX, 1>(p, lo, hi, rows, X, [&](int l, const double *v) {
                            const double n2 = nlp<EX>(nlk, XB[l], v[0]);
                            XT2[l] = sub2(n2, XN0[l]);
                            XS12[l] = padd<EX>(XN1[l], n2);
                        });
                        __syncthreads();
                    }
                    {
                        const int rows[2] = {LMEP_ROW_WHALF, LMEP_ROW_P1HALF};
                        const double *const X[2] = {XA, XT2};
                        fast_pass<NS, P, EX, 2>(p, lo, hi, rows, X, [&](int l, const double *v) {
                            const double c = padd<EX>(v[0], v[1]);
                            XC[l] = c;
                            if constexpr (!cv) XN3[l] = nlp<EX>(nlk, c, 0.0);
                        });
                    }
                    __syncthreads();
                    if constexpr (cv) {
                        const int rows[1] = {LMEP_ROW_D1};
                        const double *const X[1] = {XC};
                        fast_pass<NS, P, EX, 1>(p, lo, hi, rows, X,
                            [&](int l, const double *v) { XN3[l] = nlp<EX>(nlk, XC[l], v[0]); });
                        __syncthreads();
                    }
                    {
                        const int rows[4] = {LMEP_ROW_W, LMEP_ROW_ALPHA, LMEP_ROW_BETA, LMEP_ROW_GAMMA};
                        const double *const X[4] = {XU, XN0, XS12, XN3};
                        fast_pass<NS, P, EX, 4>(p, lo, hi, rows, X, [&](int l, const double *v) {
                            XUN[l] = padd<EX>(padd<EX>(padd<EX>(v[0], v[1]), v[2]), v[3]);
                        });
                    }
                    __syncthreads();
                    if (s == 0 && p.nl0_out)
                        for (int64_t i = O0 + tid; i < O1; i += nt) p.nl0_out[i - p.off] = XN0[i - base];
                    const int newU = sl[UN], oldU = sl[U];
                    for (int r = 0; r < NR; ++r)
                        if (sl[r] == newU) sl[r] = oldU;
                    sl[U] = newU;
                }
                bool bad = false;
                for (int64_t i = O0 + tid; i < O1; i += nt) {
                    const double v = S(sl[U])[i - base];
                    store_out(p, i - p.off, v);
                    bad |= !isfinite(v);
                }
                if (bad) *p.flag = 1;
                return;
            }
        }
        if constexpr (cv) {
            sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[N3] = 3; sl[N1] = 4; sl[S12] = 4;
            sl[B] = 5; sl[C] = 5; sl[UN] = 6;
        } else {
            sl[U] = 0; sl[N0] = 1; sl[WH] = 2; sl[A] = 3; sl[UN] = 3; sl[N1] = 4; sl[C] = 4;
            sl[S12] = 5; sl[B] = 6; sl[N3] = 6;
        }
        for (int s = 0; s < K; ++s) {
            const int u0 = (K - 1 - s) * p.ext;
            double *XU = S(sl[U]), *XN0 = S(sl[N0]), *XWH = S(sl[WH]), *XA = S(sl[A]);
            double *XN1 = S(sl[N1]), *XB = S(sl[B]), *XS12 = S(sl[S12]), *XC = S(sl[C]);
            double *XN3 = S(sl[N3]), *XUN = S(sl[UN]);
            double *XT2 = XWH;
            int lo, hi;
            // P1: n0 = N(u)  (pointwise N: step 0 was fused into the load)
            expand(u0 + 4 + 3 * cv, lo, hi);
            if (!cv && s == 0) {
            } else if constexpr (cv) {
                const int rows[1] = {LMEP_ROW_D1};
                const double *const X[1] = {XU};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) { XN0[l] = nlp<EX>(nlk, XU[l], v[0]); });
            } else {
                run_pointwise(lo, hi, [&](int l) { XN0[l] = nlp<EX>(nlk, XU[l], 0.0); });
            }
            if (cv || s > 0) {
                refresh(XN0);
                __syncthreads();
            }
            // P2: whu = wh.u ; a = whu + p1h.n0 [pin] ; (pointwise N) n1 = N(a)
            expand(u0 + 3 + 3 * cv, lo, hi);
            {
                const int rows[2] = {LMEP_ROW_WHALF, LMEP_ROW_P1HALF};
                const double *const X[2] = {XU, XN0};
                run_pass<NS, P, EX, PN, 2>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) {
                        const double a = padd<EX>(v[0], v[1]);
                        XWH[l] = v[0];
                        XA[l] = a;
                        if constexpr (!cv) XN1[l] = nlp<EX>(nlk, a, 0.0);
                    });
            }
            pin_pass(XA, lo, hi, [&](int l, double v) { if constexpr (!cv) XN1[l] = nlp<EX>(nlk, v, 0.0); });
            refresh(XWH);
            refresh(XA);
            if constexpr (!cv) refresh(XN1);
            __syncthreads();
            // P3 (convective): n1 = N(a)
            if constexpr (cv) {
                expand(u0 + 3 + 2 * cv, lo, hi);
                const int rows[1] = {LMEP_ROW_D1};
                const double *const X[1] = {XA};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) { XN1[l] = nlp<EX>(nlk, XA[l], v[0]); });
                refresh(XN1);
                __syncthreads();
            }
            // P4: b = whu + p1h.n1 [pin] ; (pointwise N) n2 = N(b), t2 = 2 n2 - n0, s12 = n1 + n2
            expand(u0 + 2 + 2 * cv, lo, hi);
            {
                const int rows[1] = {LMEP_ROW_P1HALF};
                const double *const X[1] = {XN1};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) {
                        const double b = padd<EX>(XWH[l], v[0]);
                        XB[l] = b;
                        if constexpr (!cv) {
                            const double n2 = nlp<EX>(nlk, b, 0.0);
                            XT2[l] = sub2(n2, XN0[l]);
                            XS12[l] = padd<EX>(XN1[l], n2);
                        }
                    });
            }
            pin_pass(XB, lo, hi, [&](int l, double v) {
                if constexpr (!cv) {
                    const double n2 = nlp<EX>(nlk, v, 0.0);
                    XT2[l] = sub2(n2, XN0[l]);
                    XS12[l] = padd<EX>(XN1[l], n2);
                }
            });
            refresh(XB);
            if constexpr (!cv) { refresh(XT2); refresh(XS12); }
            __syncthreads();
            // P5 (convective): n2 = N(b), t2 = 2 n2 - n0, s12 = n1 + n2
            if constexpr (cv) {
                expand(u0 + 2 + cv, lo, hi);
                const int rows[1] = {LMEP_ROW_D1};
                const double *const X[1] = {XB};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) {
                        const double n2 = nlp<EX>(nlk, XB[l], v[0]);
                        XT2[l] = sub2(n2, XN0[l]);
                        XS12[l] = padd<EX>(XN1[l], n2);
                    });
                refresh(XT2);
                refresh(XS12);
                __syncthreads();
            }
            // P6: c = wh.a + p1h.t2 [pin] ; (pointwise N) n3 = N(c)
            expand(u0 + 1 + cv, lo, hi);
            {
                const int rows[2] = {LMEP_ROW_WHALF, LMEP_ROW_P1HALF};
                const double *const X[2] = {XA, XT2};
                run_pass<NS, P, EX, PN, 2>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) {
                        const double c = padd<EX>(v[0], v[1]);
                        XC[l] = c;
                        if constexpr (!cv) XN3[l] = nlp<EX>(nlk, c, 0.0);
                    });
            }
            pin_pass(XC, lo, hi, [&](int l, double v) { if constexpr (!cv) XN3[l] = nlp<EX>(nlk, v, 0.0); });
            refresh(XC);
            if constexpr (!cv) refresh(XN3);
            __syncthreads();
            // P7 (convective): n3 = N(c)
            if constexpr (cv) {
                expand(u0 + 1, lo, hi);
                const int rows[1] = {LMEP_ROW_D1};
                const double *const X[1] = {XC};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) { XN3[l] = nlp<EX>(nlk, XC[l], v[0]); });
                refresh(XN3);
                __syncthreads();
            }
            // P8: u' = ((w.u + alpha.n0) + beta.s12) + gamma.n3 [pin]
            expand(u0, lo, hi);
            {
                const int rows[4] = {LMEP_ROW_W, LMEP_ROW_ALPHA, LMEP_ROW_BETA, LMEP_ROW_GAMMA};
                const double *const X[4] = {XU, XN0, XS12, XN3};
                run_pass<NS, P, EX, PN, 4>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                    [&](int l, const double *v) {
                        XUN[l] = padd<EX>(padd<EX>(padd<EX>(v[0], v[1]), v[2]), v[3]);
                    });
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
            const double v = S(sl[U])[i - base];
            store_out(p, i - p.off, v);
            if (!isfinite(v)) *p.flag = 1;
        }
    } else {  // SCH_ETD2: exponential multistep of order ETDS (timestep.py:187-215)
        constexpr int so = ETDS;
        // slots: 0 u | 1..so-1 history N_{k-i} | so N_k | so+1..2so-1 grad^j N | 2so u'
        int iU = 0, iK = so, iV = 2 * so;
        int iq[so > 1 ? so - 1 : 1];
#pragma unroll
        for (int i = 1; i < so; ++i) iq[i - 1] = i;
        // interior fast path (see the ETDRK4 branch): every pass over the whole
        // staged range, no clamping, boundary path, pins or ghost refresh
        const bool fast = (!PN && NS > 0) && !ring && (p.periodic || (base >= p.L_int && gend <= p.R_int));
        for (int s = 0; fast && s < K; ++s) {
            if constexpr (!PN && NS > 0) {
                double *XU = S(iU), *XK = S(iK), *XV = S(iV);
                double *XQ[so > 1 ? so - 1 : 1];
#pragma unroll
                for (int i = 1; i < so; ++i) XQ[i - 1] = S(iq[i - 1]);
                auto epi1 = [&](int l, double du) {
                    const double nk = nlp<EX>(nlk, XU[l], du);
                    XK[l] = nk;
#pragma unroll
                    for (int j = 1; j < so; ++j) {
                        double g = EX ? xadd(0.0, nk) : nk;
                        int c = 1;
#pragma unroll
                        for (int i = 1; i <= j; ++i) {
                            c = -c * (j - i + 1) / i;
                            const double q = XQ[i - 1][l];
                            g = EX ? xadd(g, xmul((double)c, q)) : g + (double)c * q;
                        }
                        S(so + j)[l] = g;
                    }
                };
                if constexpr (cv) {
                    const int rows[1] = {LMEP_ROW_D1};
                    const double *const X[1] = {XU};
                    fast_pass<NS, P, EX, 1>(p, eL, len, rows, X, [&](int l, const double *v) { epi1(l, v[0]); });
                } else {
                    fast_pointwise<P>(0, len, [&](int l) { epi1(l, 0.0); });
                }
                __syncthreads();
                {
                    int rows[so + 1];
                    const double *X[so + 1];
                    rows[0] = LMEP_ROW_W;
                    X[0] = XU;
#pragma unroll
                    for (int j = 0; j < so; ++j) {
                        rows[j + 1] = LMEP_ROW_ALPHA + j;
                        X[j + 1] = j == 0 ? XK : S(so + j);
                    }
                    const int (&rr)[so + 1] = rows;
                    const double *const (&xx)[so + 1] = X;
                    fast_pass<NS, P, EX, so + 1>(p, eL, len, rr, xx, [&](int l, const double *v) {
                        double acc = padd<EX>(v[0], v[1]);
#pragma unroll
                        for (int j = 1; j < so; ++j) {
                            const double d = EX ? xdiv(v[j + 1], p.dtj[j]) : v[j + 1] * (1.0 / p.dtj[j]);
                            acc = padd<EX>(acc, d);
                        }
                        XV[l] = acc;
                    });
                }
                __syncthreads();
                if constexpr (so > 1) {
                    const int freed = iq[so - 2];
#pragma unroll
                    for (int i = so - 2; i > 0; --i) iq[i] = iq[i - 1];
                    iq[0] = iK;
                    iK = freed;
                }
                const int t = iU; iU = iV; iV = t;
            }
        }
        for (int s = 0; !fast && s < K; ++s) {
            const int u0 = (K - 1 - s) * p.ext;
            double *XU = S(iU), *XK = S(iK), *XV = S(iV);
            double *XQ[so > 1 ? so - 1 : 1];
#pragma unroll
            for (int i = 1; i < so; ++i) XQ[i - 1] = S(iq[i - 1]);
            int lo, hi;
            // P1: nk = N(u); grad^j N = sum_i (-1)^i C(j,i) N_{k-i}, accumulated from 0
            // in i order with separate roundings, as timestep.py:208 does
            expand(u0 + 1, lo, hi);
            auto epi1 = [&](int l, double du) {
                const double nk = nlp<EX>(nlk, XU[l], du);
                XK[l] = nk;
#pragma unroll
                for (int j = 1; j < so; ++j) {
                    double g = EX ? xadd(0.0, nk) : nk;
                    int c = 1;                                   // (-1)^i C(j, i)
#pragma unroll
                    for (int i = 1; i <= j; ++i) {
                        c = -c * (j - i + 1) / i;
                        const double q = XQ[i - 1][l];
                        g = EX ? xadd(g, xmul((double)c, q)) : g + (double)c * q;
                    }
                    S(so + j)[l] = g;
                }
            };
            if constexpr (cv) {
                const int rows[1] = {LMEP_ROW_D1};
                const double *const X[1] = {XU};
                run_pass<NS, P, EX, PN, 1>(p, lo, hi, fLo, fHi, base, lbase, rows, X,
                                           [&](int l, const double *v) { epi1(l, v[0]); });
            } else {
                run_pointwise(lo, hi, [&](int l) { epi1(l, 0.0); });
            }
            refresh(XK);
#pragma unroll
            for (int j = 1; j < so; ++j) refresh(S(so + j));
            __syncthreads();
            // P2: u' = W u + sum_j P_{j+1} grad^j N / dt^j   (timestep.py:206-210)
            expand(u0, lo, hi);
            {
                int rows[so + 1];
                const double *X[so + 1];
                rows[0] = LMEP_ROW_W;
                X[0] = XU;
#pragma unroll
                for (int j = 0; j < so; ++j) {
                    rows[j + 1] = LMEP_ROW_ALPHA + j;
                    X[j + 1] = j == 0 ? XK : S(so + j);
                }
                const int (&rr)[so + 1] = rows;
                const double *const (&xx)[so + 1] = X;
                run_pass<NS, P, EX, PN, so + 1>(p, lo, hi, fLo, fHi, base, lbase, rr, xx,
                    [&](int l, const double *v) {
                        double acc = padd<EX>(v[0], v[1]);      // /dt**0 == /1.0, exact
#pragma unroll
                        for (int j = 1; j < so; ++j) {
                            const double d = EX ? xdiv(v[j + 1], p.dtj[j]) : v[j + 1] * (1.0 / p.dtj[j]);
                            acc = padd<EX>(acc, d);
                        }
                        XV[l] = acc;
                    });
            }
            pin_pass(XV, lo, hi, none);
            refresh(XV);
            __syncthreads();
            // history <- (nk, N_{k-1}, ...), u <- u'
            if constexpr (so > 1) {
                const int freed = iq[so - 2];
#pragma unroll
                for (int i = so - 2; i > 0; --i) iq[i] = iq[i - 1];
                iq[0] = iK;
                iK = freed;
            }
            const int t = iU; iU = iV; iV = t;
        }
        bool bad = false;
        double *XQ[so > 1 ? so - 1 : 1];
#pragma unroll
        for (int i = 1; i < so; ++i) XQ[i - 1] = S(iq[i - 1]);
        for (int64_t i = O0 + tid; i < O1; i += nt) {
            const double v = S(iU)[i - base];
            store_out(p, i - p.off, v);
#pragma unroll
            for (int j = 1; j < so; ++j) p.q_out[(int64_t)(j - 1) * p.qld + (i - p.off)] = XQ[j - 1][i - base];
            bad |= !isfinite(v);
        }
        if (bad) *p.flag = 1;
    }
#undef S
}

// Per-node rows of the ETD schemes use the generic-n instantiation only, as do
// ETD orders other than 2.
template <int SCH, bool EX, int P, int NLK, bool PN = false, int ETDS = 2>
inline int launch_ns(int ns_case, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    void (*k)(StepParams) = nullptr;
    if (SCH != SCH_LIN && p.wmode == LMEP_W_PERNODE) {
        k = step_kernel<SCH, 0, EX, P, NLK, true, ETDS>;
    } else if (ETDS != 2) {
        k = step_kernel<SCH, 0, EX, P, NLK, PN, ETDS>;
    } else {
        switch (ns_case) {
        case 7: k = step_kernel<SCH, 7, EX, P, NLK, PN>; break;
        case 9: k = step_kernel<SCH, 9, EX, P, NLK, PN>; break;
        case 11: k = step_kernel<SCH, 11, EX, P, NLK, PN>; break;
        case 13: k = step_kernel<SCH, 13, EX, P, NLK, PN>; break;
        default: k = step_kernel<SCH, 0, EX, P, NLK, PN>; break;
        }
    }
    if (shm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) { set_last_error("cudaFuncSetAttribute", e); return LMEP_CUDA_ERROR; }
    }
    k<<<grid, p.threads, shm, st>>>(p);
    return launch_status("step_kernel");
}

int launch_scheme_lin(bool pernode, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st);
int launch_lin_pernode(const StepParams &p, cudaStream_t st);
int launch_lin_pernode_tb(const StepParams &p, bool exact, cudaStream_t st);
int tb_nodes_per_cta(int n, bool tma);
int launch_lin_pernode_tma(const StepParams &p, bool exact, cudaStream_t st);
int try_launch_etd2_persistent(StepParams &p, int nl, bool exact, int64_t steps, cudaStream_t st);
#define STEP_DECL(S, L) \
    int launch_scheme_##S##_##L(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st);
STEP_DECL(etdrk4, none)
STEP_DECL(etdrk4, convective)
STEP_DECL(etdrk4, cubic)
STEP_DECL(etd2, none)
STEP_DECL(etd2, convective)
STEP_DECL(etd2, cubic)
#undef STEP_DECL

}  // namespace lmep
