// step_lin.cu -- instantiations of the linear step kernel.
#include <algorithm>

#include <cooperative_groups.h>

#include "step.cuh"

namespace cg = cooperative_groups;

namespace lmep {

// set by lmep_set_ring_cluster (capi.cu): 1 = cluster ring kernel when eligible

// Ring mode for the linear scheme (a periodic grid resident in one CTA, C1:
// N = 1024, 1000 steps in one launch).  The whole run is one SM, so the
// per-step latency chain and the SM's shared-memory bandwidth are the cost:
// each thread owns P consecutive nodes and loads one register window of
// P + n - 1 values (odd P: the lane stride hits distinct bank pairs), then
// runs P interleaved chains of the reference's ascending unfused
// multiply-adds (kernels.py:23-29).  Ghost mirrors are written by their
// producers, so there is one barrier per step.
template <int NS, int P>
__global__ void __launch_bounds__(1024) ring_lin_kernel(const __grid_constant__ StepParams p)
{
    extern __shared__ double rsm[];
    const int N = (int)p.N, eL = p.eL, eR = p.eR;
    const int span = N + eL + eR;
    const int slot = span + P + NS;               // overhang of the last window / chunk
    double *X0 = rsm, *X1 = rsm + slot;
    for (int i = threadIdx.x; i < span; i += blockDim.x) {
        int64_t g = (int64_t)i - eL;
        g = g < 0 ? g + N : (g >= N ? g - N : g);
        X0[i] = p.u_in[g];
    }
    __syncthreads();
    double w[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) w[j] = p.wi[LMEP_ROW_W][j];
    const int K = p.ksteps;
    for (int s = 0; s < K; ++s) {
#pragma unroll 1
        for (int i0 = P * threadIdx.x; i0 < N; i0 += P * blockDim.x) {
            const double *x = X0 + i0;                // window of node i0: staged i0 .. i0 + n - 1
            double win[P + NS - 1];
#pragma unroll
            for (int q = 0; q < P + NS - 1; ++q) win[q] = x[q];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int i = i0 + q;
                double acc = xmul(w[0], win[q]);
#pragma unroll
                for (int j = 1; j < NS; ++j) acc = xadd(acc, xmul(w[j], win[q + j]));
                if (i < N) {
                    X1[eL + i] = acc;
                    if (i >= N - eL) X1[i - (N - eL)] = acc;  // left ghosts mirror nodes N - eL ..
                    if (i < eR) X1[eL + N + i] = acc;         // right ghosts mirror nodes 0 .. eR - 1
                }
            }
        }
        __syncthreads();
        double *t = X0; X0 = X1; X1 = t;
    }
    bool bad = false;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const double v = X0[eL + i];
        p.u_out[i] = v;
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

// Ring mode over a thread-block CLUSTER: the periodic grid is split into C
// slabs of M = N / C nodes, one per CTA of one cluster (C SMs instead of one).
// Each block of kb steps starts by gathering eL*kb / eR*kb halo nodes from the
// neighbouring CTAs' shared memory (DSMEM, cluster.map_shared_rank), then the
// CTA advances kb steps on its extended range with CTA-local barriers
// (temporal blocking: the stale halo edges move inward by eL / eR per step and
// never reach the owned nodes), and publishes its owned nodes back.  Two
// cluster barriers per kb steps replace kb whole-grid barriers; the arithmetic
// is the reference's ascending unfused order, bit-identical.
template <int NS>
__global__ void __launch_bounds__(1024) ring_lin_cluster_kernel(const __grid_constant__ StepParams p, int kb)
{
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
    const int N = (int)p.N, M = N / C, eL = p.eL, eR = p.eR;
    const int HL = eL * kb, HR = eR * kb, span = HL + M + HR;
    extern __shared__ double csm[];
    double *own = csm;                            // [M] this slab's state at block boundaries
    double *A = csm + M, *B = A + span;           // ping-pong over the extended range
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < M; i += nt) own[i] = p.u_in[(int64_t)r * M + i];
    double w[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) w[j] = p.wi[LMEP_ROW_W][j];
    cl.sync();
    const double *lown = cl.map_shared_rank(own, (r + C - 1) % C);
    const double *rown = cl.map_shared_rank(own, (r + 1) % C);
    const int K = p.ksteps;
    for (int s0 = 0; s0 < K; s0 += kb) {
        const int ks = K - s0 < kb ? K - s0 : kb;
        for (int i = tid; i < span; i += nt)
            A[i] = i < HL ? lown[M - HL + i] : (i < HL + M ? own[i - HL] : rown[i - HL - M]);
        cl.sync();                                // neighbours' own[] read: it may be rewritten
        for (int j = 0; j < ks; ++j) {
            for (int i = eL + tid; i < span - eR; i += nt) {
                const double *x = A + i - eL;
                double acc = xmul(w[0], x[0]);
#pragma unroll
                for (int c = 1; c < NS; ++c) acc = xadd(acc, xmul(w[c], x[c]));
                B[i] = acc;
            }
            __syncthreads();
            double *t = A; A = B; B = t;
        }
        for (int i = tid; i < M; i += nt) own[i] = A[HL + i];
        cl.sync();                                // own[] complete before the next gather
    }
    bool bad = false;
    for (int i = tid; i < M; i += nt) {
        const double v = own[i];
        p.u_out[(int64_t)r * M + i] = v;
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

// Ring mode, warp-private slabs (small rings, BASELINE config 1): the same
// cluster of C CTAs, but inside a block of kb steps nothing is shared at all.
// Every WARP owns N / (4 C) consecutive nodes and carries its own halo of
// kb * eL / kb * eR nodes; each lane keeps J consecutive staged nodes in
// REGISTERS and builds its windows with warp shuffles from the one or two
// lanes next to it.  A step is shuffles + the n-tap chain: no shared-memory
// round trip and no barrier (the one-node-per-thread kernel above spent a
// store, a CTA barrier and n loads per step).  The warp's stale edge lanes
// move inward by eL / eR nodes per step and never reach its owned nodes.
// Between blocks the warps publish their owned nodes in the CTA's shared
// memory and gather the next halos from their own and the neighbouring CTAs'
// (DSMEM), two cluster barriers per block as above.  Arithmetic: the
// reference's ascending unfused chain, bit-identical.
template <int NS, int EL, int J>
__global__ void __launch_bounds__(128) ring_lin_warp_kernel(const __grid_constant__ StepParams p, int kb)
{
    constexpr int W = J + NS - 1;                               // staged offsets -EL .. J-1+ER
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
    const int N = (int)p.N, M = N / C, mw = M / 4;
    const int HL = EL * kb;
    extern __shared__ double csm[];
    // [2][M] this CTA's nodes between blocks, double buffered: block b gathers from
    // half b & 1 and publishes into the other, so ONE cluster barrier per block
    // orders both (every gather of half b & 1 precedes that barrier, and the next
    // store into it follows the barrier after)
    double *own = csm;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < M; i += 128) own[i] = p.u_in[(int64_t)r * M + i];
    double w[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) w[j] = p.wi[LMEP_ROW_W][j];
    // lane's staged nodes: ring index g0 + j, j < J (the warp's range starts HL before its owned nodes)
    const int ws = r * M + wid * mw;                            // first owned node of this warp
    int gr[J], gi[J];                                           // owner CTA and index of each staged node
#pragma unroll
    for (int j = 0; j < J; ++j) {
        int g = (ws - HL + lane * J + j) % N;
        if (g < 0) g += N;
        gr[j] = g / M;
        gi[j] = g % M;
    }
    cl.sync();
    const int K = p.ksteps;
    double x[J];
    int half = 0;
    for (int s0 = 0; s0 < K; s0 += kb, half ^= 1) {
        const int ks = K - s0 < kb ? K - s0 : kb;
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = cl.map_shared_rank(own + half * M, gr[j])[gi[j]];
        for (int st = 0; st < ks; ++st) {
            double win[W];                                      // staged offsets -EL .. J-1+ER of this lane
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const int o = i - EL;
                if (o < 0) {
                    const int d = (-o + J - 1) / J;             // lanes to the left
                    win[i] = __shfl_up_sync(FULL, x[o + d * J], d);
                } else if (o < J) {
                    win[i] = x[o];
                } else {
                    win[i] = __shfl_down_sync(FULL, x[o % J], o / J);
                }
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                double acc = xmul(w[0], win[j]);
#pragma unroll
                for (int c = 1; c < NS; ++c) acc = xadd(acc, xmul(w[c], win[j + c]));
                x[j] = acc;
            }
        }
        // owned nodes of the warp: staged offsets HL .. HL + mw - 1
        double *nxt = own + (half ^ 1) * M;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int so = lane * J + j - HL;
            if (so >= 0 && so < mw) nxt[wid * mw + so] = x[j];
        }
        cl.sync();                                              // published; the old half is free
    }
    bool bad = false;
    const double *fin = own + half * M;
    for (int i = tid; i < M; i += 128) {
        const double v = fin[i];
        p.u_out[(int64_t)r * M + i] = v;
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

template <int J>
static int launch_ring_warp_j(const StepParams &p, int kb, cudaStream_t st)
{
    void (*k)(StepParams, int) = nullptr;
    if (p.n == 7 && p.row == 6) k = ring_lin_warp_kernel<7, 6, J>;
    else if (p.n == 7 && p.row == 3) k = ring_lin_warp_kernel<7, 3, J>;
    else if (p.n == 7 && p.row == 0) k = ring_lin_warp_kernel<7, 0, J>;
    else if (p.n == 9 && p.row == 4) k = ring_lin_warp_kernel<9, 4, J>;
    else if (p.n == 11 && p.row == 5) k = ring_lin_warp_kernel<11, 5, J>;
    else if (p.n == 13 && p.row == 6) k = ring_lin_warp_kernel<13, 6, J>;
    if (!k) return -1;
    constexpr int C = 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = (size_t)2 * (p.N / C) * sizeof(double);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, p, kb);
    if (e != cudaSuccess) { set_last_error("cudaLaunchKernelEx(ring_lin_warp_kernel)", e); return LMEP_CUDA_ERROR; }
    return launch_status("ring_lin_warp_kernel");
}

// small rings: N a multiple of 32 (8 CTAs x 4 warps) whose per-warp slab plus a
// halo of at least 4 steps fits J <= 4 nodes per lane
static int launch_ring_warp(const StepParams &p, cudaStream_t st)
{
    const int variant = device_settings().ring_cluster.load();
    if (variant == 2) return -1;                                // 2: the shared-memory cluster kernel
    if (p.N % 32 != 0) return -1;
    const int mw = (int)(p.N / 32), reach2 = p.eL + p.eR;
    if (reach2 == 0) return -1;
    for (int J = 4; J >= 3; --J) {                              // deepest halo first: fewer cluster barriers
        const int kb = (32 * J - mw) / reach2;
        if (kb < 4) continue;
        // (halo of the first lanes must come from real nodes: kb * eL, kb * eR <= N)
        if ((int64_t)kb * std::max(p.eL, p.eR) > p.N) continue;
        return J == 3 ? launch_ring_warp_j<3>(p, kb, st) : launch_ring_warp_j<4>(p, kb, st);
    }
    return -1;
}

static int launch_ring_cluster(const StepParams &p, cudaStream_t st)
{
    constexpr int C = 8;
    const int reach = std::max(p.eL, p.eR);
    if (p.N % C != 0 || reach == 0) return -1;
    const int M = (int)(p.N / C);
    // a cluster barrier costs ~0.4 us, a local step ~0.25 us: take the deepest
    // halo that still comes from the adjacent slabs only (eL*kb, eR*kb <= M)
    const int kb = std::min(32, M / reach);
    if (kb < 2) return -1;
    const int span = p.eL * kb + M + p.eR * kb;
    const int threads = std::min(1024, (span + 31) / 32 * 32);
    const size_t shm = (size_t)(M + 2 * span) * sizeof(double);
    void (*k)(StepParams, int) = p.n == 7 ? ring_lin_cluster_kernel<7> : p.n == 9 ? ring_lin_cluster_kernel<9>
                                 : p.n == 11 ? ring_lin_cluster_kernel<11> : ring_lin_cluster_kernel<13>;
    if (shm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) return -1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, p, kb);
    if (e != cudaSuccess) { set_last_error("cudaLaunchKernelEx(ring_lin_cluster_kernel)", e); return LMEP_CUDA_ERROR; }
    return launch_status("ring_lin_cluster_kernel");
}

int launch_scheme_lin(bool pernode, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (pernode) return launch_ns<SCH_LIN, true, 1, LMEP_NL_NONE, true>(p.n, p, grid, shm, st);
    if (p.ring && p.off == 0 && p.hl == nullptr && p.hr == nullptr && p.wmode == LMEP_W_SHARED &&
        (p.n == 7 || p.n == 9 || p.n == 11 || p.n == 13)) {
        if (device_settings().ring_cluster.load()) {
            int rc = launch_ring_warp(p, st);        // small rings: warp-private slabs in registers
            if (rc >= 0) return rc;
            rc = launch_ring_cluster(p, st);
            if (rc >= 0) return rc;                  // else: shape not eligible, one-CTA kernel
        }
        constexpr int RP = 3;
        const int threads = (int)std::min<int64_t>(1024, ((p.N + RP - 1) / RP + 31) / 32 * 32);
        const size_t rshm = (size_t)2 * (p.N + p.eL + p.eR + RP + p.n) * sizeof(double);
        void (*k)(StepParams) = p.n == 7 ? ring_lin_kernel<7, RP> : p.n == 9 ? ring_lin_kernel<9, RP>
                                : p.n == 11 ? ring_lin_kernel<11, RP> : ring_lin_kernel<13, RP>;
        if (rshm > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rshm);
            if (e != cudaSuccess) { set_last_error("cudaFuncSetAttribute", e); return LMEP_CUDA_ERROR; }
        }
        k<<<1, threads, rshm, st>>>(p);
        return launch_status("ring_lin_kernel");
    }
    return launch_ns<SCH_LIN, true, 5, LMEP_NL_NONE>(p.n, p, grid, shm, st);
}

}  // namespace lmep

namespace lmep {

// Per-node linear step without boundary closure (BASELINE config 5): a lean
// streaming kernel.  Each thread produces PPT outputs spaced blockDim apart
// (coalesced SoA weight loads, all PPT*n loads of a thread issued before the
// accumulations); u is read straight from global memory, where neighbouring
// threads' windows overlap in L1.  Arithmetic is the EXACT ascending order of
// kernels.py:23-29, so it is bit-identical to the generic engine.
template <int NS, int PPT>
__global__ void __launch_bounds__(256) lin_pernode_kernel(const __grid_constant__ StepParams p)
{
    const int n = NS > 0 ? NS : p.n;
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * PPT + threadIdx.x;
    const bool single = p.hl == nullptr && p.hr == nullptr;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int64_t li = base + (int64_t)k * blockDim.x;
        if (li >= p.nloc) break;
        const int64_t g = p.off + li;
        int64_t st = g - p.row;
        if (!p.periodic) st = st < 0 ? 0 : (st > p.N - n ? p.N - n : st);
        const double *w = p.wp + li + p.wpad;
        double acc = 0.0;
        if (single && p.periodic && st >= 0 && st + n <= p.N) {
            const double *u = p.u_in + st;
#pragma unroll
            for (int j = 0; j < (NS > 0 ? NS : 1); ++j) {
                if (NS == 0) break;
                acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.wld), __ldg(u + j)));
            }
            if (NS == 0)
                for (int j = 0; j < n; ++j)
                    acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.wld), __ldg(u + j)));
        } else {
            for (int j = 0; j < n; ++j)
                acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.wld),
                                     load_node(p, p.u_in, p.hl, p.hr, st + j)));
        }
        p.u_out[li] = acc;
        if (!isfinite(acc)) *p.flag = 1;
    }
}

int launch_lin_pernode(const StepParams &p, cudaStream_t st)
{
    constexpr int PPT = 4, TPB = 256;
    const int64_t blocks = (p.nloc + (int64_t)TPB * PPT - 1) / ((int64_t)TPB * PPT);
    if (p.n == 13) lin_pernode_kernel<13, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 7) lin_pernode_kernel<7, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 9) lin_pernode_kernel<9, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 11) lin_pernode_kernel<11, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else lin_pernode_kernel<0, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    return launch_status("lin_pernode_kernel");
}

}  // namespace lmep

namespace lmep {

// Per-node linear steps with temporal blocking (periodic, no closure): a CTA
// stages u over its tile plus k*(n-1) halo nodes in shared memory and holds
// the per-node rows of every node it computes in REGISTERS, then advances k
// steps on chip.  The 8n bytes of rows per node cross HBM once per k steps
// instead of once per step.
//
// Thread t owns the J CONSECUTIVE staged nodes J*t .. J*t+J-1: one sliding
// window of J+n-1 shared-memory loads serves its J outputs (J odd: the
// stride-J lane pattern is bank-conflict free for 8-byte words), and the J
// accumulation chains interleave.  Every thread computes all its nodes every
// step (no per-node predicates, so the chains stay in one basic block); the
// staged buffers carry eL / eR pad words so edge windows stay in bounds, and
// values outside the shrinking valid range are never consumed.
// Arithmetic: the ascending, unfused order of kernels.py:23-29, with the
// chain started at the first product (0 + p0 == p0 up to the sign of zero),
// so results equal the one-step kernels.  !EX: the same chain as FMAs.
template <int NS, int J, bool EX>
__global__ void __launch_bounds__(256, 2) lin_pernode_tb_kernel(const __grid_constant__ StepParams p)
{
    extern __shared__ double sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int K = p.ksteps;
    const int eL = p.row, eR = NS - 1 - p.row;
    // tile of this shard (local indices), staged range in global indices
    const int64_t t0 = (int64_t)blockIdx.x * p.tile;
    const int64_t t1 = t0 + p.tile < p.nloc ? t0 + p.tile : p.nloc;
    const int64_t base = p.off + t0 - (int64_t)K * eL;
    const int len = (int)(t1 - t0) + K * (eL + eR);
    const bool single = p.hl == nullptr && p.hr == nullptr;
    // staged node l lives at U[eL + l]; U[0, eL) and U[eL + len, ...) are pads
    double *U0 = sm, *U1 = sm + p.slot_len;
    const int span = J * nt;
    for (int i = tid; i < span + NS - 1; i += nt) {
        const int l = i - eL;
        U0[i] = (l >= 0 && l < len) ? load_node(p, p.u_in, p.hl, p.hr, base + l) : 0.0;
        U1[i] = 0.0;
    }
    // rows: single shard -> the periodic grid's own table (wrap); sharded ->
    // this shard's table, padded with the rows of wpad halo nodes per side.
    // The J loads of one tap cover J*32 consecutive doubles per warp (L1 hits).
    double w[J][NS];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int l = J * tid + j;
        const int64_t g = base + (l < len ? l : (int64_t)K * eL);
        const int64_t wi = single ? wrap(g, p.N) : g - p.off + p.wpad;
#pragma unroll
        for (int c = 0; c < NS; ++c) w[j][c] = __ldg(p.wp + (int64_t)c * p.wld + wi);
    }
    __syncthreads();
    for (int s = 0; s < K; ++s) {
        const double *x = U0 + J * tid;          // window of node J*tid starts at U[J*tid]
        double acc[J];
#pragma unroll
        for (int i = 0; i < J + NS - 1; ++i) {
            const double v = x[i];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int c = i - j;
                if constexpr (EX) {
                    if (c == 0) acc[j] = xmul(w[j][0], v);
                    else if (c > 0 && c < NS) acc[j] = xadd(acc[j], xmul(w[j][c], v));
                } else {
                    if (c == 0) acc[j] = w[j][0] * v;
                    else if (c > 0 && c < NS) acc[j] = fma(w[j][c], v, acc[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < J; ++j) U1[eL + J * tid + j] = acc[j];
        __syncthreads();
        double *t = U0; U0 = U1; U1 = t;
    }
    bool bad = false;
    for (int64_t i = t0 + tid; i < t1; i += nt) {
        const double v = U0[eL + (int)(i + K * eL - t0)];
        p.u_out[i] = v;
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

// nodes per CTA staged range = J * 256; returns 0 if not applicable
// tma: the persistent kernel (step_lin_tma.cu, 3 x 512 nodes), else 3 x 256
int tb_nodes_per_cta(int n, bool tma)
{
    if (!(n == 13 || n == 11 || n == 9 || n == 7)) return 0;
    if (tma && device_settings().pernode_kernel.load() == 3) return 6 * 128;   // two CTAs per SM
    return 3 * (tma ? 512 : 256);
}

int launch_lin_pernode_tb(const StepParams &p, bool exact, cudaStream_t st)
{
    constexpr int J = 3, TPB = 256;
    const int64_t blocks = (p.nloc + p.tile - 1) / p.tile;
    const size_t shm = 2 * (size_t)p.slot_len * 8;
    switch (p.n) {
    case 13:
        if (exact) lin_pernode_tb_kernel<13, J, true><<<(unsigned)blocks, TPB, shm, st>>>(p);
        else lin_pernode_tb_kernel<13, J, false><<<(unsigned)blocks, TPB, shm, st>>>(p);
        break;
    case 11:
        if (exact) lin_pernode_tb_kernel<11, J, true><<<(unsigned)blocks, TPB, shm, st>>>(p);
        else lin_pernode_tb_kernel<11, J, false><<<(unsigned)blocks, TPB, shm, st>>>(p);
        break;
    case 9:
        if (exact) lin_pernode_tb_kernel<9, J, true><<<(unsigned)blocks, TPB, shm, st>>>(p);
        else lin_pernode_tb_kernel<9, J, false><<<(unsigned)blocks, TPB, shm, st>>>(p);
        break;
    case 7:
        if (exact) lin_pernode_tb_kernel<7, J, true><<<(unsigned)blocks, TPB, shm, st>>>(p);
        else lin_pernode_tb_kernel<7, J, false><<<(unsigned)blocks, TPB, shm, st>>>(p);
        break;
    default: return LMEP_INVALID_CONFIG;
    }
    return launch_status("lin_pernode_tb_kernel");
}

}  // namespace lmep

extern "C" int lmep_set_ring_cluster(int on)
{
    if (on < 0 || on > 2) return LMEP_INVALID_CONFIG;
    lmep::device_settings().ring_cluster.store(on);
    return LMEP_OK;
}
