// step_lin_tma.cu -- persistent, TMA-pipelined per-node linear steps
// (BASELINE config 5: periodic grid, one shard, per-node rows, no closure).
//
// Same schedule and arithmetic as lin_pernode_tb_kernel (step_lin.cu): a tile
// of the grid plus k*(n-1) halo nodes is staged on chip, each thread holds the
// per-node rows of its J consecutive staged nodes in registers, and the CTA
// advances k steps with one barrier per step; the rows cross HBM once per k
// steps.  What changes is that the loads of tile i+1 overlap the k steps of
// tile i:
//
//   * one CTA per SM (persistent, tiles strided by gridDim.x);
//   * one elected thread moves the next tile's rows ([n][span] slice of the
//     SoA table) and its u into shared memory with 1-D bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx), issued as soon as every
//     thread has copied the current tile's rows from shared memory into its
//     registers, so HBM streams while the FP64 pipe works;
//   * three u buffers rotate: the landed tile's initial state, its ping-pong
//     partner, and the target of the next tile's copy.
//
// Bulk copies need 16-byte aligned sources and sizes, so each row / u slice
// is fetched from the even node at or below the staged range start and the
// smem origin is shifted by that parity (`o`).  Periodic wrap splits a slice
// into two copies.  Arithmetic (EX): the ascending unfused order of
// kernels.py:23-29, bit-identical to the other per-node step kernels; !EX
// (LMEP_FLAG_EXACT clear): the same ascending chain as fused multiply-adds.
// Launch shape J = 3, NT = 512 measured best against (J, NT) = (5, 288),
// (5, 256), (7, 192): more nodes per thread cut shared-memory wavefronts but
// the fewer resident warps expose the per-step barrier and load latency.
#include "step.cuh"

namespace lmep {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// programmatic dependent launch: let the next launch on the stream start its
// prologue as SMs free up / wait until the launch before this one has completed
// and its stores are visible (no-ops for a launch without the attribute)
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// staged range of tile `tile`: global nodes [base, base + len), fetched from
// the even node `start` = base - o, cnt (even) nodes, wrapping at N
struct TileRange {
    int64_t t0, t1, base, start;
    int len, o, cnt;
};

__device__ __forceinline__ TileRange tile_range(const StepParams &p, int64_t tile, int K, int eL, int eR)
{
    TileRange r;
    if (p.tile_wrap > 0 && tile >= p.tile_wrap) tile -= p.tile_wrap;   // a launch over [lo, wrap + hi')
    // slabs (p.ext_off > 0): u_in and the row table are the slab's extended arrays
    // [ghosts | owned | ghosts] of p.N nodes, the owned nodes ext_off .. ext_off+nloc-1;
    // the staged ranges never wrap there
    r.t0 = p.ext_off + tile * p.tile;
    r.t1 = r.t0 + p.tile < p.ext_off + p.nloc ? r.t0 + p.tile : p.ext_off + p.nloc;
    r.len = (int)(r.t1 - r.t0) + K * (eL + eR);
    int64_t b = (r.t0 - (int64_t)K * eL) % p.N;
    if (b < 0) b += p.N;
    r.base = b;
    r.o = (int)(b & 1);
    r.start = b - r.o;
    r.cnt = (r.len + r.o + 1) & ~1;
    return r;
}

// copy cnt doubles of the periodic vector v (length N, even) starting at the
// even index `start` into dst: one or two bulk copies; returns the byte count
__device__ __forceinline__ uint32_t copy_wrapped(double *dst, const double *v, int64_t N,
                                                 int64_t start, int cnt, uint64_t *bar)
{
    const int64_t first = start + cnt <= N ? cnt : N - start;
    bulk_g2s(dst, v + start, (uint32_t)(first * 8), bar);
    if (first < cnt) bulk_g2s(dst + first, v, (uint32_t)((cnt - first) * 8), bar);
    return (uint32_t)cnt * 8u;
}

}  // namespace

// u buffer length (even, so every buffer starts 16-byte aligned)
__host__ __device__ constexpr int tma_ulen(int n, int span) { return (span + n + 5) & ~1; }

template <int NS, int J, int NT, bool EX>
__global__ void __launch_bounds__(NT, 1) lin_pernode_tma_kernel(const __grid_constant__ StepParams p)
{
    constexpr int SPAN = J * NT;
    constexpr int RS = SPAN + 4;                 // row slice stride (even: 16-byte aligned)
    constexpr int UL = tma_ulen(NS, SPAN);       // u buffer: pads for eL/eR and the parity shift
    extern __shared__ __align__(16) double sm[];
    double *R = sm;                              // [NS][RS]
    double *Ub = sm + NS * RS;                   // [3][UL]
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int K = p.ksteps;
    const int eL = p.row, eR = NS - 1 - p.row;
    const int64_t ntiles = p.tile_hi > 0 ? p.tile_hi : (p.nloc + p.tile - 1) / p.tile;

    // (the row slices are always overwritten by the bulk copies before they are read)
    for (int i = tid; i < 3 * UL; i += NT) Ub[i] = 0.0;
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // buffer b's origin: staged node l of a tile at Ub[b*UL + org + l] with
    // org - o even, so the bulk copy destination (org - o) is 16-byte aligned
    // dep (first tile of a programmatic dependent launch): 1 = wait for the launch
    // before this one between the row copies and the u copy, 2 = before both
    auto issue = [&](int64_t tile, int b, int dep) {
        const TileRange r = tile_range(p, tile, K, eL, eR);
        const int org = eL + ((eL - r.o) & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const uint32_t bytes = (uint32_t)r.cnt * 8u * (NS + 1);
        if (dep == 2) griddep_wait();
        mbar_expect_tx(&bar, bytes);
#pragma unroll 1
        for (int c = 0; c < NS; ++c)
            copy_wrapped(R + c * RS, p.wp + (int64_t)c * p.wld, p.N, r.start, r.cnt, &bar);
        if (dep == 1) griddep_wait();
        copy_wrapped(Ub + b * UL + org - r.o, p.u_in, p.N, r.start, r.cnt, &bar);
    };

    if (p.pdl) griddep_launch();
    int64_t tile = p.tile_lo + blockIdx.x;
    if (tid == 0 && tile < ntiles) issue(tile, 0, p.pdl);
    if (p.pdl) griddep_wait();
    bool bad = false;
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const TileRange r = tile_range(p, tile, K, eL, eR);
        const int org = eL + ((eL - r.o) & 1);
        const int bT = it % 3, bP = (it + 2) % 3;
        mbar_wait(&bar, (uint32_t)(it & 1));
        // rows of this thread's J consecutive staged nodes -> registers
        double w[J][NS];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int l = J * tid + j;
            const int ls = r.o + (l < r.len ? l : K * eL);
#pragma unroll
            for (int c = 0; c < NS; ++c) w[j][c] = R[c * RS + ls];
        }
        __syncthreads();                         // R free, previous tile's outputs stored
        const int64_t nxt = tile + gridDim.x;
        if (tid == 0 && nxt < ntiles) issue(nxt, (it + 1) % 3, 0);

        double *U0 = Ub + bT * UL + org - eL, *U1 = Ub + bP * UL + org - eL;
        for (int s = 0; s < K; ++s) {
            const double *x = U0 + J * tid;      // window of staged node J*tid
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
        for (int64_t i = r.t0 + tid; i < r.t1; i += NT) {
            const double v = U0[eL + (int)(i - r.t0) + K * eL];
            p.u_out[i - p.ext_off] = v;
            bad |= !isfinite(v);
        }
    }
    if (bad) *p.flag = 1;
}

// ---------------------------------------------------------------------------
// Register-resident variant (lin_pernode_tmx_kernel): the same tiles, TMA
// pipeline, launch plan and arithmetic, but each thread keeps its J = 6
// consecutive staged nodes' VALUES in registers across the k steps, not just
// their rows.  Per step a thread publishes its J values into a structure-of-
// arrays exchange buffer Q[slot j][thread] and reads back only the halo it
// needs -- the last EL values of thread t-1 and the first ER values of thread
// t+1 (EL, ER <= J) -- so the window of J + n - 1 values costs n - 1 shared
// loads and J stores per thread instead of J + n - 1 loads and J stores: for
// n = 13 (J = 6, 256 threads) 24 B of shared-memory traffic per output instead
// of 40 (the J = 3 kernel above was bound by those wavefronts, ncu
// profiles/r1s_c5_lin_pernode_tma_kernel.md).  Slot-major Q makes every load /
// store of a warp hit consecutive 8-byte words (conflict-free); Q is double
// buffered, so one barrier per step suffices.  Rows and the initial values
// are read from the TMA-staged natural layout with 16-byte loads (conflict-
// free at a 48-byte lane stride).  The accumulation order is the same
// ascending chain as every other per-node kernel (bit-identical in EX).
// ---------------------------------------------------------------------------
#ifdef LMEP_TMX_TIMING
// diagnostic builds (-DLMEP_TMX_TIMING): per-tile phase timestamps of two CTAs
__device__ long long g_tmx_timing[512];
#endif

template <int NS, int EL, int J, int NT, bool EX, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) lin_pernode_tmx_kernel(const __grid_constant__ StepParams p)
{
    constexpr int ER = NS - 1 - EL;
    static_assert(EL <= 2 * J && ER <= 2 * J && J % 2 == 0, "halo must come from the two nearest threads per side");
    constexpr int SPAN = J * NT;
    constexpr int RS = SPAN + 4;                 // row slice stride (even: 16-byte aligned)
    constexpr int UL = tma_ulen(NS, SPAN);
    constexpr int QS = NT + 4;                   // exchange slot stride (thread t at 2 + t)
    constexpr int W = EL + J + ER;               // window
    extern __shared__ __align__(16) double sm[];
    double *R = sm;                              // [NS][RS]
    double *Ub = sm + NS * RS;                   // [UL] landed initial values
    double *Q = Ub + UL;                         // [2][J][QS]
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int K = p.ksteps;
    const int eL = EL, eR = ER;
    const int64_t ntiles = p.tile_hi > 0 ? p.tile_hi : (p.nloc + p.tile - 1) / p.tile;

    // (the row slices are always overwritten by the bulk copies before they are read)
    for (int i = tid; i < UL + 2 * J * QS; i += NT) Ub[i] = 0.0;
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int64_t tile, int dep) {
        const TileRange r = tile_range(p, tile, K, eL, eR);
        const int org = eL + ((eL - r.o) & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const uint32_t bytes = (uint32_t)r.cnt * 8u * (NS + 1);
        if (dep == 2) griddep_wait();
        mbar_expect_tx(&bar, bytes);
#pragma unroll 1
        for (int c = 0; c < NS; ++c)
            copy_wrapped(R + c * RS, p.wp + (int64_t)c * p.wld, p.N, r.start, r.cnt, &bar);
        if (dep == 1) griddep_wait();
        copy_wrapped(Ub + org - r.o, p.u_in, p.N, r.start, r.cnt, &bar);
    };

    if (p.pdl) griddep_launch();
    int64_t tile = p.tile_lo + blockIdx.x;
    if (tid == 0 && tile < ntiles) issue(tile, p.pdl);
    if (p.pdl) griddep_wait();
    bool bad = false;
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const TileRange r = tile_range(p, tile, K, eL, eR);
        const int org = eL + ((eL - r.o) & 1);
#ifdef LMEP_TMX_TIMING
        long long tq0 = clock64();
#endif
        mbar_wait(&bar, (uint32_t)(it & 1));
#ifdef LMEP_TMX_TIMING
        long long tq1 = clock64();
#endif
        // rows and initial values of this thread's J staged nodes -> registers
        // (nodes past the staged range keep finite placeholders; their results
        // only reach nodes that are never stored)
        double w[J][NS], x[J];
        const int l0 = J * tid;
        if (r.o == 0 && l0 + J <= r.len) {
#pragma unroll
            for (int c = 0; c < NS; ++c) {
#pragma unroll
                for (int j = 0; j < J; j += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(R + c * RS + l0 + j);
                    w[j][c] = v.x;
                    w[j + 1][c] = v.y;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int ls = r.o + (l0 + j < r.len ? l0 + j : K * eL);
#pragma unroll
                for (int c = 0; c < NS; ++c) w[j][c] = R[c * RS + ls];
            }
        }
#pragma unroll
        for (int j = 0; j < J; ++j) x[j] = Ub[org + (l0 + j < r.len ? l0 + j : K * eL)];
        __syncthreads();                         // R and Ub free for the next tile's copies
        const int64_t nxt = tile + gridDim.x;
#ifdef LMEP_TMX_TIMING
        long long tq2 = clock64();
#endif
        if (tid == 0 && nxt < ntiles) issue(nxt, 0);
#ifdef LMEP_TMX_TIMING
        long long tq3 = clock64();
#endif

        for (int s = 0; s < K; ++s) {
            double *Qb = Q + (s & 1) * (J * QS);
#pragma unroll
            for (int j = 0; j < J; ++j) Qb[j * QS + 2 + tid] = x[j];
            if constexpr (!EX) {
                // Fused mode: ONE chain per node, ordered for the operand reuse cache.
                // A DFMA whose three operands are all fresh register pairs costs three
                // register-file cycles against two issue cycles (tools/rf_probe.cu), and
                // only the window value can be shared between products (every weight is
                // used once, the accumulator comes from the chain's previous product).
                // ptxas interleaves the J independent chains round-robin whatever the
                // source order, so the order WITHIN a chain is what decides: product k of
                // every node's chain reads the same window value, and products k of
                // consecutive nodes then take it from the reuse cache.
                //   * first the thread's own values x[0 .. J-1] (window slots EL .. EL+J-1,
                //     shared by all J nodes): these need no exchange, so ptxas runs them
                //     between the stores and the barrier and behind the halo loads;
                //   * then node j takes its right-halo values R_0 .. R_(nr-1) and after them
                //     its left-halo values L_j .. L_(EL-1): at n = 13 position m pairs R_m
                //     (nodes j >= m) with L_(m-1) (nodes j < m).
                // 18 distinct values feed the 78 products at n = 13; ptxas marks 51 of
                // them .reuse (26 with separate own / halo chains in tap order).
                // (The generated schedule is sensitive to the source shape: this form --
                // own[] / hal[] arrays, the two switches below at their defaults --
                // measured 1.60 ms for C5's 200 steps, an equivalent rewrite 1.63.)
                double own[J], hal[J];
                auto own_chain = [&](int j) {
                    // taps c with EL <= j + c < EL + J (window slots of this thread's values)
                    double a = 0.0;
#pragma unroll
                    for (int c = 0; c < NS; ++c) {
                        const int i = j + c;
                        if (i >= EL && i < EL + J) a = fma(w[j][c], x[i - EL], a);
                    }
                    return a;
                };
#ifndef LMEP_TMX_ONECHAIN
#define LMEP_TMX_ONECHAIN 1
#endif
#ifndef LMEP_TMX_OWN_PRE
#define LMEP_TMX_OWN_PRE (J / 2)
#endif
#pragma unroll
                for (int j = 0; j < LMEP_TMX_OWN_PRE; ++j) own[j] = own_chain(j);
                __syncthreads();
                double hl[EL > 0 ? EL : 1], hr[ER > 0 ? ER : 1];
                // window slot EL + o is staged node J tid + o: slot (o mod J) of thread
                // tid + floor(o / J) -- the one or two nearest threads on each side
                // (loads in the order the chains consume them: R_0, L_0, R_1, L_1, ...)
#pragma unroll
                for (int m = 0; m < (EL > ER ? EL : ER); ++m) {
                    if (m < ER) {
                        const int o = J + m;
                        hr[m] = Qb[(o % J) * QS + 2 + tid + o / J];
                    }
                    if (m < EL) {
                        const int o = m - EL;                              // -EL .. -1
                        const int dt = -((-o + J - 1) / J);                // floor(o / J)
                        hl[m] = Qb[(o - dt * J) * QS + 2 + tid + dt];
                    }
                }
#pragma unroll
                for (int j = LMEP_TMX_OWN_PRE; j < J; ++j) own[j] = own_chain(j);
                // the chains continue (LMEP_TMX_ONECHAIN) with the halo values
#pragma unroll
                for (int j = 0; j < J; ++j) hal[j] = LMEP_TMX_ONECHAIN ? own[j] : 0.0;
#pragma unroll
                for (int k = 0; k < EL + ER; ++k) {
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        constexpr int dR = ER - J + 1;                        // node j reads R_0 .. R_{j+dR-1}
                        const int nr = j + dR < 0 ? 0 : (j + dR > ER ? ER : j + dR);
                        if (k < nr) {
                            hal[j] = fma(w[j][EL + J + k - j], hr[k], hal[j]);
                        } else {
                            const int i = j + (k - nr);                       // left value L_i, tap i - j
                            if (i < EL) hal[j] = fma(w[j][i - j], hl[i], hal[j]);
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < J; ++j) x[j] = LMEP_TMX_ONECHAIN ? hal[j] : own[j] + hal[j];
            } else {
                __syncthreads();
                double win[W];
#pragma unroll
                for (int m = 0; m < EL; ++m) {
                    const int o = m - EL, dt = -((-o + J - 1) / J);
                    win[m] = Qb[(o - dt * J) * QS + 2 + tid + dt];
                }
#pragma unroll
                for (int j = 0; j < J; ++j) win[EL + j] = x[j];
#pragma unroll
                for (int m = 0; m < ER; ++m) {
                    const int o = J + m;
                    win[EL + J + m] = Qb[(o % J) * QS + 2 + tid + o / J];
                }
                // each node's ascending chain (the reference order), the J chains
                // interleaved tap by tap
                double acc[J];
#pragma unroll
                for (int j = 0; j < J; ++j) acc[j] = xmul(w[j][0], win[j]);
#pragma unroll
                for (int c = 1; c < NS; ++c) {
#pragma unroll
                    for (int j = 0; j < J; ++j) acc[j] = xadd(acc[j], xmul(w[j][c], win[j + c]));
                }
#pragma unroll
                for (int j = 0; j < J; ++j) x[j] = acc[j];
            }
        }
        // outputs: staged nodes [K eL, K eL + (t1 - t0)) -> u_out[t0 ...]
#ifdef LMEP_TMX_TIMING
        long long tq4 = clock64();
#endif
        // (pairs of nodes as one 16-byte store where the pair is aligned and owned: a
        // thread's J values are contiguous in u_out, lanes 8 J bytes apart, so every
        // store instruction touches 32 sectors whatever its width)
        {
            double *uo = p.u_out + (r.t0 - p.ext_off) + (l0 - K * eL);
            const bool vec = (((uintptr_t)uo) & 15) == 0;
#pragma unroll
            for (int j = 0; j < J; j += 2) {
                const int64_t i = r.t0 + (int64_t)(l0 + j - K * eL);
                if (vec && i >= r.t0 && i + 1 < r.t1) {
                    *reinterpret_cast<double2 *>(uo + j) = make_double2(x[j], x[j + 1]);
                    bad |= !isfinite(x[j]) | !isfinite(x[j + 1]);
                } else {
                    if (i >= r.t0 && i < r.t1) { uo[j] = x[j]; bad |= !isfinite(x[j]); }
                    if (i + 1 >= r.t0 && i + 1 < r.t1) { uo[j + 1] = x[j + 1]; bad |= !isfinite(x[j + 1]); }
                }
            }
        }
#ifdef LMEP_TMX_TIMING
        if (tid == 32 && (blockIdx.x == 0 || blockIdx.x == 77) && it < 30) {
            long long *o = g_tmx_timing + (blockIdx.x ? 256 : 0) + it * 6;
            o[0] = tq0; o[1] = tq1; o[2] = tq2; o[3] = tq3; o[4] = tq4; o[5] = clock64();
        }
#endif
    }
    if (bad) *p.flag = 1;
}

// launch as a programmatic dependent of the launch before it on the stream
// (programmatic stream serialization): the CTAs may start while that launch
// drains and wait for it inside the kernel (griddepcontrol.wait)
static void launch_dependent(void (*k)(StepParams), unsigned grid, unsigned threads, size_t shm,
                             cudaStream_t st, const StepParams &p)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, p);
}

// (n, row) pairs with both halo widths <= 6 that the register-resident kernel
// is instantiated for: the centred stencils and the n = 7 one-sided ones
template <bool EX, int NT, int MINB, int J = 6>
static int launch_tmx(const StepParams &p, unsigned grid, cudaStream_t st)
{
    const size_t shm = (size_t)(p.n * (J * NT + 4) + tma_ulen(p.n, J * NT) + 2 * J * (NT + 4)) * 8;
    void (*k)(StepParams) = nullptr;
    if (p.n == 13 && p.row == 6) k = lin_pernode_tmx_kernel<13, 6, J, NT, EX, MINB>;
    else if (p.n == 11 && p.row == 5) k = lin_pernode_tmx_kernel<11, 5, J, NT, EX, MINB>;
    else if (p.n == 9 && p.row == 4) k = lin_pernode_tmx_kernel<9, 4, J, NT, EX, MINB>;
    else if (p.n == 7 && p.row == 3) k = lin_pernode_tmx_kernel<7, 3, J, NT, EX, MINB>;
    else if (p.n == 7 && p.row == 6) k = lin_pernode_tmx_kernel<7, 6, J, NT, EX, MINB>;
    else if (p.n == 7 && p.row == 0) k = lin_pernode_tmx_kernel<7, 0, J, NT, EX, MINB>;
    if (!k) return -1;
    // (the attribute is per device and per kernel: set once for each (n, row) here)
    static std::atomic<uint64_t> attr_done[LMEP_MAX_N + 1][LMEP_MAX_N + 1];
    const int dev = current_device();
    if (!done_on_device(attr_done[p.n][p.row], dev)) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        mark_device(attr_done[p.n][p.row], dev);
    }
    if (p.pdl) launch_dependent(k, grid, NT, shm, st, p);
    else k<<<grid, NT, shm, st>>>(p);
    return launch_status("lin_pernode_tmx_kernel");
}

size_t tma_smem_bytes(int n, int span) { return (size_t)(n * (span + 4) + 3 * tma_ulen(n, span)) * 8; }

int launch_lin_pernode_tma(const StepParams &p, bool exact, cudaStream_t st)
{
    constexpr int J = 3, NT = 512;
    const size_t shm = tma_smem_bytes(p.n, J * NT);
    const int64_t ntiles = (p.tile_hi > 0 ? p.tile_hi : (p.nloc + p.tile - 1) / p.tile) - p.tile_lo;
    const int nsm = device_sm_count();
    const unsigned grid = (unsigned)(ntiles < nsm ? ntiles : nsm);
    if ((p.N & 1) || (p.wld & 1) || ((uintptr_t)p.wp & 15) || ((uintptr_t)p.u_in & 15))
        return LMEP_INVALID_CONFIG;
    // auto: the register-resident kernel for the fused mode (C5 200 steps,
    // 25 per launch: 10.2 vs 10.6 us/step), the window kernel for the exact
    // order (11.7 vs 12.3: two roundings per tap double its FP64 work and the
    // window kernel's 16 warps hide that latency better)
    const int pk = device_settings().pernode_kernel.load();
    if (pk == 3) {
        // two CTAs of 128 threads per SM, each on its own 768-node tile: while one
        // exchanges halos through shared memory the other keeps the FP64 pipe busy
        const unsigned g2 = (unsigned)(ntiles < 2 * nsm ? ntiles : 2 * nsm);
        const int rc = exact ? launch_tmx<true, 128, 2>(p, g2, st) : launch_tmx<false, 128, 2>(p, g2, st);
        if (rc >= 0) return rc;
        return LMEP_INVALID_CONFIG;
    }
    if (pk == 4) {
        // four nodes per thread, 384 threads (three warps per scheduler): the halo
        // comes from the two nearest threads on each side
        const int rc = exact ? launch_tmx<true, 384, 1, 4>(p, grid, st) : launch_tmx<false, 384, 1, 4>(p, grid, st);
        if (rc >= 0) return rc;
        return LMEP_INVALID_CONFIG;
    }
    if (pk == 1 || (pk == 2 && !exact)) {
        const int rc = exact ? launch_tmx<true, 256, 1>(p, grid, st) : launch_tmx<false, 256, 1>(p, grid, st);
        if (rc >= 0) return rc;                  // else: (n, row) not instantiated
    }
#define LMEP_TMA_CASE(NS_)                                                                        \
    case NS_:                                                                                     \
        if (exact) {                                                                              \
            cudaFuncSetAttribute(lin_pernode_tma_kernel<NS_, J, NT, true>,                        \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);          \
            if (p.pdl) launch_dependent(lin_pernode_tma_kernel<NS_, J, NT, true>, grid, NT, shm, st, p); \
            else lin_pernode_tma_kernel<NS_, J, NT, true><<<grid, NT, shm, st>>>(p);              \
        } else {                                                                                  \
            cudaFuncSetAttribute(lin_pernode_tma_kernel<NS_, J, NT, false>,                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);          \
            if (p.pdl) launch_dependent(lin_pernode_tma_kernel<NS_, J, NT, false>, grid, NT, shm, st, p); \
            else lin_pernode_tma_kernel<NS_, J, NT, false><<<grid, NT, shm, st>>>(p);             \
        }                                                                                         \
        break;
    switch (p.n) {
        LMEP_TMA_CASE(13)
        LMEP_TMA_CASE(11)
        LMEP_TMA_CASE(9)
        LMEP_TMA_CASE(7)
    default: return LMEP_INVALID_CONFIG;
    }
#undef LMEP_TMA_CASE
    return launch_status("lin_pernode_tma_kernel");
}

}  // namespace lmep

#ifdef LMEP_TMX_TIMING
extern "C" int lmep_debug_tmx_timing(long long *host_out)
{
    return cudaMemcpyFromSymbol(host_out, lmep::g_tmx_timing, sizeof(long long) * 512) == cudaSuccess ? 0 : 4;
}
#endif

extern "C" int lmep_set_pernode_kernel(int variant)
{
    if (variant < 0 || variant > 4) return LMEP_INVALID_CONFIG;
    lmep::device_settings().pernode_kernel.store(variant);
    return LMEP_OK;
}
