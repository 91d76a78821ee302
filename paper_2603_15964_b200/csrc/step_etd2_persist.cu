// step_etd2_persist.cu -- K5 on mid-size periodic grids (BASELINE config 2:
// N = 65536, 5000 steps): ONE cooperative launch for the whole run.
//
// The tiled ETD2 path re-stages every tile from HBM each launch and needs
// steps / k launches (C2: 625 launches of 256 CTAs, 2 us per step inside the
// kernels).  The whole state of such a grid is ~1 MB, so here it never leaves
// the chip: every CTA (one per SM, cooperative launch = all co-resident) owns
// T = N / G consecutive nodes for the whole run,
//
//   * u in shared memory, the multistep history N_{k-1} in registers (it is
//     only ever consumed by its own node), three nodes per thread;
//   * a chunk of K steps runs on the owned nodes plus H = K * ext * reach halo
//     nodes per side (halo recompute, as in the tiled kernels);
//   * between chunks a CTA publishes its first / last H owned values of u and
//     of the history in a global exchange buffer (L2), bumps its chunk counter
//     with a release store, and its two neighbours wait for that counter with
//     acquire loads -- no grid-wide barrier, no relaunch.  The buffer is
//     double buffered by chunk parity: a CTA publishes chunk c + 1 only after it
//     has seen both neighbours' counters for chunk c, i.e. after they finished
//     reading chunk c - 1's copy of the same half.
//
// Per step (timestep.py:187-215, s = 2), register-resident as step_rk4.cuh:
//   A  window u:    N_k = N(u) (D1 u for the convective kind), W u kept in
//                   registers, g = N_k - N_{k-1};       stores N_k, g
//   B  windows N_k, g:  u' = (W u + P1 N_k) + (P2 g) / dt   in place of u
// EX instantiations keep the reference's roundings (bit-identical to the tiled
// path and to the numba / Python loops).
#include "step.cuh"

namespace lmep {

namespace {

constexpr int PE_NT = 256;     // threads per CTA
constexpr int PE_P = 3;        // staged nodes per thread
constexpr int PE_PAD = 16;     // slot origin: windows of the first staged node stay in bounds
constexpr int PE_CAP = PE_NT * PE_P;

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct PersistArgs {
    double *xbuf;              // [2 parity][G][2 edges (first, last)][2 fields (u, q)][H]
    unsigned *flags;           // [G] chunks published
    int H, T, K, nchunks;
    int64_t steps;
};

template <int NS, int NLK, bool EX>
__global__ void __launch_bounds__(PE_NT, 1)
etd2_persist_kernel(const __grid_constant__ StepParams p, const PersistArgs a)
{
    constexpr int P = PE_P, W = P + NS - 1;
    constexpr bool cv = NLK == LMEP_NL_CONVECTIVE;
    extern __shared__ double sm[];
    const int tid = threadIdx.x, cta = blockIdx.x, G = gridDim.x;
    const int H = a.H, T = a.T;
    const int64_t o0 = (int64_t)cta * T;
    const int tc = (int)(o0 + T <= p.N ? T : p.N - o0);        // owned nodes
    const int len = tc + 2 * H;                                // staged nodes: s in [0, len)
    const int slen = (int)p.slot_len;
    double *XU = sm + PE_PAD, *XK = sm + slen + PE_PAD, *XG = sm + 2 * slen + PE_PAD;
    const int eL = p.eL;
    const int s0 = tid * P;                                    // this thread's staged nodes s0 .. s0+P-1
    const bool act = s0 < len;
    for (int i = tid; i < 3 * slen; i += PE_NT) sm[i] = 0.0;
    __syncthreads();
    // ---- initial state: staged node s is global node o0 - H + s (periodic) ----
    for (int s = tid; s < len; s += PE_NT) XU[s] = p.u_in[wrap(o0 - H + s, p.N)];
    double hq[P];
#pragma unroll
    for (int q = 0; q < P; ++q) hq[q] = (s0 + q < len) ? p.q_in[wrap(o0 - H + s0 + q, p.N)] : 0.0;
    __syncthreads();
    const int left = (cta + G - 1) % G, right = (cta + 1) % G;
    auto edge = [&](int parity, int who, int which, int field) {
        return a.xbuf + ((((int64_t)parity * G + who) * 2 + which) * 2 + field) * H;
    };
    const double inv_dt = 1.0 / p.dtj[1];
    int64_t done = 0;
    for (int c = 0; c < a.nchunks; ++c) {
        const int ks = (int)(a.steps - done < a.K ? a.steps - done : a.K);
        if (c > 0) {
            // ghosts of chunk c: the left neighbour's last H owned values, the right
            // neighbour's first H (both published after their chunk c - 1)
            if (tid == 0) {
                while (ld_acquire(a.flags + left) < (unsigned)c) {}
                while (ld_acquire(a.flags + right) < (unsigned)c) {}
            }
            __syncthreads();
            const double *lu = edge(c & 1, left, 1, 0), *lq = edge(c & 1, left, 1, 1);
            const double *ru = edge(c & 1, right, 0, 0), *rq = edge(c & 1, right, 0, 1);
            for (int i = tid; i < H; i += PE_NT) {
                XU[i] = __ldcg(lu + i);
                XU[tc + H + i] = __ldcg(ru + i);
            }
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int s = s0 + q;
                if (s < H) hq[q] = __ldcg(lq + s);
                else if (s >= tc + H && s < len) hq[q] = __ldcg(rq + (s - tc - H));
            }
            __syncthreads();
        }
        for (int st = 0; st < ks; ++st) {
            double v0[P];
            if (act) {                                         // A: N_k, g = N_k - N_{k-1}, W u
                double uw[W], uc[P];
                const double *x = XU + (s0 - eL);
#pragma unroll
                for (int i = 0; i < W; ++i) uw[i] = x[i];
#pragma unroll
                for (int q = 0; q < P; ++q) uc[q] = XU[s0 + q];
                // the 2 P product chains advance tap by tap (independent FMAs back to
                // back: each chain is n dependent operations)
                double du[P];
#pragma unroll
                for (int q = 0; q < P; ++q) { du[q] = 0.0; v0[q] = 0.0; }
#pragma unroll
                for (int j = 0; j < NS; ++j) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        if constexpr (cv) du[q] = macc<EX>(du[q], p.wi[LMEP_ROW_D1][j], uw[q + j]);
                        v0[q] = macc<EX>(v0[q], p.wi[LMEP_ROW_W][j], uw[q + j]);
                    }
                }
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const double nk = nlp<EX>(NLK, uc[q], du[q]);
                    // grad^1 N = N_k - N_{k-1}, accumulated from 0 as timestep.py:208 does
                    const double g = EX ? xadd(xadd(0.0, nk), xmul(-1.0, hq[q])) : nk + (-1.0) * hq[q];
                    XK[s0 + q] = nk;
                    XG[s0 + q] = g;
                    hq[q] = nk;
                }
            }
            __syncthreads();
            if (act) {                                         // B: u' in place of u
                double kw[W], gw[W];
                const double *xk = XK + (s0 - eL), *xg = XG + (s0 - eL);
#pragma unroll
                for (int i = 0; i < W; ++i) { kw[i] = xk[i]; gw[i] = xg[i]; }
                double v1[P], v2[P];
#pragma unroll
                for (int q = 0; q < P; ++q) { v1[q] = 0.0; v2[q] = 0.0; }
#pragma unroll
                for (int j = 0; j < NS; ++j) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        v1[q] = macc<EX>(v1[q], p.wi[LMEP_ROW_ALPHA][j], kw[q + j]);
                        v2[q] = macc<EX>(v2[q], p.wi[LMEP_ROW_BETA][j], gw[q + j]);
                    }
                }
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    double acc = padd<EX>(v0[q], v1[q]);
                    acc = padd<EX>(acc, EX ? xdiv(v2[q], p.dtj[1]) : v2[q] * inv_dt);
                    XU[s0 + q] = acc;
                }
            }
            __syncthreads();
        }
        done += ks;
        if (c + 1 < a.nchunks) {
            // publish this CTA's edges for chunk c + 1
            double *fu = edge((c + 1) & 1, cta, 0, 0), *fq = edge((c + 1) & 1, cta, 0, 1);
            double *lu = edge((c + 1) & 1, cta, 1, 0), *lq = edge((c + 1) & 1, cta, 1, 1);
            for (int i = tid; i < H; i += PE_NT) {
                __stcg(fu + i, XU[H + i]);
                __stcg(lu + i, XU[tc + i]);
            }
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int s = s0 + q;
                if (s >= H && s < 2 * H) __stcg(fq + (s - H), hq[q]);
                if (s >= tc && s < tc + H) __stcg(lq + (s - tc), hq[q]);
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release(a.flags + cta, (unsigned)(c + 1));
        }
    }
    // ---- results: owned nodes s in [H, H + tc) ---------------------------------
    bool bad = false;
    for (int i = tid; i < tc; i += PE_NT) {
        const double v = XU[H + i];
        p.u_out[o0 + i] = v;
        bad |= !isfinite(v);
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int s = s0 + q;
        if (s >= H && s < H + tc) p.q_out[o0 + (s - H)] = hq[q];
    }
    if (bad) *p.flag = 1;
}

template <int NS, int NLK>
int launch_pe(bool exact, const StepParams &p, const PersistArgs &a, int G, size_t shm, cudaStream_t st)
{
    void *args[2] = {(void *)&p, (void *)&a};
    const void *fn = exact ? (const void *)etd2_persist_kernel<NS, NLK, true>
                           : (const void *)etd2_persist_kernel<NS, NLK, false>;
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(G), dim3(PE_NT), args, shm, st);
    if (e != cudaSuccess) {
        // not co-resident on this device (or no cooperative launch in this context):
        // the caller takes the tiled launches
        cudaGetLastError();
        return -1;
    }
    return launch_status("etd2_persist_kernel");
}

template <int NS>
int launch_pe_nl(int nl, bool exact, const StepParams &p, const PersistArgs &a, int G, size_t shm,
                 cudaStream_t st)
{
    if (nl == LMEP_NL_CONVECTIVE) return launch_pe<NS, LMEP_NL_CONVECTIVE>(exact, p, a, G, shm, st);
    if (nl == LMEP_NL_CUBIC) return launch_pe<NS, LMEP_NL_CUBIC>(exact, p, a, G, shm, st);
    return launch_pe<NS, LMEP_NL_NONE>(exact, p, a, G, shm, st);
}

}  // namespace

// Plan and launch; returns -1 when the grid does not suit the resident schedule
// (the caller then takes the tiled path).  p carries the grid, rows, dt and the
// in / out pointers of a whole-grid ETD2 call.
int try_launch_etd2_persistent(StepParams &p, int nl, bool exact, int64_t steps, cudaStream_t st)
{
    const int n = p.n;
    if (!(n == 7 || n == 9 || n == 11 || n == 13)) return -1;
    if (!device_settings().etd2_persistent.load()) return -1;
    const int reach = std::max(p.eL, p.eR);
    if (reach > PE_PAD - 2 || steps < 2) return -1;
    const int ext = 1 + (nl == LMEP_NL_CONVECTIVE ? 1 : 0);
    int G = device_sm_count();
    int dev = current_device(), coop = 0;
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess || !coop) return -1;
    // owned nodes per CTA, and the deepest halo (steps per exchange) that still
    // fits three nodes per thread
    int T = 0, K = 0, H = 0;
    for (;; --G) {
        if (G < 8) return -1;
        T = (int)((p.N + G - 1) / G);
        const int g2 = (int)((p.N + T - 1) / T);
        if (g2 != G) continue;                               // this G leaves an empty CTA
        const int last = (int)(p.N - (int64_t)(G - 1) * T);
        K = (int)std::min<int64_t>(24, steps);
        while (K > 1 && (T + 2 * K * ext * reach > PE_CAP || K * ext * reach > last)) --K;
        H = K * ext * reach;
        if (T + 2 * H <= PE_CAP && H <= last) break;
    }
    if (T < 64) return -1;                                   // tiny grids: ring mode serves them
    PersistArgs a{};
    a.H = H; a.T = T; a.K = K; a.steps = steps;
    a.nchunks = (int)((steps + K - 1) / K);
    const int64_t slen = ((int64_t)T + 2 * H + PE_PAD + PE_P + LMEP_MAX_N + 3) & ~int64_t(3);
    p.slot_len = slen;
    const size_t shm = (size_t)3 * slen * 8;
    const size_t xbytes = (size_t)2 * G * 2 * 2 * H * 8;
    char *buf = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&buf, xbytes + (size_t)G * 4 + 16, st);
    if (e != cudaSuccess) { set_last_error("cudaMallocAsync", e); return LMEP_CUDA_ERROR; }
    a.xbuf = (double *)buf;
    a.flags = (unsigned *)(buf + xbytes);
    cudaMemsetAsync(a.flags, 0, (size_t)G * 4, st);
    int rc;
    switch (n) {
    case 7: rc = launch_pe_nl<7>(nl, exact, p, a, G, shm, st); break;
    case 9: rc = launch_pe_nl<9>(nl, exact, p, a, G, shm, st); break;
    case 11: rc = launch_pe_nl<11>(nl, exact, p, a, G, shm, st); break;
    default: rc = launch_pe_nl<13>(nl, exact, p, a, G, shm, st); break;
    }
    cudaFreeAsync(buf, st);
    return rc;
}

}  // namespace lmep

extern "C" int lmep_set_etd2_persistent(int on)
{
    lmep::device_settings().etd2_persistent.store(on ? 1 : 0);
    return LMEP_OK;
}
