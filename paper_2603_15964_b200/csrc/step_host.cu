// step_host.cu -- host side of the step kernels: validation, launch planning,
// temporal-blocking launch loop and the C-ABI entry points (lmep.h).
#include <math.h>

#include "step.cuh"

namespace lmep {

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
static int nslots(int sch, int etds = 2) { return sch == SCH_LIN ? 2 : (sch == SCH_ETD2 ? 2 * etds + 1 : 7); }

// per-step dependency extent in stencil units
static int step_ext(int sch, int nl)
{
    const int cv = nl == LMEP_NL_CONVECTIVE ? 1 : 0;
    if (sch == SCH_LIN) return 1;
    if (sch == SCH_ETD2) return 1 + cv;
    return 4 + 4 * cv;
}

static int num_sms() { return device_sm_count(); }

static const int64_t kSmemBudget = 200 * 1024;  // bytes per CTA we allow ourselves

int plan_launch(const lmep_grid &g, int sch, int nl, int64_t steps, bool sharded, bool pernode,
                lmep_tuning &t, int64_t pernode_pad, int etds, bool tma_ok, bool slab_tma = false)
{
    const int n = g.n, eL = g.row, eR = n - 1 - g.row;
    const int ext = step_ext(sch, nl);
    const int ns = nslots(sch, etds);
    const int P = pernode ? 1 : (sch == SCH_ETD2 ? STEP_P_ETD2 : (sch == SCH_ETDRK4 ? step_p_etdrk4(nl, n) : 5));
    const int64_t rad = (int64_t)ext * (eL + eR);
    // ring mode: whole periodic grid on one CTA for all steps
    const int64_t ring_bytes = (int64_t)ns * (g.N + n + SLOT_PAD + P) * 8;
    if (t.ring == 0 && t.tile == 0 && g.periodic && !sharded && g.nloc == g.N && !pernode &&
        ring_bytes <= kSmemBudget && g.N >= 4 * n && g.N <= 8192 && steps > 1) {
        t.ring = 1;
    }
    if (t.ring) {
        if (!g.periodic || sharded || pernode || ring_bytes > kSmemBudget) return LMEP_INVALID_CONFIG;
        t.tile = (int32_t)g.N;
        t.ksteps = (int32_t)std::max<int64_t>(1, steps);
        return LMEP_OK;
    }
    int64_t tile = t.tile, k = t.ksteps, rk4_k = 0;
    if (pernode && sch == SCH_LIN && g.periodic && tb_nodes_per_cta(n, false) > 0 && steps > 1 &&
        t.tile == 0 && (!sharded || pernode_pad >= steps * std::max(eL, eR))) {
        // per-node rows held in registers for k steps: single shard with an
        // even N -> the persistent TMA-pipelined kernel (lin_pernode_tma_kernel),
        // else lin_pernode_tb_kernel; sharded: the caller fuses `steps` steps
        // per halo exchange
        // steps per launch: the rows cross HBM once per launch; past ~25 steps the
        // halo recompute (k (n-1) of the 1536-node span) outweighs it (C5 sweep
        // tools/c5_variant_sweep.py: k = 16 10.4, 25 9.3, 34 9.4 us/step)
        const int64_t kdef = (!sharded && (g.N % 2) == 0 && g.N >= tb_nodes_per_cta(n, true)) ? 25 : 16;
        k = sharded ? steps : (t.ksteps > 0 ? t.ksteps : std::min<int64_t>(kdef, steps));
        // (slab_tma: a slab whose ghosts sit right next to it and whose extended range
        // fits the span takes the persistent kernel too)
        const bool tma = tma_ok && (sharded ? slab_tma : ((g.N % 2) == 0 && g.N >= tb_nodes_per_cta(n, true)));
        const int64_t span = tb_nodes_per_cta(n, tma);
        while (k > 1 && span - k * (n - 1) < span / 2) --k;
        t.tile = (int32_t)(span - k * (n - 1));
        t.ksteps = (int32_t)k;
        t.ring = 0;
        t.threads = 256;
        return LMEP_OK;
    }
    if (pernode && (sch == SCH_LIN || sharded)) k = 1;
    const int64_t nsm = num_sms();
    if (tile <= 0) {
        if (pernode) tile = 2048;
        else if (sch == SCH_LIN) tile = 4096;
        else if (sch == SCH_ETD2) tile = 2048;
        // ETDRK4: + halo ~ 256 chunks of 5; large unsharded grids take wider tiles
        // with several steps per launch (C4 2^24: 254 -> 192 us/step, C3 2^20:
        // 36.7 -> 33.0, tools/prof_cases.py sweeps over tile x k)
        else {
            // register-resident ETDRK4 passes (step_rk4.cuh): one chunk of P staged
            // nodes per thread, so tile + k * rad <= 256 P; large unsharded grids
            // fuse several steps per launch
            const bool big = !sharded && g.nloc >= (int64_t)1800 * 2 * nsm;
            const int64_t kk = k > 0 ? k : (big ? (nl == LMEP_NL_CONVECTIVE ? 3 : 6) : 1);
            tile = (int64_t)STEP_THREADS * P - kk * rad;
            if (tile < 512 || pernode) tile = big ? 1800 : 1200;
            else if (big) rk4_k = kk;
        }
        // small grids: enough tiles to cover the SMs
        while (tile > 256 && (g.nloc + tile - 1) / tile < 2 * nsm) tile /= 2;
        tile = std::min<int64_t>(tile, g.nloc);
    }
    if (k <= 0) {
        const int64_t ntiles = (g.nloc + tile - 1) / tile;
        k = 1;
        if (sch == SCH_LIN && !pernode) k = 8;                  // HBM-bound: reuse u on chip
        else if (ntiles < 2 * nsm)
            // latency-bound small grids: deeper halos, fewer launches (ETD2 C2 at
            // 2^16: k 4 -> 8, 2.57 -> 2.12 us/step FMA)
            k = std::max<int64_t>(1, tile / ((sch == SCH_ETD2 ? 2 : 4) * std::max<int64_t>(rad, 1)));
        else if (rk4_k > 0) k = rk4_k;
        k = std::min<int64_t>(k, std::max<int64_t>(steps, 1));
        k = std::max<int64_t>(k, 1);
    }
    // respect the shared-memory budget
    while (k > 1 && (int64_t)ns * (tile + k * rad + SLOT_PAD + P) * 8 > kSmemBudget) --k;
    while (tile > 64 && (int64_t)ns * (tile + k * rad + SLOT_PAD + P) * 8 > kSmemBudget) tile /= 2;
    if ((int64_t)ns * (tile + k * rad + SLOT_PAD + P) * 8 > kSmemBudget) return LMEP_INVALID_CONFIG;
    if (!g.periodic && tile < 2 * n && tile < g.nloc) tile = std::min<int64_t>(g.nloc, 2 * n);
    t.tile = (int32_t)tile;
    t.ksteps = (int32_t)k;
    t.ring = 0;
    if (t.threads <= 0 && sch != SCH_LIN) {
        // one chunk of P nodes per thread for the widest pass of a step:
        // a pass is a single round, nobody waits for a second one at the barrier
        int64_t widest = tile + (int64_t)ext * (eL + eR);
        // ETDRK4: the register-resident passes keep one chunk per thread over the
        // whole staged range (tile + k * rad) when that fits the CTA
        if (sch == SCH_ETDRK4 && !pernode && tile + k * rad <= (int64_t)STEP_THREADS * P)
            widest = tile + k * rad;
        int64_t th = ((widest + P - 1) / P + 31) / 32 * 32;
        t.threads = (int32_t)std::max<int64_t>(32, std::min<int64_t>(256, th));
    }
    return LMEP_OK;
}

static int launch_step(int sch, bool exact, bool pernode, const StepParams &p, dim3 grid,
                       size_t shm, cudaStream_t st)
{
    if (sch == SCH_LIN) return launch_scheme_lin(pernode, p, grid, shm, st);
    if (sch == SCH_ETDRK4) {
        if (p.nl == LMEP_NL_CONVECTIVE) return launch_scheme_etdrk4_convective(exact, p, grid, shm, st);
        if (p.nl == LMEP_NL_CUBIC) return launch_scheme_etdrk4_cubic(exact, p, grid, shm, st);
        return launch_scheme_etdrk4_none(exact, p, grid, shm, st);
    }
    if (p.nl == LMEP_NL_CONVECTIVE) return launch_scheme_etd2_convective(exact, p, grid, shm, st);
    if (p.nl == LMEP_NL_CUBIC) return launch_scheme_etd2_cubic(exact, p, grid, shm, st);
    return launch_scheme_etd2_none(exact, p, grid, shm, st);
}

int run_steps(const StepCall &c)
{
    if (!c.grid || !c.w) return LMEP_INVALID_CONFIG;
    const lmep_grid &g = *c.grid;
    const lmep_weights &w = *c.w;
    if (g.n < 1 || g.n > LMEP_MAX_N || g.row < 0 || g.row >= g.n) return LMEP_DIMENSION;
    if (g.N < g.n || g.nloc < 1 || g.off < 0 || g.off + g.nloc > g.N) return LMEP_DIMENSION;
    if (c.steps < 0) return LMEP_INVALID_CONFIG;
    if (c.nl < 0 || c.nl > 2) return LMEP_INVALID_CONFIG;
    const bool pernode = w.mode == LMEP_W_PERNODE;
    if (w.mode < 0 || w.mode > 2) return LMEP_INVALID_CONFIG;
    if (c.sch == SCH_ETD2 && (c.etds < 1 || c.etds > 5)) return LMEP_INVALID_CONFIG;
    const int need = c.sch == SCH_LIN ? 1 : (c.sch == SCH_ETD2 ? c.etds + 1 : 6);
    const int need_rows = c.nl == LMEP_NL_CONVECTIVE ? LMEP_ROW_D1 + 1 : need;
    if (w.nrows < need_rows || w.nrows > LMEP_MAX_ROWS) return LMEP_DIMENSION;
    if (!pernode && !w.interior) return LMEP_INVALID_CONFIG;
    if (pernode && (!w.pernode || w.pernode_pad < 0)) return LMEP_INVALID_CONFIG;
    if (w.mode == LMEP_W_CLASS) {
        if (!w.classes || w.nleft < 0 || w.nright < 0 || w.nleft + w.nright >= g.N)
            return LMEP_INVALID_CONFIG;
    }
    const bool sharded = c.halo && (c.halo->left || c.halo->right);
    if (pernode && sharded && c.sch != SCH_LIN) return LMEP_INVALID_CONFIG;  // halo rows not held
    if (!sharded && g.nloc != g.N) return LMEP_INVALID_CONFIG;
    const int bck = c.bc ? c.bc->kind : LMEP_BC_NONE;
    if (bck < 0 || bck > 2) return LMEP_INVALID_CONFIG;
    if (bck != LMEP_BC_NONE && g.periodic) return LMEP_INVALID_CONFIG;
    if (bck == LMEP_BC_NEUMANN && (!c.bc->dl || !c.bc->dr)) return LMEP_INVALID_CONFIG;
    if (!g.periodic && g.N < 2 * g.n) return LMEP_INVALID_CONFIG;
    if (c.steps == 0) {
        cudaError_t e = cudaMemcpyAsync(c.u_out, c.u_in, g.nloc * 8, cudaMemcpyDeviceToDevice, c.stream);
        if (e == cudaSuccess && c.sch == SCH_ETD2 && c.etds > 1)
            e = cudaMemcpyAsync(c.q_out, c.q_in, (c.etds - 1) * g.nloc * 8, cudaMemcpyDeviceToDevice,
                                c.stream);
        if (e != cudaSuccess) { set_last_error("cudaMemcpyAsync", e); return LMEP_CUDA_ERROR; }
        return LMEP_OK;
    }

    lmep_tuning t{};
    if (c.tuning) t = *c.tuning;
    if (sharded) { t.ring = 0; }
    // the TMA kernel bulk-copies u_in and the rows: both 16-byte aligned (a
    // contiguous view at an odd element offset takes the register-blocked kernel)
    bool tma_ok = ((uintptr_t)c.u_in & 15) == 0 && ((uintptr_t)w.pernode & 15) == 0;
    // a slab of a sharded per-node run whose ghost cells are stored right around it
    // ([ghosts | u | ghosts] contiguous, as wide as the row table's pad): the
    // persistent TMA kernels read that extended array like a whole grid
    bool slab_tma = false;
    if (sharded && pernode && c.sch == SCH_LIN && g.periodic && bck == LMEP_BC_NONE && c.halo->left &&
        c.halo->right) {
        const int64_t G = c.halo->width;
        slab_tma = c.halo->left + G == c.u_in && c.halo->right == c.u_in + g.nloc && w.pernode_pad == G &&
                   (g.nloc % 2) == 0 && ((uintptr_t)c.halo->left & 15) == 0 &&
                   ((uintptr_t)w.pernode & 15) == 0 && g.nloc + 2 * G >= tb_nodes_per_cta(g.n, true) &&
                   device_settings().pernode_kernel.load() != 3;
        if (slab_tma) tma_ok = true;
    }
    int st = plan_launch(g, c.sch, c.nl, c.steps, sharded, pernode, t, pernode ? w.pernode_pad : 0,
                         c.etds, tma_ok, slab_tma);
    if (st) return st;

    // host staging of the (large) parameter block, one per calling thread: the
    // launches copy it, so concurrent callers on other streams never share it
    static thread_local StepParams p;
    p = StepParams{};
    p.N = g.N; p.off = g.off; p.nloc = g.nloc;
    p.n = g.n; p.row = g.row; p.periodic = g.periodic ? 1 : 0; p.ring = t.ring;
    p.eL = g.row; p.eR = g.n - 1 - g.row;
    p.wmode = w.mode; p.nrows = w.nrows; p.nleft = w.nleft; p.nright = w.nright;
    if (w.interior)
        for (int r = 0; r < w.nrows; ++r)
            for (int j = 0; j < g.n; ++j) p.wi[r][j] = w.interior[r * g.n + j];
    p.wc = w.classes;
    p.wp = w.pernode;
    p.wpad = pernode ? w.pernode_pad : 0;
    p.wld = g.nloc + 2 * p.wpad;
    if (g.periodic) {
        p.L_int = INT64_MIN / 4;
        p.R_int = INT64_MAX / 4;
    } else {
        p.L_int = g.row;
        p.R_int = g.N - (g.n - 1 - g.row);
        if (w.mode == LMEP_W_CLASS) {
            p.L_int = std::max<int64_t>(p.L_int, w.nleft);
            p.R_int = std::min<int64_t>(p.R_int, g.N - w.nright);
        }
    }
    p.nl = c.nl;
    p.bc = bck;
    if (c.bc) {
        p.lo = c.bc->lo;
        p.hi = c.bc->hi;
        if (bck == LMEP_BC_NEUMANN)
            for (int j = 0; j < g.n; ++j) { p.dl[j] = c.bc->dl[j]; p.dr[j] = c.bc->dr[j]; }
    }
    p.dt = c.dt;
    p.etds = c.etds;
    p.qld = g.nloc;
    for (int j = 0; j < 6; ++j) p.dtj[j] = pow(c.dt, (double)j);   // Python's dt**j
    p.ext = step_ext(c.sch, c.nl);
    p.tile = t.tile;
    p.threads = t.threads > 0 ? t.threads : STEP_THREADS;
    if (p.threads % 32 != 0 || p.threads > STEP_THREADS) return LMEP_INVALID_CONFIG;
    const int P = pernode ? 1 : (c.sch == SCH_ETD2 ? STEP_P_ETD2 : (c.sch == SCH_ETDRK4 ? step_p_etdrk4(c.nl, g.n) : 5));
    const int64_t rad = (int64_t)p.ext * (p.eL + p.eR);
    p.slot_len = t.ring ? (g.N + g.n + SLOT_PAD + P) : (t.tile + (int64_t)t.ksteps * rad + SLOT_PAD + P);
    p.slot_len = (p.slot_len + 3) & ~int64_t(3);
    const size_t shm = (size_t)nslots(c.sch, c.etds) * p.slot_len * 8;

    // Keep freed stream-ordered allocations in the device pool: with the
    // default release threshold (0) every synchronize returns them to the OS
    // and the next cudaMallocAsync maps fresh pages (milliseconds per call).
    static std::atomic<uint64_t> pool_tuned{0};
    const int dev = current_device();
    if (!done_on_device(pool_tuned, dev)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        mark_device(pool_tuned, dev);
    }
    // finiteness flag
    int *flag = c.nonfinite;
    int *own_flag = nullptr;
    if (!flag) {
        cudaError_t e = cudaMallocAsync((void **)&own_flag, sizeof(int), c.stream);
        if (e != cudaSuccess) { set_last_error("cudaMallocAsync", e); return LMEP_CUDA_ERROR; }
        flag = own_flag;
    }
    cudaMemsetAsync(flag, 0, sizeof(int), c.stream);
    p.flag = flag;

    // ETD2 on a mid-size periodic grid with shared rows (C2): the whole run in one
    // cooperative launch, the state resident on chip (step_etd2_persist.cu)
    if (c.sch == SCH_ETD2 && c.etds == 2 && !sharded && !t.ring && g.periodic &&
        w.mode == LMEP_W_SHARED && bck == LMEP_BC_NONE && !(c.tuning && (c.tuning->tile > 0 || c.tuning->ksteps > 0))) {
        p.u_in = c.u_in; p.u_out = c.u_out; p.q_in = c.q_in; p.q_out = c.q_out;
        const int prc = try_launch_etd2_persistent(p, c.nl, (c.flags & LMEP_FLAG_EXACT) != 0, c.steps, c.stream);
        if (prc >= 0) {
            if (own_flag) cudaFreeAsync(own_flag, c.stream);
            return prc;
        }
    }
    const int64_t kmax = t.ksteps;
    const int64_t nlaunch = (c.steps + kmax - 1) / kmax;
    if (sharded) {
        if (nlaunch != 1) return LMEP_INVALID_CONFIG;     // caller exchanges halos per launch
        const int64_t need_w = c.steps * p.ext * std::max(p.eL, p.eR);
        if (c.halo->width < need_w) return LMEP_INVALID_CONFIG;
        if (c.sch == SCH_ETD2 && c.etds > 1 && (!c.halo->hist_left && !c.halo->hist_right))
            return LMEP_INVALID_CONFIG;
    }
    // scratch ping-pong
    double *scr = c.scratch, *own_scr = nullptr;
    const int64_t scr_need = (c.sch == SCH_ETD2 ? c.etds : 1) * g.nloc;
    if (nlaunch > 1 && !scr) {
        cudaError_t e = cudaMallocAsync((void **)&own_scr, scr_need * 8, c.stream);
        if (e != cudaSuccess) { set_last_error("cudaMallocAsync", e); return LMEP_CUDA_ERROR; }
        scr = own_scr;
    }
    const dim3 grid(t.ring ? 1u : (unsigned)((g.nloc + t.tile - 1) / t.tile));
    const double *src = c.u_in, *qsrc = c.q_in;
    int rc = LMEP_OK;
    bool host_copied = false;
    int64_t done = 0;
    // persistent TMA per-node kernel: the steps spread evenly over the launches, each
    // launch's tile widened to the span its k leaves (tile + k (n-1) = span): C5's
    // 200 steps run as 8 x 15 + 5 x 16 instead of 12 x 16 + 8
    const bool tma_path = c.sch == SCH_LIN && pernode && p.bc == LMEP_BC_NONE && g.periodic &&
                          (!sharded || slab_tma) && t.threads == 256 &&
                          t.tile + (int64_t)t.ksteps * (g.n - 1) == tb_nodes_per_cta(g.n, true);
    for (int64_t L = 0; L < nlaunch; ++L) {
        int64_t k = std::min<int64_t>(kmax, c.steps - done);
        if (tma_path) {
            k = (c.steps - done + (nlaunch - L) - 1) / (nlaunch - L);
            p.tile = tb_nodes_per_cta(g.n, true) - k * (g.n - 1);
        }
        // the last launch must land in u_out
        const bool to_out = ((nlaunch - 1 - L) % 2) == 0;
        double *dst = to_out ? c.u_out : scr;
        double *qdst = (c.sch == SCH_ETD2 && c.etds > 1) ? (to_out ? c.q_out : scr + g.nloc) : nullptr;
        p.ksteps = (int)k;
        p.u_in = src;
        p.u_out = dst;
        p.q_in = qsrc;
        p.q_out = qdst;
        p.nl0_out = (L == 0) ? c.nl0_out : nullptr;
        // (unsharded) every launch after the first depends on the one before it only
        // through u: its CTAs start as that one drains and prefetch their first rows
        p.pdl = (tma_path && !sharded && L > 0) ? 1 : 0;
        if (sharded && tma_path) {
            // the slab's extended arrays: u from its left ghosts on, the padded row table
            p.u_in = c.halo->left;
            p.ext_off = c.halo->width;
            p.N = g.nloc + 2 * c.halo->width;
        } else if (sharded) {
            p.hl = c.halo->left; p.hr = c.halo->right;
            p.qhl = c.halo->hist_left; p.qhr = c.halo->hist_right;
            p.G = c.halo->width;
            if (c.halo->push_width > 0 && (c.halo->push_left || c.halo->push_right)) {
                // fused peer stores: the shared / class-row step_kernel launches only
                if (pernode || c.sch == SCH_ETD2 || c.halo->push_width > g.nloc) return LMEP_INVALID_CONFIG;
                p.push_l = c.halo->push_left;
                p.push_r = c.halo->push_right;
                p.push_w = c.halo->push_width;
            }
        }
        if (tma_path && c.host_out && L == nlaunch - 1 && c.parts > 1) {
            // last launch, result wanted on the host: one launch per tile range, each
            // range copied on the copy stream as soon as its launch has finished
            const int64_t ntl = (g.nloc + p.tile - 1) / p.tile;
            const int parts = (int)std::min<int64_t>(c.parts, std::max<int64_t>(1, ntl / (2 * num_sms())));
            cudaEvent_t ev;
            for (int part = 0; part < parts && rc == LMEP_OK; ++part) {
                p.tile_lo = ntl * part / parts;
                p.tile_hi = ntl * (part + 1) / parts;
                rc = launch_lin_pernode_tma(p, (c.flags & LMEP_FLAG_EXACT) != 0, c.stream);
                if (rc) break;
                const int64_t a = p.tile_lo * p.tile, b = std::min<int64_t>(g.nloc, p.tile_hi * p.tile);
                if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventRecord(ev, c.stream) != cudaSuccess ||
                    cudaStreamWaitEvent(c.copy_stream, ev, 0) != cudaSuccess ||
                    cudaMemcpyAsync(c.host_out + a, dst + a, (size_t)(b - a) * 8, cudaMemcpyDeviceToHost,
                                    c.copy_stream) != cudaSuccess) {
                    set_last_error("lmep_step_linear_host (part copy)", cudaGetLastError());
                    rc = LMEP_CUDA_ERROR;
                }
                cudaEventDestroy(ev);                // released once the recorded work completes
            }
            p.tile_lo = p.tile_hi = 0;
            host_copied = true;
        } else if (tma_path)
            rc = launch_lin_pernode_tma(p, (c.flags & LMEP_FLAG_EXACT) != 0, c.stream);      // persistent, TMA-pipelined (C5)
        else if (c.sch == SCH_LIN && pernode && p.bc == LMEP_BC_NONE && g.periodic &&
            t.threads == 256 && t.tile + (int64_t)t.ksteps * (g.n - 1) == tb_nodes_per_cta(g.n, false))
            rc = launch_lin_pernode_tb(p, (c.flags & LMEP_FLAG_EXACT) != 0, c.stream);       // rows in registers, k steps
        else if (c.sch == SCH_LIN && pernode && p.bc == LMEP_BC_NONE && k == 1 && !t.ring)
            rc = launch_lin_pernode(p, c.stream);          // lean streaming kernel
        else
            rc = launch_step(c.sch, (c.flags & LMEP_FLAG_EXACT) != 0, pernode, p, grid, shm, c.stream);
        if (rc) break;
        src = dst;
        qsrc = qdst;
        done += k;
    }
    if (rc == LMEP_OK && c.host_out && !host_copied) {
        // every other path: one copy behind the last launch
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(ev, c.stream) != cudaSuccess ||
            cudaStreamWaitEvent(c.copy_stream, ev, 0) != cudaSuccess ||
            cudaMemcpyAsync(c.host_out, c.u_out, (size_t)g.nloc * 8, cudaMemcpyDeviceToHost,
                            c.copy_stream) != cudaSuccess) {
            set_last_error("lmep_step_linear_host (copy)", cudaGetLastError());
            rc = LMEP_CUDA_ERROR;
        }
        cudaEventDestroy(ev);
    }
    if (own_scr) cudaFreeAsync(own_scr, c.stream);
    if (own_flag) cudaFreeAsync(own_flag, c.stream);
    return rc;
}

__global__ void rows_to_soa_kernel(const double *__restrict__ rows, int64_t N, int n,
                                   double *__restrict__ soa)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * n) return;
    const int64_t i = e / n;
    const int j = (int)(e - i * n);
    soa[(int64_t)j * N + i] = rows[e];
}

}  // namespace lmep

using namespace lmep;

extern "C" int lmep_step_linear(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                                const lmep_halo *halo, const double *u_in, double *u_out,
                                double *scratch, int64_t steps, int32_t flags,
                                const lmep_tuning *tuning, int32_t *nonfinite, void *stream)
{
    StepCall c{};
    c.sch = SCH_LIN; c.grid = grid; c.w = w; c.bc = bc; c.halo = halo; c.nl = 0;
    // LMEP_FLAG_EXACT clear selects fused multiply-adds in the temporally blocked
    // per-node kernels (FP64-issue-bound); every other linear kernel is always exact
    c.u_in = u_in; c.u_out = u_out; c.scratch = scratch; c.steps = steps; c.flags = flags;
    c.tuning = tuning; c.nonfinite = nonfinite; c.stream = (cudaStream_t)stream;
    return run_steps(c);
}

extern "C" int lmep_step_linear_host(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                                     const lmep_halo *halo, const double *u_in, double *u_out,
                                     double *scratch, int64_t steps, int32_t flags,
                                     const lmep_tuning *tuning, int32_t *nonfinite, void *stream,
                                     double *host_out, int parts, void *copy_stream)
{
    if (!host_out || parts < 1 || steps < 1) return LMEP_INVALID_CONFIG;
    StepCall c{};
    c.sch = SCH_LIN; c.grid = grid; c.w = w; c.bc = bc; c.halo = halo; c.nl = 0;
    c.u_in = u_in; c.u_out = u_out; c.scratch = scratch; c.steps = steps; c.flags = flags;
    c.tuning = tuning; c.nonfinite = nonfinite; c.stream = (cudaStream_t)stream;
    c.host_out = host_out; c.parts = parts; c.copy_stream = (cudaStream_t)copy_stream;
    return run_steps(c);
}

extern "C" int lmep_step_etdrk4(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                                const lmep_halo *halo, int nl_kind, const double *u_in,
                                double *u_out, double *scratch, int64_t steps, double *nl0_out,
                                int32_t flags, const lmep_tuning *tuning, int32_t *nonfinite,
                                void *stream)
{
    StepCall c{};
    c.sch = SCH_ETDRK4; c.grid = grid; c.w = w; c.bc = bc; c.halo = halo; c.nl = nl_kind;
    c.u_in = u_in; c.u_out = u_out; c.scratch = scratch; c.steps = steps; c.flags = flags;
    c.tuning = tuning; c.nonfinite = nonfinite; c.nl0_out = nl0_out; c.stream = (cudaStream_t)stream;
    return run_steps(c);
}

extern "C" int lmep_step_etds(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                              const lmep_halo *halo, int nl_kind, int order, double delta_t,
                              const double *u_in, const double *hist_in, double *u_out,
                              double *hist_out, double *scratch, int64_t steps, int32_t flags,
                              const lmep_tuning *tuning, int32_t *nonfinite, void *stream)
{
    if (order < 1 || order > 5) return LMEP_INVALID_CONFIG;
    if (order > 1 && (!hist_in || !hist_out)) return LMEP_INVALID_CONFIG;
    if (!(delta_t > 0.0)) return LMEP_INVALID_CONFIG;
    StepCall c{};
    c.sch = SCH_ETD2; c.etds = order; c.grid = grid; c.w = w; c.bc = bc; c.halo = halo;
    c.nl = nl_kind; c.dt = delta_t; c.u_in = u_in; c.q_in = hist_in; c.u_out = u_out;
    c.q_out = hist_out; c.scratch = scratch; c.steps = steps; c.flags = flags; c.tuning = tuning;
    c.nonfinite = nonfinite; c.stream = (cudaStream_t)stream;
    return run_steps(c);
}

extern "C" int lmep_step_etd2(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                              const lmep_halo *halo, int nl_kind, double delta_t,
                              const double *u_in, const double *hist_in, double *u_out,
                              double *hist_out, double *scratch, int64_t steps, int32_t flags,
                              const lmep_tuning *tuning, int32_t *nonfinite, void *stream)
{
    return lmep_step_etds(grid, w, bc, halo, nl_kind, 2, delta_t, u_in, hist_in, u_out, hist_out,
                          scratch, steps, flags, tuning, nonfinite, stream);
}

extern "C" int lmep_banded_matvec(const lmep_grid *grid, const lmep_weights *w,
                                  const lmep_halo *halo, const double *u, double *out,
                                  int32_t flags, void *stream)
{
    lmep_tuning t{};
    t.ksteps = 1;
    StepCall c{};
    c.sch = SCH_LIN; c.grid = grid; c.w = w; c.bc = nullptr; c.halo = halo; c.nl = 0;
    c.u_in = u; c.u_out = out; c.steps = 1; c.flags = flags | LMEP_FLAG_EXACT; c.tuning = &t;
    c.stream = (cudaStream_t)stream;
    return run_steps(c);
}

extern "C" int lmep_plan(const lmep_grid *grid, int scheme, int nl_kind, int weight_mode,
                         int64_t steps, lmep_tuning *out)
{
    if (!grid || !out) return LMEP_INVALID_CONFIG;
    if (scheme < 0 || scheme > 2) return LMEP_INVALID_CONFIG;
    lmep_tuning t = *out;
    int st = plan_launch(*grid, scheme, nl_kind, steps, grid->nloc != grid->N,
                         weight_mode == LMEP_W_PERNODE, t, 0, 2, true);
    *out = t;
    return st;
}

extern "C" int lmep_rows_to_soa(const double *rows, int64_t N, int n, double *soa, void *stream)
{
    if (N * n == 0) return LMEP_OK;
    const int tpb = 256;
    rows_to_soa_kernel<<<(unsigned)((N * n + tpb - 1) / tpb), tpb, 0, (cudaStream_t)stream>>>(rows, N, n, soa);
    return launch_status("rows_to_soa_kernel");
}
