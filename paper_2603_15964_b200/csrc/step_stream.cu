// step_stream.cu -- streamed linear steps: the k-step launches of the persistent
// per-node kernels (step_lin_tma.cu) issued in a skewed space-time order, so
// that stepping starts while the per-node rows are still being harvested and
// the result starts leaving for the host while the last nodes still step.
//
// timestep.run (timestep.py:255-394) harvests every row, then steps, then
// copies the snapshot: three phases in a row.  On config 5 from host arrays the
// upload of the coefficients (PCIe) and the harvest already overlap slice by
// slice; here the steps join that pipeline.  The rows and the initial values
// become valid as a growing PREFIX [0, ready) of the periodic grid.  Launch
// level l (its k_l steps, tile T_l) reads the output of level l-1 and may run
// every tile whose staged range (tile + k_l halo nodes per side) lies inside
// what level l-1 has produced so far, so after each harvested slice every
// level advances its own frontier, one tile behind the level before it:
//
//      nodes ->   0 ............. ready ........... N
//      level 1    . [=============)                      (. = held back: its halo
//      level 2    . . [===========)                        wraps to nodes that are
//      level 3    . . . [=========)                        not ready yet)
//
// When the last slice has landed, each level finishes with ONE launch over the
// rest of the ring, [frontier, N) continued at [0, first tile) (tile_wrap).
// Every tile is computed by the same kernel on the same staged range as in the
// level-by-level order of run_steps, so the result is bit-identical to it.
//
// Buffers: level 1 reads u_in, the levels then alternate between scratch and
// u_out as in run_steps (the last level writes u_out).  A level never writes
// nodes another level may still read: frontiers keep a margin of
// max_l k_l * max(eL, eR) nodes (see advance()).  The last level's new nodes
// are copied to host_out on copy_stream behind an event after every call.
#include <math.h>

#include <algorithm>
#include <vector>

#include "step.cuh"

namespace lmep {
int plan_launch(const lmep_grid &g, int sch, int nl, int64_t steps, bool sharded, bool pernode,
                lmep_tuning &t, int64_t pernode_pad, int etds, bool tma_ok, bool slab_tma);
}

using namespace lmep;

struct lmep_lin_stream {
    StepParams p;
    bool exact = true;
    int dev = 0;
    int64_t N = 0, margin = 0, ready = 0;
    std::vector<int> k;                 // steps of level l
    std::vector<int64_t> tile;          // owned nodes per tile at level l
    std::vector<int64_t> jlo, jhi;      // tiles [jlo, jhi) of level l are done (jhi < 0: none yet)
    std::vector<const double *> src;
    std::vector<double *> dst;
    double *host_out = nullptr;
    cudaStream_t copy_stream = nullptr;
    bool finished = false;
    int64_t launches = 0;
};

static int copy_out(lmep_lin_stream *s, int64_t a, int64_t b, cudaStream_t st)
{
    if (!s->host_out || b <= a) return LMEP_OK;
    const double *res = s->dst.back();
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, st) != cudaSuccess ||
        cudaStreamWaitEvent(s->copy_stream, ev, 0) != cudaSuccess ||
        cudaMemcpyAsync(s->host_out + a, res + a, (size_t)(b - a) * 8, cudaMemcpyDeviceToHost,
                        s->copy_stream) != cudaSuccess) {
        set_last_error("lmep_lin_stream (copy)", cudaGetLastError());
        return LMEP_CUDA_ERROR;
    }
    cudaEventDestroy(ev);                        // released once the recorded work completes
    return LMEP_OK;
}

static int launch_level(lmep_lin_stream *s, int l, int64_t lo, int64_t hi, int64_t wrap, cudaStream_t st)
{
    StepParams &p = s->p;
    p.ksteps = s->k[l];
    p.tile = s->tile[l];
    p.u_in = s->src[l];
    p.u_out = s->dst[l];
    p.tile_lo = lo;
    p.tile_hi = hi;
    p.tile_wrap = wrap;
    // level 1 follows the harvest of its rows; a deeper level follows the level before
    // it (its rows landed long ago): a programmatic dependent that prefetches them
    p.pdl = l > 0 ? 1 : 0;
    ++s->launches;
    return launch_lin_pernode_tma(p, s->exact, st);
}

extern "C" int lmep_lin_stream_begin(const lmep_grid *grid, const lmep_weights *w, const double *u_in,
                                     double *u_out, double *scratch, int64_t steps, int32_t flags,
                                     const lmep_tuning *tuning, int32_t *nonfinite, double *host_out,
                                     void *copy_stream, void *stream, lmep_lin_stream **out)
{
    if (!grid || !w || !u_in || !u_out || !scratch || !nonfinite || !out || steps < 1)
        return LMEP_INVALID_CONFIG;
    *out = nullptr;
    const lmep_grid &g = *grid;
    if (g.n < 1 || g.n > LMEP_MAX_N || g.row < 0 || g.row >= g.n) return LMEP_DIMENSION;
    if (g.N < g.n || g.nloc != g.N || g.off != 0) return LMEP_INVALID_CONFIG;
    if (!g.periodic || w->mode != LMEP_W_PERNODE || !w->pernode || w->pernode_pad != 0 || w->nrows < 1)
        return LMEP_INVALID_CONFIG;
    if (u_in == u_out || u_in == scratch || u_out == scratch) return LMEP_INVALID_CONFIG;
    if (((uintptr_t)u_in & 15) || ((uintptr_t)u_out & 15) || ((uintptr_t)scratch & 15) ||
        ((uintptr_t)w->pernode & 15))
        return LMEP_INVALID_CONFIG;
    lmep_tuning t{};
    if (tuning) t = *tuning;
    int rc = plan_launch(g, SCH_LIN, 0, steps, false, true, t, 0, 2, true, false);
    if (rc) return rc;
    const int64_t span = tb_nodes_per_cta(g.n, true);
    // the persistent TMA plan only (run_steps' tma_path): even N, at least one span
    if (t.ring || t.threads != 256 || span <= 0 || (g.N & 1) || g.N < span ||
        t.tile + (int64_t)t.ksteps * (g.n - 1) != span)
        return LMEP_INVALID_CONFIG;

    auto *s = new lmep_lin_stream();
    s->exact = (flags & LMEP_FLAG_EXACT) != 0;
    s->dev = current_device();
    s->N = g.N;
    s->host_out = host_out;
    s->copy_stream = (cudaStream_t)copy_stream;
    StepParams &p = s->p;
    p = StepParams{};
    p.N = g.N; p.off = 0; p.nloc = g.N;
    p.n = g.n; p.row = g.row; p.periodic = 1; p.ring = 0;
    p.eL = g.row; p.eR = g.n - 1 - g.row;
    p.wmode = w->mode; p.nrows = w->nrows;
    p.wp = w->pernode; p.wpad = 0; p.wld = g.N;
    p.L_int = INT64_MIN / 4; p.R_int = INT64_MAX / 4;
    p.nl = 0; p.bc = LMEP_BC_NONE; p.ext = 1; p.threads = 256; p.qld = g.N;
    p.flag = nonfinite;
    // the launch levels of run_steps: the steps spread evenly over the launches
    const int64_t kmax = t.ksteps;
    const int64_t nl = (steps + kmax - 1) / kmax;
    int64_t done = 0;
    for (int64_t L = 0; L < nl; ++L) {
        const int64_t k = (steps - done + (nl - L) - 1) / (nl - L);
        s->k.push_back((int)k);
        s->tile.push_back(span - k * (g.n - 1));
        const bool to_out = ((nl - 1 - L) % 2) == 0;
        s->src.push_back(L == 0 ? u_in : s->dst.back());
        s->dst.push_back(to_out ? u_out : scratch);
        s->margin = std::max<int64_t>(s->margin, k * std::max(p.eL, p.eR));
        done += k;
    }
    s->jlo.assign(nl, 0);
    s->jhi.assign(nl, -1);
    if (cudaMemsetAsync(nonfinite, 0, sizeof(int), (cudaStream_t)stream) != cudaSuccess) {
        set_last_error("lmep_lin_stream_begin", cudaGetLastError());
        delete s;
        return LMEP_CUDA_ERROR;
    }
    *out = s;
    return LMEP_OK;
}

extern "C" int lmep_lin_stream_info(const lmep_lin_stream *s, int64_t *tile, int64_t *margin,
                                    int32_t *levels, int32_t *sms)
{
    if (!s) return LMEP_INVALID_CONFIG;
    if (tile) *tile = s->tile[0];
    if (margin) *margin = s->margin;
    if (levels) *levels = (int32_t)s->k.size();
    if (sms) *sms = device_sm_count();
    return LMEP_OK;
}

extern "C" int lmep_lin_stream_advance(lmep_lin_stream *s, int64_t nodes_ready, void *stream)
{
    if (!s || s->finished || nodes_ready < s->ready || nodes_ready > s->N) return LMEP_INVALID_CONFIG;
    if (current_device() != s->dev) return LMEP_INVALID_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    s->ready = nodes_ready;
    const int nl = (int)s->k.size();
    const int64_t N = s->N, M = s->margin;
    const int last = nl - 1;
    int rc = LMEP_OK;
    if (nodes_ready < N) {
        // input of level l valid on [lo, hi) (no wrap): run the tiles whose owned
        // range extended by the margin lies inside.  The margin (>= every level's
        // halo) also keeps writers clear of readers: level l+1 writes the buffer
        // level l-1 wrote and level l still reads, but only below
        // hi_l - M <= (first unread tile of level l) - halo, and from lo_l + M on,
        // above what the held-back first tiles of level l will read.
        int64_t lo = 0, hi = nodes_ready;
        for (int l = 0; l < nl && rc == LMEP_OK; ++l) {
            const int64_t T = s->tile[l];
            if (hi - M < T) break;
            const int64_t nlo = (lo + M + T - 1) / T, nhi = (hi - M) / T;
            if (s->jhi[l] < 0) {
                if (nhi <= nlo) break;
                s->jlo[l] = nlo;
                s->jhi[l] = nlo;
            }
            const int64_t from = s->jhi[l];
            if (nhi > from) {
                rc = launch_level(s, l, from, nhi, 0, st);
                s->jhi[l] = nhi;
                if (rc == LMEP_OK && l == last) rc = copy_out(s, from * T, nhi * T, st);
            }
            lo = s->jlo[l] * T;
            hi = s->jhi[l] * T;
        }
        return rc;
    }
    // everything has landed: each level finishes the ring in one launch
    for (int l = 0; l < nl && rc == LMEP_OK; ++l) {
        const int64_t T = s->tile[l], nt = (N + T - 1) / T;
        if (s->jhi[l] < 0) {
            rc = launch_level(s, l, 0, nt, 0, st);
            if (rc == LMEP_OK && l == last) rc = copy_out(s, 0, N, st);
        } else if (l == last && s->host_out) {
            // the last launch of all: in up to three tile ranges, each copied to the
            // host while the next one runs (only the last range's copy is exposed)
            const int64_t lo = s->jhi[l], hi = nt + s->jlo[l];
            const int64_t waves = (hi - lo) / std::max(1, device_sm_count());
            const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(3, waves));
            for (int q = 0; q < parts && rc == LMEP_OK; ++q) {
                const int64_t a = lo + (hi - lo) * q / parts, b = lo + (hi - lo) * (q + 1) / parts;
                if (b <= a) continue;
                rc = launch_level(s, l, a, b, nt, st);
                if (rc == LMEP_OK && a < nt) rc = copy_out(s, a * T, std::min(b, nt) * T < N ? std::min(b, nt) * T : N, st);
                if (rc == LMEP_OK && b > nt) rc = copy_out(s, std::max<int64_t>(a - nt, 0) * T, (b - nt) * T, st);
            }
        } else {
            if (nt + s->jlo[l] > s->jhi[l]) rc = launch_level(s, l, s->jhi[l], nt + s->jlo[l], nt, st);
            if (rc == LMEP_OK && l == last) {
                rc = copy_out(s, s->jhi[l] * T, N, st);
                if (rc == LMEP_OK) rc = copy_out(s, 0, s->jlo[l] * T, st);
            }
        }
    }
    s->p.tile_lo = s->p.tile_hi = s->p.tile_wrap = 0;
    s->finished = true;
    return rc;
}

extern "C" int lmep_lin_stream_end(lmep_lin_stream *s, int64_t *launches)
{
    if (!s) return LMEP_INVALID_CONFIG;
    const int rc = s->finished ? LMEP_OK : LMEP_INVALID_CONFIG;
    if (launches) *launches = s->launches;
    delete s;
    return rc;
}

// ---- slice transfers of a streamed run --------------------------------------
// One call queues what a slice needs on the link: its coefficients and its part
// of the initial state go up on `up_stream` (an event behind each: the harvest
// of the slice waits for the first only), and that part of snapshot 0
// (timestep.py:313) goes back down on `down_stream` behind the second.  The
// host side of a streamed run is on the critical path until the first harvest
// is queued; a slice costs one library call instead of a dozen host-API calls
// from Python.
extern "C" int lmep_event_create(void **ev)
{
    if (!ev) return LMEP_INVALID_CONFIG;
    cudaEvent_t e;
    const cudaError_t rc = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (rc != cudaSuccess) { set_last_error("cudaEventCreateWithFlags", rc); return LMEP_CUDA_ERROR; }
    *ev = (void *)e;
    return LMEP_OK;
}

extern "C" int lmep_event_destroy(void *ev)
{
    if (ev) cudaEventDestroy((cudaEvent_t)ev);
    return LMEP_OK;
}

extern "C" int lmep_stream_wait_event(void *stream, void *ev)
{
    if (!ev) return LMEP_INVALID_CONFIG;
    const cudaError_t rc = cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0);
    if (rc != cudaSuccess) { set_last_error("cudaStreamWaitEvent", rc); return LMEP_CUDA_ERROR; }
    return LMEP_OK;
}

extern "C" int lmep_upload_slice(void *coef_dev, const void *coef_host, size_t coef_bytes,
                                 void *u_dev, const void *u_host, void *snap_host, size_t u_bytes,
                                 void *up_stream, void *down_stream, void *ev_coef, void *ev_all)
{
    if (!ev_coef || !ev_all || (coef_bytes && (!coef_dev || !coef_host)) ||
        (u_bytes && (!u_dev || !u_host)))
        return LMEP_INVALID_CONFIG;
    cudaStream_t up = (cudaStream_t)up_stream, down = (cudaStream_t)down_stream;
    cudaError_t rc = cudaSuccess;
    if (coef_bytes) rc = cudaMemcpyAsync(coef_dev, coef_host, coef_bytes, cudaMemcpyHostToDevice, up);
    if (rc == cudaSuccess) rc = cudaEventRecord((cudaEvent_t)ev_coef, up);
    if (rc == cudaSuccess && u_bytes) rc = cudaMemcpyAsync(u_dev, u_host, u_bytes, cudaMemcpyHostToDevice, up);
    if (rc == cudaSuccess) rc = cudaEventRecord((cudaEvent_t)ev_all, up);
    if (rc == cudaSuccess && snap_host && u_bytes) {
        rc = cudaStreamWaitEvent(down, (cudaEvent_t)ev_all, 0);
        if (rc == cudaSuccess) rc = cudaMemcpyAsync(snap_host, u_dev, u_bytes, cudaMemcpyDeviceToHost, down);
    }
    if (rc != cudaSuccess) { set_last_error("lmep_upload_slice", rc); return LMEP_CUDA_ERROR; }
    return LMEP_OK;
}
