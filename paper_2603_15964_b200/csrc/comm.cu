// comm.cu -- K6: the shard communicator behind the C ABI (lmep.h, "sharded
// runs").  One process per GPU; the only data exchange of a sharded run is
// the halo of the 1D slab decomposition (the reference advances
// one array in timestep.run, timestep.py:255-394, and has no collectives).
//
// Two transports:
//   NCCL  ncclSend / ncclRecv in one group on the caller's stream.  libnccl is
//         resolved at run time (dlopen "libnccl.so.2": the copy already in the
//         process when the host framework brought one, else the system one),
//         so liblmep.so itself has no NCCL link dependency.
//   PEER  CUDA IPC on one node.  Every rank owns a double-buffered device
//         mailbox; an exchange stores this rank's edges straight into its
//         neighbours' mailboxes with one kernel (peer stores over NVLink, or
//         plain stores when both ranks share a device), records an
//         interprocess event, publishes the exchange number in a host page
//         shared with the neighbours, waits (host) until they have published
//         theirs, makes the stream wait for their events and copies its own
//         mailbox into the caller's ghost buffers.  No kernel ever spins on
//         another rank's progress, so two ranks may share one GPU (tests).
//
// Why double buffering is enough: rank r stores into q's mailbox half
// (seq & 1) in exchange seq.  q reads that half in its exchange seq (copy-out,
// after waiting for r's event).  r's next store into the same half is in
// exchange seq + 2, issued after r's exchange seq + 1 waited for q's event of
// seq + 1, which q recorded after its copy-out of seq in stream order.
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#include <mutex>

#include "common.cuh"

namespace lmep {

// ---------------------------------------------------------------------------
// libnccl, resolved at run time
// ---------------------------------------------------------------------------
struct NcclApi {
    void *handle = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    bool ok = false;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static const NcclApi *nccl_api()
{
    std::call_once(g_nccl_once, [] {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            g_nccl.handle = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
            if (g_nccl.handle) break;
        }
        if (!g_nccl.handle) return;
        void *h = g_nccl.handle;
#define LMEP_NCCL_SYM(f) g_nccl.f = (decltype(g_nccl.f))dlsym(h, "nccl" #f)
        LMEP_NCCL_SYM(GetUniqueId);
        LMEP_NCCL_SYM(CommInitRank);
        LMEP_NCCL_SYM(CommDestroy);
        LMEP_NCCL_SYM(GroupStart);
        LMEP_NCCL_SYM(GroupEnd);
        LMEP_NCCL_SYM(Send);
        LMEP_NCCL_SYM(Recv);
        LMEP_NCCL_SYM(AllReduce);
        LMEP_NCCL_SYM(GetErrorString);
#undef LMEP_NCCL_SYM
        g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy &&
                    g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.Send && g_nccl.Recv &&
                    g_nccl.AllReduce && g_nccl.GetErrorString;
    });
    return g_nccl.ok ? &g_nccl : nullptr;
}

static int nccl_fail(const char *what, ncclResult_t r)
{
    set_last_error_text(what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "NCCL error");
    return LMEP_CUDA_ERROR;
}
#define NCCL_TRY(call)                                         \
    do {                                                       \
        ncclResult_t r_ = (call);                              \
        if (r_ != ncclSuccess) return nccl_fail(#call, r_);    \
    } while (0)
#define CUDA_TRY(call)                                         \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) {                               \
            set_last_error(#call, e_);                         \
            return LMEP_CUDA_ERROR;                            \
        }                                                      \
    } while (0)

// ---------------------------------------------------------------------------
// PEER transport pieces
// ---------------------------------------------------------------------------
struct HostPage {                       // one per rank, mapped by its neighbours
    std::atomic<uint64_t> posted;       // number of the last exchange whose event is recorded
};

struct PeerBlob {                       // what lmep_comm_export hands out (<= LMEP_COMM_BLOB_BYTES)
    uint32_t magic;
    int32_t rank;
    int32_t device;
    int32_t pid;
    int64_t max_width;
    cudaIpcMemHandle_t mem;
    cudaIpcEventHandle_t ev[2];
    char page_path[160];
};
static_assert(sizeof(PeerBlob) <= LMEP_COMM_BLOB_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0x4c4d4550u;   // "LMEP"

struct PeerLink {                       // one neighbour, as seen from this rank
    int rank = -1;
    bool self = false;
    double *mailbox = nullptr;          // the neighbour's mailbox (IPC-mapped unless self)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    HostPage *page = nullptr;
    bool opened = false;                // IPC mappings to release
};

constexpr int kPushThreads = 256;

struct PushArgs {
    const double *src[LMEP_COMM_MAX_FIELDS];
    double *to_left;                    // left neighbour's "from right" slots of this half (or null)
    double *to_right;                   // right neighbour's "from left" slots of this half
    int64_t nloc, width, slot_ld;
    int nfields;
};

// One launch stores every field's two edges into the neighbours' mailboxes.
__global__ void halo_push_kernel(PushArgs a)
{
    const int64_t per = a.width;
    const int64_t total = per * a.nfields * 2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int side = (int)(e / (per * a.nfields));          // 0: to the left, 1: to the right
        const int64_t r = e - (int64_t)side * per * a.nfields;
        const int f = (int)(r / per);
        const int64_t j = r - (int64_t)f * per;
        if (side == 0) {
            if (a.to_left) a.to_left[f * a.slot_ld + j] = a.src[f][j];
        } else {
            if (a.to_right) a.to_right[f * a.slot_ld + j] = a.src[f][a.nloc - per + j];
        }
    }
}

struct PullArgs {
    double *gl[LMEP_COMM_MAX_FIELDS];
    double *gr[LMEP_COMM_MAX_FIELDS];
    const double *from_left;            // this rank's mailbox, "from left" slots of this half
    const double *from_right;
    int64_t width, slot_ld;
    int nfields;
    int has_left, has_right;
};

__global__ void halo_pull_kernel(PullArgs a)
{
    const int64_t per = a.width;
    const int64_t total = per * a.nfields * 2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int side = (int)(e / (per * a.nfields));
        const int64_t r = e - (int64_t)side * per * a.nfields;
        const int f = (int)(r / per);
        const int64_t j = r - (int64_t)f * per;
        if (side == 0) {
            if (a.has_left) a.gl[f][j] = a.from_left[f * a.slot_ld + j];
        } else {
            if (a.has_right) a.gr[f][j] = a.from_right[f * a.slot_ld + j];
        }
    }
}

}  // namespace lmep

using namespace lmep;

struct lmep_comm {
    int rank = 0, world = 1, periodic = 0, transport = LMEP_COMM_NCCL;
    int left = -1, right = -1;
    int device = 0;
    ncclComm_t nccl = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // PEER
    int64_t max_width = 0;
    double *mailbox = nullptr;          // [2 halves][2 sides][MAX_FIELDS][max_width]
    cudaEvent_t ev[2] = {nullptr, nullptr};
    HostPage *page = nullptr;
    char page_path[160] = "";
    PeerLink lnk_left, lnk_right;
    bool connected = false;
    uint64_t seq = 0;
};

struct lmep_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
};

namespace {

int64_t half_len(const lmep_comm *c) { return 2 * (int64_t)LMEP_COMM_MAX_FIELDS * c->max_width; }
// slots of one half: side 0 = filled by the left neighbour, side 1 = by the right one
double *slot(double *box, const lmep_comm *c, int half, int side)
{
    return box + (int64_t)half * half_len(c) + (int64_t)side * LMEP_COMM_MAX_FIELDS * c->max_width;
}

void close_link(PeerLink &l)
{
    if (l.opened) {
        if (l.mailbox) cudaIpcCloseMemHandle(l.mailbox);
        for (auto &e : l.ev)
            if (e) cudaEventDestroy(e);
        if (l.page) munmap(l.page, sizeof(HostPage));
    }
    l = PeerLink{};
}

int open_link(lmep_comm *c, PeerLink &l, int nb, const PeerBlob *blobs)
{
    l = PeerLink{};
    if (nb < 0) return LMEP_OK;
    l.rank = nb;
    if (nb == c->rank) {
        l.self = true;
        l.mailbox = c->mailbox;
        l.ev[0] = c->ev[0];
        l.ev[1] = c->ev[1];
        l.page = c->page;
        return LMEP_OK;
    }
    const PeerBlob &b = blobs[nb];
    if (b.magic != kBlobMagic || b.rank != nb || b.max_width != c->max_width) {
        set_last_error_text("lmep_comm_connect", "peer blob does not match this communicator");
        return LMEP_INVALID_CONFIG;
    }
    if (b.pid == (int)getpid()) {
        set_last_error_text("lmep_comm_connect", "two ranks of one process cannot share IPC handles");
        return LMEP_INVALID_CONFIG;
    }
    void *p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, b.mem, cudaIpcMemLazyEnablePeerAccess));
    l.mailbox = (double *)p;
    l.opened = true;
    for (int i = 0; i < 2; ++i) CUDA_TRY(cudaIpcOpenEventHandle(&l.ev[i], b.ev[i]));
    const int fd = open(b.page_path, O_RDWR);
    if (fd < 0) {
        set_last_error_text("lmep_comm_connect", "cannot open the neighbour's host page");
        return LMEP_CUDA_ERROR;
    }
    void *m = mmap(nullptr, sizeof(HostPage), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) {
        set_last_error_text("lmep_comm_connect", "cannot map the neighbour's host page");
        return LMEP_CUDA_ERROR;
    }
    l.page = (HostPage *)m;
    return LMEP_OK;
}

// Host wait until the neighbour has recorded the event of exchange `seq`.
int wait_posted(const PeerLink &l, uint64_t seq)
{
    if (l.self) return LMEP_OK;
    timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const char *env = getenv("LMEP_PEER_TIMEOUT_S");
    const double limit = env ? atof(env) : 120.0;
    for (uint64_t spins = 0;; ++spins) {
        if (l.page->posted.load(std::memory_order_acquire) >= seq) return LMEP_OK;
        if ((spins & 1023) == 1023) {
            timespec t;
            clock_gettime(CLOCK_MONOTONIC, &t);
            if ((t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec) > limit) {
                set_last_error_text("lmep_halo_exchange", "timed out waiting for a neighbour rank");
                return LMEP_CUDA_ERROR;
            }
            sched_yield();
        }
    }
}

int exchange_nccl(lmep_comm *c, int nf, const double *const *fields, int64_t nloc, int64_t W,
                  double *const *gl, double *const *gr, cudaStream_t st)
{
    const NcclApi *api = nccl_api();
    if (!api || !c->nccl) return LMEP_INVALID_CONFIG;
    // posting order per rank and field: right edge -> right, left ghosts <- left,
    // left edge -> left, right ghosts <- right.  Messages between a pair match in
    // posting order, so the 2-rank ring (left == right) and the 1-rank
    // self-exchange come out right.
    NCCL_TRY(api->GroupStart());
    ncclResult_t r = ncclSuccess;
    for (int f = 0; f < nf && r == ncclSuccess; ++f) {
        if (c->right >= 0) r = api->Send(fields[f] + nloc - W, W, ncclDouble, c->right, c->nccl, st);
        if (r == ncclSuccess && c->left >= 0) r = api->Recv(gl[f], W, ncclDouble, c->left, c->nccl, st);
        if (r == ncclSuccess && c->left >= 0) r = api->Send(fields[f], W, ncclDouble, c->left, c->nccl, st);
        if (r == ncclSuccess && c->right >= 0) r = api->Recv(gr[f], W, ncclDouble, c->right, c->nccl, st);
    }
    const ncclResult_t e = api->GroupEnd();          // always closes the group
    if (r != ncclSuccess) return nccl_fail("ncclSend/ncclRecv", r);
    if (e != ncclSuccess) return nccl_fail("ncclGroupEnd", e);
    return LMEP_OK;
}

// --- PEER primitives.  c->seq counts this rank's signals; exchange number e
// uses mailbox half e & 1. ---------------------------------------------------
int peer_check(lmep_comm *c, const char *what, cudaStream_t st)
{
    if (c->transport != LMEP_COMM_PEER || !c->connected) return LMEP_INVALID_CONFIG;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
        set_last_error_text(what, "the PEER transport cannot be captured in a graph");
        return LMEP_INVALID_CONFIG;
    }
    return LMEP_OK;
}

// where this rank's edges go for the NEXT signal: my right edge becomes the right
// neighbour's left ghosts (its side 0), my left edge the left neighbour's right
// ghosts (its side 1)
void peer_targets(lmep_comm *c, int field, double **to_left, double **to_right)
{
    const int half = (int)((c->seq + 1) & 1);
    const int64_t fo = (int64_t)field * c->max_width;
    *to_left = c->left >= 0 ? slot(c->lnk_left.mailbox, c, half, 1) + fo : nullptr;
    *to_right = c->right >= 0 ? slot(c->lnk_right.mailbox, c, half, 0) + fo : nullptr;
}

// the edges of the next exchange are stored (by the push kernel, or by a step
// kernel's fused peer stores): record the event, publish the exchange number
int peer_signal(lmep_comm *c, cudaStream_t st)
{
    const uint64_t seq = ++c->seq;
    CUDA_TRY(cudaEventRecord(c->ev[seq & 1], st));
    c->page->posted.store(seq, std::memory_order_release);
    return LMEP_OK;
}

// the stream waits for the neighbours' signal number c->seq
int peer_wait(lmep_comm *c, cudaStream_t st)
{
    const uint64_t seq = c->seq;
    const int half = (int)(seq & 1);
    int rc;
    if (c->left >= 0) {
        if ((rc = wait_posted(c->lnk_left, seq))) return rc;
        CUDA_TRY(cudaStreamWaitEvent(st, c->lnk_left.ev[half], 0));
    }
    if (c->right >= 0 && c->right != c->left) {
        if ((rc = wait_posted(c->lnk_right, seq))) return rc;
        CUDA_TRY(cudaStreamWaitEvent(st, c->lnk_right.ev[half], 0));
    }
    return LMEP_OK;
}

int peer_push(lmep_comm *c, int nf, const double *const *fields, int64_t nloc, int64_t W,
              cudaStream_t st)
{
    if (W > c->max_width) return LMEP_DIMENSION;
    PushArgs pa{};
    for (int f = 0; f < nf; ++f) pa.src[f] = fields[f];
    peer_targets(c, 0, &pa.to_left, &pa.to_right);
    pa.nloc = nloc; pa.width = W; pa.slot_ld = c->max_width; pa.nfields = nf;
    const int64_t total = 2 * W * nf;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + kPushThreads - 1) / kPushThreads, 1184);
    halo_push_kernel<<<blocks, kPushThreads, 0, st>>>(pa);
    int rc = launch_status("halo_push_kernel");
    if (rc) return rc;
    return peer_signal(c, st);
}

int exchange_peer(lmep_comm *c, int nf, const double *const *fields, int64_t nloc, int64_t W,
                  double *const *gl, double *const *gr, cudaStream_t st)
{
    int rc = peer_check(c, "lmep_halo_exchange", st);
    if (rc) return rc;
    if ((rc = peer_push(c, nf, fields, nloc, W, st))) return rc;
    if ((rc = peer_wait(c, st))) return rc;
    const int half = (int)(c->seq & 1);
    PullArgs pl{};
    for (int f = 0; f < nf; ++f) { pl.gl[f] = gl[f]; pl.gr[f] = gr[f]; }
    pl.from_left = slot(c->mailbox, c, half, 0);
    pl.from_right = slot(c->mailbox, c, half, 1);
    pl.width = W; pl.slot_ld = c->max_width; pl.nfields = nf;
    pl.has_left = c->left >= 0; pl.has_right = c->right >= 0;
    const int64_t total = 2 * W * nf;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + kPushThreads - 1) / kPushThreads, 1184);
    halo_pull_kernel<<<blocks, kPushThreads, 0, st>>>(pl);
    return launch_status("halo_pull_kernel");
}

}  // namespace

extern "C" int lmep_comm_unique_id(void *id)
{
    static_assert(sizeof(ncclUniqueId) == LMEP_COMM_ID_BYTES, "ncclUniqueId size");
    const NcclApi *api = nccl_api();
    if (!api) {
        set_last_error_text("lmep_comm_unique_id", "libnccl.so.2 not found");
        return LMEP_INVALID_CONFIG;
    }
    if (!id) return LMEP_INVALID_CONFIG;
    ncclUniqueId u;
    NCCL_TRY(api->GetUniqueId(&u));
    memcpy(id, &u, sizeof(u));
    return LMEP_OK;
}

extern "C" int lmep_comm_init(lmep_comm **out, int rank, int world, int periodic, int transport,
                              const void *id, int64_t max_width)
{
    if (!out || world < 1 || rank < 0 || rank >= world) return LMEP_INVALID_CONFIG;
    if (transport != LMEP_COMM_NCCL && transport != LMEP_COMM_PEER) return LMEP_INVALID_CONFIG;
    lmep_comm *c = new lmep_comm;
    c->rank = rank; c->world = world; c->periodic = periodic ? 1 : 0; c->transport = transport;
    c->device = current_device();
    // neighbours: ring or open chain; a periodic 1-rank ring is its own neighbour
    c->left = (periodic || rank > 0) ? (rank + world - 1) % world : -1;
    c->right = (periodic || rank < world - 1) ? (rank + 1) % world : -1;
    auto fail = [&](int code) { lmep_comm_destroy(c); return code; };
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        set_last_error("lmep_comm_init", cudaGetLastError());
        return fail(LMEP_CUDA_ERROR);
    }
    if (transport == LMEP_COMM_NCCL) {
        const NcclApi *api = nccl_api();
        if (!api) {
            set_last_error_text("lmep_comm_init", "libnccl.so.2 not found");
            return fail(LMEP_INVALID_CONFIG);
        }
        if (!id) return fail(LMEP_INVALID_CONFIG);
        ncclUniqueId u;
        memcpy(&u, id, sizeof(u));
        ncclResult_t r = api->CommInitRank(&c->nccl, world, u, rank);
        if (r != ncclSuccess) { c->nccl = nullptr; return fail(nccl_fail("ncclCommInitRank", r)); }
    } else {
        if (max_width < 1) return fail(LMEP_INVALID_CONFIG);
        c->max_width = max_width;
        // cudaMalloc, not the stream-ordered pool: IPC handles need a plain allocation
        if (cudaMalloc((void **)&c->mailbox, 2 * half_len(c) * sizeof(double)) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev[0], cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev[1], cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess) {
            set_last_error("lmep_comm_init (mailbox)", cudaGetLastError());
            return fail(LMEP_CUDA_ERROR);
        }
        const char *dirs[] = {"/dev/shm", "/tmp"};
        int fd = -1;
        for (const char *d : dirs) {
            snprintf(c->page_path, sizeof(c->page_path), "%s/lmep_comm_%d_%d_XXXXXX", d, (int)getpid(), rank);
            fd = mkstemp(c->page_path);
            if (fd >= 0) break;
        }
        if (fd < 0 || ftruncate(fd, sizeof(HostPage)) != 0) {
            if (fd >= 0) close(fd);
            set_last_error_text("lmep_comm_init", "cannot create the shared host page");
            return fail(LMEP_CUDA_ERROR);
        }
        void *m = mmap(nullptr, sizeof(HostPage), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) {
            set_last_error_text("lmep_comm_init", "cannot map the shared host page");
            return fail(LMEP_CUDA_ERROR);
        }
        c->page = (HostPage *)m;
        c->page->posted.store(0, std::memory_order_release);
    }
    *out = c;
    return LMEP_OK;
}

extern "C" int lmep_comm_export(lmep_comm *c, void *blob)
{
    if (!c || !blob) return LMEP_INVALID_CONFIG;
    memset(blob, 0, LMEP_COMM_BLOB_BYTES);
    if (c->transport != LMEP_COMM_PEER) return LMEP_OK;
    PeerBlob b{};
    b.magic = kBlobMagic; b.rank = c->rank; b.device = c->device; b.pid = (int)getpid();
    b.max_width = c->max_width;
    CUDA_TRY(cudaIpcGetMemHandle(&b.mem, c->mailbox));
    for (int i = 0; i < 2; ++i) CUDA_TRY(cudaIpcGetEventHandle(&b.ev[i], c->ev[i]));
    memcpy(b.page_path, c->page_path, sizeof(b.page_path));
    memcpy(blob, &b, sizeof(b));
    return LMEP_OK;
}

extern "C" int lmep_comm_connect(lmep_comm *c, const void *blobs)
{
    if (!c) return LMEP_INVALID_CONFIG;
    if (c->transport != LMEP_COMM_PEER) return LMEP_OK;
    if (c->connected) return LMEP_INVALID_CONFIG;
    // blobs are LMEP_COMM_BLOB_BYTES apart; PeerBlob is a prefix of each
    PeerBlob *tab = new PeerBlob[c->world];
    const bool need = (c->left >= 0 && c->left != c->rank) || (c->right >= 0 && c->right != c->rank);
    if (need && !blobs) { delete[] tab; return LMEP_INVALID_CONFIG; }
    for (int r = 0; r < c->world && blobs; ++r)
        memcpy(&tab[r], (const char *)blobs + (size_t)r * LMEP_COMM_BLOB_BYTES, sizeof(PeerBlob));
    int rc = open_link(c, c->lnk_left, c->left, tab);
    if (!rc) {
        if (c->right == c->left) {
            c->lnk_right = c->lnk_left;
            c->lnk_right.opened = false;            // one mapping, released through lnk_left
        } else {
            rc = open_link(c, c->lnk_right, c->right, tab);
        }
    }
    delete[] tab;
    if (rc) return rc;
    c->connected = true;
    return LMEP_OK;
}

extern "C" int lmep_comm_destroy(lmep_comm *c)
{
    if (!c) return LMEP_OK;
    if (c->side) cudaStreamSynchronize(c->side);
    close_link(c->lnk_right);
    close_link(c->lnk_left);
    if (c->nccl) {
        const NcclApi *api = nccl_api();
        if (api) api->CommDestroy(c->nccl);
    }
    if (c->mailbox) cudaFree(c->mailbox);
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->page) munmap(c->page, sizeof(HostPage));
    if (c->page_path[0]) unlink(c->page_path);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->side) cudaStreamDestroy(c->side);
    delete c;
    return LMEP_OK;
}

extern "C" int lmep_comm_info(const lmep_comm *c, int *rank, int *world, int *left, int *right,
                              int *transport)
{
    if (!c) return LMEP_INVALID_CONFIG;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (left) *left = c->left;
    if (right) *right = c->right;
    if (transport) *transport = c->transport;
    return LMEP_OK;
}

extern "C" int lmep_halo_exchange(lmep_comm *c, int nfields, const double *const *fields,
                                  int64_t nloc, int64_t width, double *const *ghost_left,
                                  double *const *ghost_right, void *stream)
{
    if (!c || !fields || !ghost_left || !ghost_right) return LMEP_INVALID_CONFIG;
    if (nfields < 1 || nfields > LMEP_COMM_MAX_FIELDS) return LMEP_INVALID_CONFIG;
    if (width < 1 || nloc < width) return LMEP_DIMENSION;   // a slab narrower than its halo
    for (int f = 0; f < nfields; ++f) {
        if (!fields[f]) return LMEP_INVALID_CONFIG;
        if (c->left >= 0 && !ghost_left[f]) return LMEP_INVALID_CONFIG;
        if (c->right >= 0 && !ghost_right[f]) return LMEP_INVALID_CONFIG;
    }
    if (c->left < 0 && c->right < 0) return LMEP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->transport == LMEP_COMM_NCCL)
        return exchange_nccl(c, nfields, fields, nloc, width, ghost_left, ghost_right, st);
    return exchange_peer(c, nfields, fields, nloc, width, ghost_left, ghost_right, st);
}

// ---- PEER: the pieces of an exchange, for step launches that store their own
// edges into the neighbours' mailboxes (lmep_halo.push_*) --------------------
extern "C" int lmep_comm_push(lmep_comm *c, int nfields, const double *const *fields, int64_t nloc,
                              int64_t width, void *stream)
{
    if (!c || !fields || nfields < 1 || nfields > LMEP_COMM_MAX_FIELDS) return LMEP_INVALID_CONFIG;
    if (width < 1 || nloc < width) return LMEP_DIMENSION;
    int rc = peer_check(c, "lmep_comm_push", (cudaStream_t)stream);
    if (rc) return rc;
    return peer_push(c, nfields, fields, nloc, width, (cudaStream_t)stream);
}

extern "C" int lmep_comm_signal(lmep_comm *c, void *stream)
{
    if (!c) return LMEP_INVALID_CONFIG;
    int rc = peer_check(c, "lmep_comm_signal", (cudaStream_t)stream);
    if (rc) return rc;
    return peer_signal(c, (cudaStream_t)stream);
}

extern "C" int lmep_comm_wait(lmep_comm *c, void *stream)
{
    if (!c) return LMEP_INVALID_CONFIG;
    int rc = peer_check(c, "lmep_comm_wait", (cudaStream_t)stream);
    if (rc) return rc;
    return peer_wait(c, (cudaStream_t)stream);
}

extern "C" int lmep_comm_ghosts(lmep_comm *c, int field, const double **left, const double **right)
{
    if (!c || c->transport != LMEP_COMM_PEER || !c->connected) return LMEP_INVALID_CONFIG;
    if (field < 0 || field >= LMEP_COMM_MAX_FIELDS) return LMEP_INVALID_CONFIG;
    const int half = (int)(c->seq & 1);
    const int64_t fo = (int64_t)field * c->max_width;
    if (left) *left = c->left >= 0 ? slot(c->mailbox, c, half, 0) + fo : nullptr;
    if (right) *right = c->right >= 0 ? slot(c->mailbox, c, half, 1) + fo : nullptr;
    return LMEP_OK;
}

extern "C" int lmep_comm_targets(lmep_comm *c, int field, double **to_left, double **to_right)
{
    if (!c || c->transport != LMEP_COMM_PEER || !c->connected) return LMEP_INVALID_CONFIG;
    if (field < 0 || field >= LMEP_COMM_MAX_FIELDS || !to_left || !to_right) return LMEP_INVALID_CONFIG;
    peer_targets(c, field, to_left, to_right);
    return LMEP_OK;
}

extern "C" int lmep_comm_gather(lmep_comm *c, const double *u, const int64_t *counts, double *out,
                                int root, void *stream)
{
    if (!c || !u || !counts || root < 0 || root >= c->world) return LMEP_INVALID_CONFIG;
    if (c->transport != LMEP_COMM_NCCL) return LMEP_INVALID_CONFIG;
    const NcclApi *api = nccl_api();
    if (!api || !c->nccl) return LMEP_INVALID_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->rank == root && !out) return LMEP_INVALID_CONFIG;
    NCCL_TRY(api->GroupStart());
    if (c->rank == root) {
        int64_t off = 0;
        for (int r = 0; r < c->world; ++r) {
            if (r == root) {
                cudaError_t e = cudaMemcpyAsync(out + off, u, counts[r] * sizeof(double),
                                                cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) { api->GroupEnd(); set_last_error("cudaMemcpyAsync", e); return LMEP_CUDA_ERROR; }
            } else if (counts[r] > 0) {
                NCCL_TRY(api->Recv(out + off, counts[r], ncclDouble, r, c->nccl, st));
            }
            off += counts[r];
        }
    } else if (counts[c->rank] > 0) {
        NCCL_TRY(api->Send(u, counts[c->rank], ncclDouble, root, c->nccl, st));
    }
    NCCL_TRY(api->GroupEnd());
    return LMEP_OK;
}

extern "C" int lmep_comm_flag_max(lmep_comm *c, int32_t *flag, int count, void *stream)
{
    if (!c || !flag || count < 1) return LMEP_INVALID_CONFIG;
    if (c->transport != LMEP_COMM_NCCL) return LMEP_INVALID_CONFIG;
    const NcclApi *api = nccl_api();
    if (!api || !c->nccl) return LMEP_INVALID_CONFIG;
    NCCL_TRY(api->AllReduce(flag, flag, count, ncclInt32, ncclMax, c->nccl, (cudaStream_t)stream));
    return LMEP_OK;
}

extern "C" void *lmep_comm_side_stream(lmep_comm *c) { return c ? (void *)c->side : nullptr; }

extern "C" int lmep_comm_fork(lmep_comm *c, void *stream)
{
    if (!c) return LMEP_INVALID_CONFIG;
    CUDA_TRY(cudaEventRecord(c->ev_fork, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    return LMEP_OK;
}

extern "C" int lmep_comm_join(lmep_comm *c, void *stream)
{
    if (!c) return LMEP_INVALID_CONFIG;
    CUDA_TRY(cudaEventRecord(c->ev_join, c->side));
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_join, 0));
    return LMEP_OK;
}

// ---------------------------------------------------------------------------
// one chunk of a sharded run in one call
// ---------------------------------------------------------------------------
extern "C" int lmep_comm_chunk(lmep_comm *c, const lmep_chunk_args *a, void *stream)
{
    if (!c || !a || !a->grid || !a->w || !a->u_in || !a->u_out || !a->nonfinite) return LMEP_INVALID_CONFIG;
    if (a->scheme != SCH_LIN && a->scheme != SCH_ETDRK4) return LMEP_INVALID_CONFIG;
    if (a->w->mode == LMEP_W_PERNODE || a->steps < 1 || a->next_steps < 0) return LMEP_INVALID_CONFIG;
    const lmep_grid &G = *a->grid;
    const int reach = G.row > G.n - 1 - G.row ? G.row : G.n - 1 - G.row;
    const int ext = a->scheme == SCH_LIN ? 1 : (a->nl_kind == LMEP_NL_CONVECTIVE ? 8 : 4);
    const int64_t W = a->steps * ext * reach, nloc = G.nloc;
    const int64_t Wn = std::min<int64_t>(a->next_steps * ext * reach, W);
    if (W < 1 || W > nloc || W > a->ghost_cells) return LMEP_DIMENSION;
    cudaStream_t st = (cudaStream_t)stream;
    const bool hasL = c->left >= 0, hasR = c->right >= 0;
    lmep_tuning tun{0, (int32_t)a->steps, 0, 0};
    const double *u = a->u_in;
    double *o = a->u_out;
    // k steps of the sub-range [off, off + n) of the slab: an ordinary step call
    auto sub = [&](int64_t off, int64_t n, const double *gl, const double *gr, double *pl, double *pr,
                   int64_t pw, int32_t *flag, cudaStream_t s) {
        lmep_grid g = G;
        g.off = G.off + off;
        g.nloc = n;
        lmep_halo h{gl, gr, nullptr, nullptr, W, pl, pr, pw};
        StepCall sc{};
        sc.sch = a->scheme; sc.grid = &g; sc.w = a->w; sc.bc = a->bc;
        sc.halo = (gl || gr) ? &h : nullptr;
        sc.nl = a->nl_kind; sc.u_in = u + off; sc.u_out = o + off; sc.steps = a->steps;
        sc.flags = a->flags; sc.tuning = &tun; sc.nonfinite = flag; sc.stream = s;
        return run_steps(sc);
    };
    if (!hasL && !hasR)                                  // one slab: nothing to exchange
        return sub(0, nloc, nullptr, nullptr, nullptr, nullptr, 0, a->nonfinite, st);
    const bool split = nloc >= 3 * W;
    int rc;
    if (c->transport == LMEP_COMM_NCCL) {
        // ghosts are stored right around u_in; exchange and edge strips on the side
        // stream, beside the interior
        double *gl = const_cast<double *>(u) - W, *gr = const_cast<double *>(u) + nloc;
        const double *fields[1] = {u};
        double *gls[1] = {gl}, *grs[1] = {gr};
        const double *cgl = hasL ? gl : nullptr, *cgr = hasR ? gr : nullptr;
        if (!split) {
            if ((rc = exchange_nccl(c, 1, fields, nloc, W, gls, grs, st))) return rc;
            return sub(0, nloc, cgl, cgr, nullptr, nullptr, 0, a->nonfinite + 1, st);
        }
        if ((rc = lmep_comm_fork(c, st))) return rc;
        if ((rc = exchange_nccl(c, 1, fields, nloc, W, gls, grs, c->side))) return rc;
        if ((rc = sub(0, W, cgl, u + W, nullptr, nullptr, 0, a->nonfinite + 2, c->side))) return rc;
        if ((rc = sub(nloc - W, W, u + nloc - 2 * W, cgr, nullptr, nullptr, 0, a->nonfinite + 3, c->side))) return rc;
        if ((rc = sub(W, nloc - 2 * W, u, u + nloc - W, nullptr, nullptr, 0, a->nonfinite + 1, st))) return rc;
        return lmep_comm_join(c, st);
    }
    // PEER: no exchange kernel between chunks -- ghosts are read in place from this
    // rank's mailbox and the edge launches store the next chunk's halo into the
    // neighbours' mailboxes themselves
    if ((rc = peer_check(c, "lmep_comm_chunk", st))) return rc;
    if (W > c->max_width) return LMEP_DIMENSION;
    if (a->pushed_cells < W) {
        const double *fields[1] = {u};
        if ((rc = peer_push(c, 1, fields, nloc, W, st))) return rc;
    }
    double *tl = nullptr, *tr = nullptr;
    if (Wn > 0) peer_targets(c, 0, &tl, &tr);
    auto ghosts = [&](const double **gl, const double **gr) {
        const int half = (int)(c->seq & 1);
        *gl = hasL ? slot(c->mailbox, c, half, 0) : nullptr;
        *gr = hasR ? slot(c->mailbox, c, half, 1) : nullptr;
    };
    const double *gl, *gr;
    if (!split) {
        if ((rc = peer_wait(c, st))) return rc;
        ghosts(&gl, &gr);
        if ((rc = sub(0, nloc, gl, gr, tl, tr, Wn, a->nonfinite + 1, st))) return rc;
        return Wn > 0 ? peer_signal(c, st) : LMEP_OK;
    }
    if ((rc = lmep_comm_fork(c, st))) return rc;
    if ((rc = sub(W, nloc - 2 * W, u, u + nloc - W, nullptr, nullptr, 0, a->nonfinite + 1, c->side))) return rc;
    if ((rc = peer_wait(c, st))) return rc;
    ghosts(&gl, &gr);
    if ((rc = sub(0, W, gl, u + W, tl, nullptr, Wn, a->nonfinite + 2, st))) return rc;
    if ((rc = sub(nloc - W, W, u + nloc - 2 * W, gr, nullptr, tr, Wn, a->nonfinite + 3, st))) return rc;
    if (Wn > 0 && (rc = peer_signal(c, st))) return rc;
    return lmep_comm_join(c, st);
}

// ---------------------------------------------------------------------------
// graphs
// ---------------------------------------------------------------------------
// the library's own launches recorded by the capture in progress on this thread
static thread_local int64_t t_capture_base = 0;

extern "C" int lmep_graph_begin(void *stream)
{
    CUDA_TRY(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
    t_capture_base = lmep_launch_count();
    return LMEP_OK;
}

extern "C" int lmep_graph_end(void *stream, lmep_graph **out)
{
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture((cudaStream_t)stream, &g);
    if (e != cudaSuccess || !g) {
        set_last_error("cudaStreamEndCapture", e);
        cudaGetLastError();
        return LMEP_CUDA_ERROR;
    }
    if (!out) { cudaGraphDestroy(g); return LMEP_INVALID_CONFIG; }
    lmep_graph *G = new lmep_graph;
    G->graph = g;
    e = cudaGraphInstantiate(&G->exec, g, 0);
    if (e != cudaSuccess) {
        set_last_error("cudaGraphInstantiate", e);
        cudaGraphDestroy(g);
        delete G;
        return LMEP_CUDA_ERROR;
    }
    // the library's launches were counted when they were recorded, not run:
    // take them back here and count them on every replay instead
    G->kernels = lmep_launch_count() - t_capture_base;
    count_launches(-G->kernels);
    *out = G;
    return LMEP_OK;
}

extern "C" int lmep_graph_launch(lmep_graph *G, void *stream)
{
    if (!G || !G->exec) return LMEP_INVALID_CONFIG;
    CUDA_TRY(cudaGraphLaunch(G->exec, (cudaStream_t)stream));
    count_launches(G->kernels);
    return LMEP_OK;
}

extern "C" int lmep_graph_destroy(lmep_graph *G)
{
    if (!G) return LMEP_OK;
    if (G->exec) cudaGraphExecDestroy(G->exec);
    if (G->graph) cudaGraphDestroy(G->graph);
    delete G;
    return LMEP_OK;
}
