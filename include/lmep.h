/*
 * lmep.h -- C ABI of the B200-native LMEP hot path (liblmep.so).
 *
 * This is the drop-in boundary for the reference package `localexp`
 * (/root/reference/pkg/src/localexp).  The reference has no FFI: its seam is
 * the Python API listed below, and every entry point here replaces one
 * reference function (file:line).  The Python mirror of that API
 * (paper_2603_15964_b200/{harvest,kernels,timestep,...}.py) binds these
 * symbols with ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions (all entry points):
 *   - plain C types only; every array argument is a DEVICE pointer unless the
 *     comment says "host";
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream);
 *   - the return value is an lmep_status; inputs are never modified
 *     (reference: kernels.py:35,74 copy u0, harvest.py:59-62 read-only rows);
 *   - all arithmetic is IEEE fp64.
 */
#ifndef LMEP_H
#define LMEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  They map 1:1 onto localexp.errors (errors.py:4-50). */
typedef enum {
    LMEP_OK = 0,
    LMEP_NONFINITE = 1,        /* NonFinite        (expm.py:35-41, timestep.py:345-348) */
    LMEP_DIMENSION = 2,        /* DimensionMismatch (harvest.py:57-58,77-78,113-114)    */
    LMEP_INVALID_CONFIG = 3,   /* InvalidConfig / ValueError (harvest.py:85-86)         */
    LMEP_CUDA_ERROR = 4,       /* launch or runtime failure                             */
    LMEP_ORDER_TOO_HIGH = 5,   /* OrderTooHigh     (localop.py:69-70,115-116)           */
    LMEP_DUPLICATE_NODES = 6   /* DuplicateNodes   (localop.py:71-74)                   */
} lmep_status;

#define LMEP_MAX_N 32          /* largest stencil size n                              */
#define LMEP_MAX_DIM 32        /* largest exponentiated dimension d = n + s - 1       */
#define LMEP_MAX_ROWS 7        /* operator rows per step: w, alpha, beta, gamma,      */
                               /* w_half, p1_half, d1 (timestep.py:141-156)           */

/* Row slots of the operator set passed to the step kernels. */
enum {
    LMEP_ROW_W = 0,            /* linear: exp(dt L); etdrk4: w_full; etd2: exp(dt L)   */
    LMEP_ROW_ALPHA = 1,        /* etdrk4 alpha;  etd2: dt*phi1 (raw harvest row)       */
    LMEP_ROW_BETA = 2,         /* etdrk4 beta;   etd2: dt^2*phi2 (raw harvest row)     */
    LMEP_ROW_GAMMA = 3,        /* etdrk4 gamma                                         */
    LMEP_ROW_WHALF = 4,        /* etdrk4 w_half                                        */
    LMEP_ROW_P1HALF = 5,       /* etdrk4 p1_half                                       */
    LMEP_ROW_D1 = 6            /* banded first derivative for N(u) = -u * (D1 u)       */
};

/* Nonlinearity kinds: kernels.py:17-19. */
enum { LMEP_NL_NONE = 0, LMEP_NL_CONVECTIVE = 1, LMEP_NL_CUBIC = 2 };

/* Weight storage modes of the step kernels. */
enum {
    LMEP_W_SHARED = 0,         /* one row set for every node (periodic uniform grid)  */
    LMEP_W_CLASS = 1,          /* nleft + 1 + nright row sets selected by position    */
    LMEP_W_PERNODE = 2         /* per-node rows, SoA [nrows][n][nloc]                  */
};

/* Boundary handling applied where the reference pins (kernels.py:39-41,93-95,
 * 101-103,112-114,129-131). */
enum { LMEP_BC_NONE = 0, LMEP_BC_DIRICHLET = 1, LMEP_BC_NEUMANN = 2 };

/* Step flags. */
enum {
    LMEP_FLAG_EXACT = 1        /* separate multiply/add roundings, ascending order:   */
                               /* bit-identical to the numba loops (kernels.py:8-9)    */
};

/* 1D stencil geometry of one shard (grid.py:136-175).  Node t of the global grid
 * (0 <= t < N) reads the window start(t) .. start(t)+n-1 with
 *   periodic:     start(t) = t - row (mod N)
 *   non-periodic: start(t) = clamp(t - row, 0, N - n).
 * The shard owns global nodes off .. off+nloc-1. */
typedef struct {
    int64_t N;
    int64_t off;
    int64_t nloc;
    int32_t n;
    int32_t row;
    int32_t periodic;
    int32_t reserved;
} lmep_grid;

/* Operator rows.  `interior` is a HOST pointer to [nrows][n] rows used for
 * every interior node (mode SHARED and CLASS).  CLASS: `classes` is a device
 * [nleft+1+nright][nrows][n] table; node t uses class t for t < nleft,
 * nleft+1+(t-(N-nright)) for t >= N-nright, and the interior set otherwise.
 * PERNODE: `pernode` is a device SoA [nrows][n][nloc + 2*pernode_pad] table of
 * this shard: local node i at column i + pernode_pad, the pad columns holding
 * the rows of the halo nodes (needed to fuse several steps per exchange). */
typedef struct {
    int32_t mode;
    int32_t nrows;
    int32_t nleft;
    int32_t nright;
    const double *interior;    /* host   */
    const double *classes;     /* device */
    const double *pernode;     /* device */
    int64_t pernode_pad;
} lmep_weights;

/* Boundary closure (non-periodic grids).  DIRICHLET pins u[0]=lo, u[N-1]=hi
 * (timestep.py:129-133).  NEUMANN applies the zero-gradient closure
 *   u[0]   = -sum_{j>=1} dl[j] u[j] / dl[0]
 *   u[N-1] = -sum_{j<n-1} dr[j] u[N-n+j] / dr[n-1]
 * (SURVEY Appendix B.2).  dl/dr are HOST pointers to n values. */
typedef struct {
    int32_t kind;
    int32_t reserved;
    double lo, hi;
    const double *dl;
    const double *dr;
} lmep_bc;

/* Ghost cells of a sharded run (1D slab decomposition, filled by the caller's
 * halo exchange).  `left` holds global nodes off-width .. off-1 and `right`
 * holds off+nloc .. off+nloc+width-1 (wrapped on periodic grids).  All NULL:
 * a single shard covering the whole grid (periodic wrap is done in-kernel). */
typedef struct {
    const double *left;
    const double *right;
    const double *hist_left;   /* etd2 history ghosts */
    const double *hist_right;
    int64_t width;
    /* Fused peer stores (optional, linear and ETDRK4 launches with shared / class
     * rows): besides u_out, the launch stores its first push_width results at
     * push_left[0 ..] and its last push_width results at push_right[0 ..] --
     * the neighbours' mailbox slots from lmep_comm_targets, i.e. peer memory over
     * NVLink -- so the next chunk's halo needs no exchange kernel at all. */
    double *push_left;
    double *push_right;
    int64_t push_width;
} lmep_halo;

/* Optional launch shape.  0 = library heuristic. */
typedef struct {
    int32_t tile;              /* owned nodes per CTA                                 */
    int32_t ksteps;            /* time steps fused per launch (temporal blocking)     */
    int32_t ring;              /* 1: whole periodic grid resident in one CTA          */
    int32_t threads;           /* threads per CTA (multiple of 32, <= 256)            */
} lmep_tuning;

/* ---- library ------------------------------------------------------------ */
int lmep_version(void);
const char *lmep_status_string(int status);
/* Last CUDA error string seen by the library (host, static storage). */
const char *lmep_last_error(void);
/* Number of kernels this library has launched in this process (for the
 * bench's gpu_launches accounting). */
int64_t lmep_launch_count(void);

/* ---- harvest (K1, K2) --------------------------------------------------- */

/* Fornberg weight tables, one thread per item b:
 *   out[b][k][j] = weight of sample x_b[j] for d^k/dx^k at z[b], k = 0..m.
 * x is [B][n] with row stride x_stride (0 = one node set shared by all items).
 * Replaces localop.fornberg_weights (localop.py:61-96); bit-identical. */
int lmep_fornberg(const double *z, const double *x, int64_t x_stride, int n, int m,
                  int64_t B, double *out, void *stream);

/* Batched exp(A) of B dense d x d matrices (row-major [B][d][d]), one warp per
 * matrix: balancing (permute=False), Pade scaling-and-squaring (Al-Mohy &
 * Higham 2009, the algorithm scipy.linalg.expm implements), unbalancing.
 * Replaces expm.expm (expm.py:24-42).  status[b] (nullable) gets
 * LMEP_OK / LMEP_NONFINITE per matrix, ms[b] (nullable) = m | (squarings << 8).
 * Returns LMEP_NONFINITE only via status[]; the call itself returns launch status. */
int lmep_expm(const double *A, int d, int64_t B, double *E, int32_t *status, int32_t *ms,
              void *stream);

/* Batched weight harvest (harvest.py:73-121 + 135-159), one warp per item.
 * Item b's local operator is assembled in shared memory exactly as
 * localop.local_operator (localop.py:111-128) does it:
 *   L = sum_t coef[b*coef_stride + t] * tables[table_idx[b]][t]   (ascending t)
 *   L[i][i] += c0[b*c0_stride]                                      (if != 0)
 * where tables is [ntab][nterms][n][n] (derivative matrices D^(k) on that
 * item's local coordinates, e.g. from lmep_fornberg).  If `L` is non-NULL it
 * is used instead ([B][n][n], explicit operators; tables/coef/c0 ignored).
 * Rows listed in the frozen bitmask are zeroed (harvest.py:116-117).  The
 * exponential is taken of the reduced (n+s-1) x (n+s-1) transposed
 * augmentation [[dt L^T, dt e_r, 0], [0, 0, dt J]] instead of the sn x sn block
 * companion (harvest.py:82-94); both yield the same rows.
 * Output rows: w_lin = row r of exp(dt L), then the raw dt^j phi_j rows,
 * j = 1..s-1 (harvest.py:119-120).
 *   layout 0: w_out[b][j][i]  ([B][s][n], reference order)
 *   layout 1: w_out[j][i][b]  ([s][n][B], SoA for LMEP_W_PERNODE)
 * target_row / frozen are per item (nullable -> the *_default value). */
int lmep_harvest(int n, int s, int nterms, const double *tables, const int32_t *table_idx,
                 const double *coef, int64_t coef_stride, const double *c0, int64_t c0_stride,
                 const double *L, double delta_t, const int32_t *target_row, int row_default,
                 const uint64_t *frozen, uint64_t frozen_default, int64_t B, int layout,
                 double *w_out, int32_t *status, int32_t *ms, void *stream);

/* Row-scaled variable coefficients: with a map, local
 * row i of item b takes coef[m * coef_stride + t] and c0[m * c0_stride] of
 * node m = node0 + b - row_b + i (mod nnodes when periodic) -- the operator
 * sum_t diag(c_t) D^(k_t) + diag(c0) restricted to the stencil, instead of
 * the coefficients frozen at the target node.  coef / c0 then index the
 * whole grid (nnodes rows), items are the consecutive nodes node0, node0+1, ...
 * Table mode only (L == NULL). */
typedef struct lmep_coef_map {
    int64_t node0;
    int64_t nnodes;
    int32_t periodic;
    int32_t reserved;
} lmep_coef_map;

int lmep_harvest_mapped(int n, int s, int nterms, const double *tables, const int32_t *table_idx,
                        const double *coef, int64_t coef_stride, const double *c0,
                        int64_t c0_stride, const double *L, double delta_t,
                        const int32_t *target_row, int row_default, const uint64_t *frozen,
                        uint64_t frozen_default, int64_t B, int layout, double *w_out,
                        int32_t *status, int32_t *ms, const lmep_coef_map *map, void *stream);

/* One slice of a larger per-node harvest (host-pipelined uploads): as
 * lmep_harvest_mapped, but the layout-1 output [s][n][out_ld] has leading
 * dimension out_ld >= B.  To harvest items [a, a+B) of a table of out_ld
 * items, offset coef / c0 by a rows, target_row / frozen / status / ms by a,
 * w_out by a, and map->node0 by a.  Layout 0 ignores out_ld.
 * Replaces the per-node loop of harvest._harvest_rows (harvest.py:135-159)
 * for one contiguous node range. */
int lmep_harvest_chunk(int n, int s, int nterms, const double *tables, const int32_t *table_idx,
                       const double *coef, int64_t coef_stride, const double *c0,
                       int64_t c0_stride, const double *L, double delta_t,
                       const int32_t *target_row, int row_default, const uint64_t *frozen,
                       uint64_t frozen_default, int64_t B, int layout, double *w_out,
                       int32_t *status, int32_t *ms, const lmep_coef_map *map, int64_t out_ld,
                       void *stream);

/* Slices of ONE harvest (lmep_harvest_chunk / lmep_harvest_ex calls over
 * consecutive item ranges of one table): while on (per host thread), a
 * constant-table harvest whose tables, step and shape equal those of the
 * device's previous one keeps that call's prepared block (the balancing of the
 * first slice's first item), so the rows equal a one-launch harvest's bit for
 * bit whatever the slicing, and later slices skip the prep kernel. */
int lmep_harvest_reuse_prep(int on);

/* All harvest options in one argument block (lmep_harvest_chunk's arguments
 * plus two):
 *   half_out   (nullable, s >= 2) also the (w_lin, raw dt/2 phi_1) rows of
 *              every item at delta_t / 2 -- the ETDRK4 half-step set
 *              (timestep.py:294-299) -- in the layout of w_out with s = 2
 *              (layout 1: leading dimension out_ld).  The per-item kernel takes
 *              them from the same exponential (an even number of scaling reps,
 *              the iterate after half of them); kernels that emit one set are
 *              followed by a second launch at delta_t / 2.
 *   status_any (nullable, device int32, needs `status`) set to 1 when any
 *              item's status is not LMEP_OK (never cleared: the caller zeroes
 *              it and may share it between harvests). */
typedef struct lmep_harvest_args {
    int32_t n, s, nterms, layout;
    const double *tables;
    const int32_t *table_idx;
    const double *coef;
    int64_t coef_stride;
    const double *c0;
    int64_t c0_stride;
    const double *L;
    double delta_t;
    const int32_t *target_row;
    int64_t row_default;
    const uint64_t *frozen;
    uint64_t frozen_default;
    int64_t B;
    int64_t out_ld;
    double *w_out;
    int32_t *status;
    int32_t *ms;
    const lmep_coef_map *map;
    double *half_out;
    int32_t *status_any;
} lmep_harvest_args;

int lmep_harvest_ex(const lmep_harvest_args *args, void *stream);

/* Set *flag (device int32) to 1 if any of status[0..B) is not LMEP_OK. */
int lmep_status_any(const int32_t *status, int64_t B, int32_t *flag, void *stream);

/* Ordered linear combination of row arrays, harvest.combine (harvest.py:225-235):
 *   out[r*ld_out + j] = (((0 + c[0]*in[0][r*ld_in[0] + j]) + c[1]*in[1][...]) + ...)
 * for r < rows, j < cols, numpy's two roundings per term in list order.  `in`,
 * `ld_in` and `coef` are HOST arrays of nterm <= 8 entries; the data is device
 * memory.  timestep.etdrk4_operators (timestep.py:141-156) composes alpha,
 * beta and gamma with it straight from the harvest output. */
int lmep_combine(int nterm, const double *const *in, const int64_t *ld_in, const double *coef,
                 int64_t rows, int64_t cols, double *out, int64_t ld_out, void *stream);

/* Compare every row of a device (N, n) weight array with row `ref`:
 * out3 (device uint64[3]) = {first equal row, last equal row, count}.  The
 * shim's compression of reference-style weights into shared / class /
 * per-node rows reads these three numbers instead of the whole array. */
int lmep_rows_classify(const double *rows, int64_t N, int n, int64_t ref, uint64_t *out3,
                       void *stream);

/* Symbol of one weight row on [0, kmax] (analysis.spectral_footprint,
 * analysis.py:42-64): for k_i = i kmax / (num_k - 1),
 *   G(k) = sum_j w[j] exp(i k offsets_h[j]),  |G|,  arg(G exp(i k shift)).
 * w and offsets_h (offsets times h) are HOST arrays of n <= 32 values; the
 * four outputs are device arrays of num_k doubles. */
int lmep_spectral_footprint(const double *w, const double *offsets_h, int n, double kmax,
                            int num_k, double shift, double *g_re, double *g_im, double *g_abs,
                            double *dispersion, void *stream);

/* Harvest algorithm for d <= 16:
 *   0 (default) = expm-multiply: large single-geometry batches (n in
 *     {7, 9, 11, 13}, B >= 4096; s = 1 with <= 2 tables, or s <= 4 with two
 *     tables and no reaction) take the constant-table
 *     kernel (harvest_mvc.cu: one item per lane, launch-uniform balancing,
 *     tables as constant-bank operands); other large single-geometry
 *     batches (B >= 4096, one
 *     shared table, one target row, no frozen rows) take the block-balanced
 *     kernel (harvest_mvb.cuh: one balancing per superblock of 1024 items folded into the
 *     tables, inf-norm bound scaling, rigorous Taylor tail stop, 2 lanes per
 *     item for d <= 13, else 4); everything else the per-item kernel
 *     (harvest_mv.cuh: per-item balancing, 4 lanes per item);
 *   1 = full Pade scaling-and-squaring per warp (harvest.cu);
 *   2 / 3 = retired (the first-generation kernel): LMEP_INVALID_CONFIG;
 *   4 = the per-item kernel with 8 lanes per item for d > 8;
 *   5 = the per-item kernel only (no block-balanced path);
 *   6 / 7 / 8 = as 0 with the block-balanced kernel forced to 8 / 2 / 4 lanes
 *     per item (tuning, tests), no constant-table kernel;
 *   9 = as 0 without the constant-table kernel.
 * lmep_expm always uses the Pade kernel.  The setting belongs to the calling
 * thread's current CUDA device; returns LMEP_INVALID_CONFIG for other codes. */
int lmep_set_harvest_method(int method);

/* Ring mode of the linear scheme (a periodic grid resident on chip for all
 * steps, BASELINE config 1): 1 (default) = one thread-block cluster of 8 CTAs
 * exchanging halos through distributed shared memory every kb steps -- small
 * rings (N % 32 == 0, N up to ~3000) with warp-private slabs held in registers
 * and windows built by warp shuffles (ring_lin_warp_kernel), larger ones with
 * one node per thread in shared memory (ring_lin_cluster_kernel, N % 8 == 0);
 * 2 = the shared-memory cluster kernel only; 0 = one CTA (ring_lin_kernel).
 * Per-device setting (the current device); results are bit-identical either way. */
int lmep_set_ring_cluster(int on);

/* Kernel of the persistent TMA-pipelined per-node linear steps (BASELINE
 * config 5): 1 = register-resident values with a slot-major halo exchange
 * (lin_pernode_tmx_kernel; centred n <= 13 and n = 7 one-sided), 0 = the
 * shared-memory window kernel (lin_pernode_tma_kernel), 2 (default) = the
 * register kernel for fused multiply-adds, the window kernel for the exact
 * order.  Per-device setting; results are bit-identical in the exact mode. */
int lmep_set_pernode_kernel(int variant);

/* ---- sharded runs (K6): communicator, halo exchange, graphs --------------- */

/* One communicator per rank (one process per GPU) of a 1D slab decomposition
 * (the reference has no collectives -- timestep.run, timestep.py:
 * 255-394, advances one array).  Rank r's neighbours are r-1 / r+1, wrapped
 * on a periodic ring; with world == 1 and periodic != 0 the rank is its own
 * neighbour on both sides (the self-exchange that checks the data path on one
 * GPU).  Two transports move the halos:
 *   LMEP_COMM_NCCL  ncclSend / ncclRecv pairs in one group on the caller's
 *                   stream (libnccl.so.2 is resolved at run time);
 *   LMEP_COMM_PEER  CUDA IPC on one node: every rank owns a device mailbox,
 *                   the exchange STORES its edges straight into the
 *                   neighbours' mailboxes (one kernel writing peer memory
 *                   over NVLink), signals with an interprocess event and
 *                   copies its own mailbox out after waiting for the
 *                   neighbours' events.  Mailboxes are double buffered; all
 *                   exchanges of a communicator must be issued in one stream
 *                   order.  Not capturable in a CUDA graph (the ranks meet on
 *                   the host before each wait).
 * Bootstrap is out of band, as with ncclUniqueId: the caller moves a few
 * bytes between the ranks with whatever it has (MPI, a torch.distributed
 * store, a file). */
typedef struct lmep_comm lmep_comm;
enum { LMEP_COMM_NCCL = 0, LMEP_COMM_PEER = 1 };
#define LMEP_COMM_ID_BYTES 128     /* ncclUniqueId                                    */
#define LMEP_COMM_BLOB_BYTES 512   /* one rank's IPC handles (PEER transport)         */
#define LMEP_COMM_MAX_FIELDS 8     /* arrays exchanged together (u + ETD history)     */

/* NCCL: rank 0 fills id (host, LMEP_COMM_ID_BYTES) and hands it to every rank. */
int lmep_comm_unique_id(void *id);

/* Create rank `rank` of `world` on the calling thread's current device.
 * NCCL: `id` from lmep_comm_unique_id (collective: every rank calls).
 * PEER: id is ignored; max_width = the widest halo (doubles per field and
 * side) the mailboxes must hold; the communicator is usable after
 * lmep_comm_connect. */
int lmep_comm_init(lmep_comm **comm, int rank, int world, int periodic, int transport,
                   const void *id, int64_t max_width);
/* PEER: this rank's IPC handles (host, LMEP_COMM_BLOB_BYTES) ... */
int lmep_comm_export(lmep_comm *comm, void *blob);
/* ... and, once the caller has gathered them, every rank's blobs in rank
 * order (host, world * LMEP_COMM_BLOB_BYTES).  NCCL: both are no-ops. */
int lmep_comm_connect(lmep_comm *comm, const void *blobs);
int lmep_comm_destroy(lmep_comm *comm);
/* left / right = neighbour ranks, -1 at the ends of an open chain. */
int lmep_comm_info(const lmep_comm *comm, int *rank, int *world, int *left, int *right,
                   int *transport);

/* Fill the ghost cells of nfields arrays of nloc doubles each: ghost_left[f]
 * receives the left neighbour's last `width` values of field f, ghost_right[f]
 * the right neighbour's first `width` (a rank without a neighbour on a side
 * leaves that buffer alone).  fields / ghost_left / ghost_right are HOST
 * arrays of nfields device pointers.  One NCCL group (or one peer-store
 * kernel) moves all fields.  Asynchronous on `stream`. */
int lmep_halo_exchange(lmep_comm *comm, int nfields, const double *const *fields, int64_t nloc,
                       int64_t width, double *const *ghost_left, double *const *ghost_right,
                       void *stream);

/* PEER transport, piecewise (what lmep_halo_exchange does in one call is
 * push + wait + a copy out of the mailbox):
 *   lmep_comm_targets  where this rank's edges of field f go for its NEXT signal:
 *                      the neighbours' mailbox slots (peer pointers; NULL without
 *                      a neighbour).  A step launch given them as lmep_halo.push_*
 *                      stores its edges there itself.
 *   lmep_comm_push     store the edges of `fields` there with the library's kernel
 *                      and signal (the first chunk, or after a standalone step).
 *   lmep_comm_signal   the edges are stored (stream order): record the
 *                      interprocess event and publish the exchange number.
 *   lmep_comm_wait     make `stream` wait for the neighbours' signal that matches
 *                      this rank's latest one (the host meets them first).
 *   lmep_comm_ghosts   this rank's own mailbox slots of that exchange: pass them as
 *                      lmep_halo.left / right, no copy. */
int lmep_comm_targets(lmep_comm *comm, int field, double **to_left, double **to_right);
int lmep_comm_push(lmep_comm *comm, int nfields, const double *const *fields, int64_t nloc,
                   int64_t width, void *stream);
int lmep_comm_signal(lmep_comm *comm, void *stream);
int lmep_comm_wait(lmep_comm *comm, void *stream);
int lmep_comm_ghosts(lmep_comm *comm, int field, const double **left, const double **right);

/* One chunk (halo exchange + k fused steps) of a sharded linear / ETDRK4 run on
 * shared or class rows, in one call.  u_in / u_out are the slab's nloc values
 * with `ghost_cells` cells stored right before and after them (extended
 * arrays [ghosts | owned | ghosts]).  The library does what a caller would do
 * with the pieces above:
 *   NCCL  fork; side stream: exchange into the ghost cells around u_in, then
 *         the two edge strips; step stream: the interior sub-slab (its ghosts
 *         are the slab's own edge values); join.  Capturable (lmep_graph_*).
 *   PEER  the edges of u_in go out with lmep_comm_push unless `pushed_cells`
 *         says the previous chunk already stored them; fork; side stream: the
 *         interior; step stream: wait for the neighbours, the strips with their
 *         ghosts read in place from the mailbox and -- when next_steps > 0 --
 *         the next chunk's halo stored straight into the neighbours'
 *         mailboxes; signal; join.
 * Slabs narrower than three halos run unsplit.  nonfinite: device int32[4]
 * (one flag per launch; the run is finite when all are 0). */
typedef struct lmep_chunk_args {
    const lmep_grid *grid;      /* the slab: off, nloc                                 */
    const lmep_weights *w;      /* LMEP_W_SHARED or LMEP_W_CLASS                       */
    const lmep_bc *bc;          /* nullable                                            */
    int32_t scheme;             /* 0 linear, 1 ETDRK4                                  */
    int32_t nl_kind;            /* LMEP_NL_*                                           */
    const double *u_in;
    double *u_out;
    int64_t ghost_cells;        /* cells stored on each side of u_in / u_out           */
    int64_t steps;              /* k of this chunk                                     */
    int64_t next_steps;         /* k of the chunk that follows (0: none)               */
    int64_t pushed_cells;       /* PEER: edge cells of u_in already in the neighbours' mailboxes */
    int32_t flags;              /* LMEP_FLAG_*                                         */
    int32_t reserved;
    int32_t *nonfinite;
} lmep_chunk_args;
int lmep_comm_chunk(lmep_comm *comm, const lmep_chunk_args *args, void *stream);

/* Concatenate the slabs on `root`: rank r contributes nloc_r = counts[r]
 * doubles (counts: HOST array of world entries, the same on every rank); out
 * (root only) receives them in rank order.  NCCL transport only (PEER runs
 * gather through the host). */
int lmep_comm_gather(lmep_comm *comm, const double *u, const int64_t *counts, double *out,
                     int root, void *stream);
/* flag[0..count) (device int32) <- max over ranks.  NCCL transport only. */
int lmep_comm_flag_max(lmep_comm *comm, int32_t *flag, int count, void *stream);

/* A second stream owned by the communicator, for overlapping the exchange
 * with the interior of the slab: fork makes the side stream wait for the
 * work queued on `stream` so far, join makes `stream` wait for the side
 * stream.  Both are capturable (event record + wait). */
void *lmep_comm_side_stream(lmep_comm *comm);
int lmep_comm_fork(lmep_comm *comm, void *stream);
int lmep_comm_join(lmep_comm *comm, void *stream);

/* CUDA graph of a chunk (halo exchange + fused k-step launch, with the
 * interior / edge split on two streams): begin starts a thread-local capture
 * on `stream`, every lmep_* call issued on it (and on streams forked from it)
 * until lmep_graph_end is recorded instead of run.  lmep_graph_launch replays
 * it.  Device pointers are baked in: capture one graph per ping-pong
 * direction.  NCCL exchanges are capturable once the communicator has run
 * one exchange outside a capture.  Destroy every graph that captured a
 * communicator's exchanges BEFORE lmep_comm_destroy: ncclCommDestroy waits
 * for the graphs that hold its work. */
typedef struct lmep_graph lmep_graph;
int lmep_graph_begin(void *stream);
int lmep_graph_end(void *stream, lmep_graph **graph);
int lmep_graph_launch(lmep_graph *graph, void *stream);
int lmep_graph_destroy(lmep_graph *graph);

/* ETD2 (order 2) on a periodic grid with shared rows whose slabs of N / #SMs
 * nodes fit three nodes per thread (N up to ~75k; BASELINE config 2): 1
 * (default) = the whole run in ONE cooperative launch, state resident on chip,
 * neighbour CTAs trading halos through L2 every K <= 24 steps
 * (step_etd2_persist.cu); 0 = the tiled launches.  Per-device; bit-identical
 * either way in the exact mode. */
int lmep_set_etd2_persistent(int on);

/* ---- stepping (K3, K4, K5) ---------------------------------------------- */

/* Linear banded propagation u <- W u for `steps` steps (kernels.py:33-43,
 * run_linear).  u_in is not modified; the result lands in u_out.  `scratch`
 * (nloc doubles, nullable = library-allocated) is the ping-pong buffer.
 * nonfinite (nullable, device int32) is set to 1 if any produced value is
 * not finite (the caller raises NonFinite, timestep.py:345-348).
 * flags: LMEP_FLAG_EXACT clear lets the temporally blocked per-node kernels
 * (config 5) fuse each multiply-add; every other linear kernel is exact. */
int lmep_step_linear(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                     const lmep_halo *halo, const double *u_in, double *u_out,
                     double *scratch, int64_t steps, int32_t flags,
                     const lmep_tuning *tuning, int32_t *nonfinite, void *stream);

/* lmep_step_linear whose result also lands in HOST memory (the snapshot
 * timestep.run takes after each chunk, timestep.py:341-350): host_out (nloc
 * doubles; page-locked for the copies to be asynchronous) receives u_out
 * through copy_stream.  On the persistent per-node kernels (config 5) the last
 * launch is issued as `parts` launches over consecutive tile ranges and every
 * range is copied as soon as its launch has finished, so the device-to-host
 * copy overlaps the tail of the steps; every other path copies once behind the
 * last launch.  The caller synchronises copy_stream before reading host_out. */
int lmep_step_linear_host(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                          const lmep_halo *halo, const double *u_in, double *u_out,
                          double *scratch, int64_t steps, int32_t flags,
                          const lmep_tuning *tuning, int32_t *nonfinite, void *stream,
                          double *host_out, int parts, void *copy_stream);

/* Streamed linear steps: timestep.run's harvest -> steps -> snapshot sequence
 * (timestep.py:284-350) as ONE pipeline.  For per-node rows on a periodic
 * grid (one shard, even N, the persistent per-node kernels' plan; anything
 * else returns LMEP_INVALID_CONFIG and the caller steps with
 * lmep_step_linear_host once everything has landed), the rows `w->pernode` and
 * the initial values `u_in` may still be arriving when stepping starts: the
 * caller reports, in stream order, that nodes [0, nodes_ready) of both are
 * valid, and every call launches all the k-step launches whose inputs are
 * complete, in a skewed space-time order (step_stream.cu).  The call with
 * nodes_ready = N finishes the ring.  u_in, u_out and scratch are three
 * distinct N-vectors (16-byte aligned); the result lands in u_out and, range by
 * range behind the last level's launches, in host_out (nullable, page-locked)
 * through copy_stream.  Bit-identical to lmep_step_linear on the same rows.
 * `nonfinite` as in lmep_step_linear (cleared on `stream` by _begin).
 * _info: level-1 tile size (nodes), frontier margin (nodes), number of launch
 * levels and SM count, from which a caller sizes its slices (a slice ending at
 * margin + c * sms * tile gives every level c full waves of tiles).
 * _end frees the plan (LMEP_INVALID_CONFIG if the ring was never finished) and
 * reports how many launches it issued. */
typedef struct lmep_lin_stream lmep_lin_stream;
int lmep_lin_stream_begin(const lmep_grid *grid, const lmep_weights *w, const double *u_in,
                          double *u_out, double *scratch, int64_t steps, int32_t flags,
                          const lmep_tuning *tuning, int32_t *nonfinite, double *host_out,
                          void *copy_stream, void *stream, lmep_lin_stream **out);
int lmep_lin_stream_info(const lmep_lin_stream *s, int64_t *tile, int64_t *margin,
                         int32_t *levels, int32_t *sms);
int lmep_lin_stream_advance(lmep_lin_stream *s, int64_t nodes_ready, void *stream);
int lmep_lin_stream_end(lmep_lin_stream *s, int64_t *launches);

/* Slice transfers of a streamed run (timestep.py:284-313: the uploads of the
 * coefficient table and the initial state, and snapshot 0).  lmep_upload_slice
 * queues, on up_stream, coef_bytes of coefficients (event ev_coef behind them)
 * and u_bytes of the initial state (event ev_all behind both), and, on
 * down_stream behind ev_all, the copy of that part of the initial state into
 * snap_host (nullable).  Host buffers should be page-locked.  Events come from
 * lmep_event_create (no timing) and may be re-recorded once their waiters have
 * been queued; lmep_stream_wait_event makes a stream wait for one. */
int lmep_event_create(void **ev);
int lmep_event_destroy(void *ev);
int lmep_stream_wait_event(void *stream, void *ev);
int lmep_upload_slice(void *coef_dev, const void *coef_host, size_t coef_bytes,
                      void *u_dev, const void *u_host, void *snap_host, size_t u_bytes,
                      void *up_stream, void *down_stream, void *ev_coef, void *ev_all);

/* Fused four-stage ETDRK4 (kernels.py:62-132, run_etdrk4): rows W, ALPHA, BETA,
 * GAMMA, WHALF, P1HALF (and D1 for LMEP_NL_CONVECTIVE).  nl0_out (nullable)
 * receives N(u_in) on the owned nodes (the history entry the ETD multistep
 * warm-up stores, timestep.py:375-378). */
int lmep_step_etdrk4(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                     const lmep_halo *halo, int nl_kind, const double *u_in,
                     double *u_out, double *scratch, int64_t steps, double *nl0_out,
                     int32_t flags, const lmep_tuning *tuning, int32_t *nonfinite,
                     void *stream);

/* Exponential multistep of order 2 (timestep.py:187-215, s=2):
 *   N_k = N(u);  u <- W u + P1 N_k + P2 (N_k - N_{k-1}) / dt
 * with rows W (exp), ALPHA (raw dt*phi1), BETA (raw dt^2*phi2) and D1.
 * hist_in = N_{k-1}; hist_out receives the last N_k.  scratch: 2*nloc doubles. */
int lmep_step_etd2(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                   const lmep_halo *halo, int nl_kind, double delta_t, const double *u_in,
                   const double *hist_in, double *u_out, double *hist_out, double *scratch,
                   int64_t steps, int32_t flags, const lmep_tuning *tuning,
                   int32_t *nonfinite, void *stream);

/* Exponential multistep of order s = `order` (1..5), the literal formula of
 * timestep.py:187-215 (without gamma-coefficient conversion):
 *   u <- W u + sum_{j<s} P_{j+1} grad^j N / dt^j,
 *   grad^j N = sum_{i<=j} (-1)^i C(j,i) N_{k-i}
 * rows W (exp) and P_j = raw dt^j phi_j at slots 0..s (ALPHA = P_1 ...), D1 for
 * convective N.  hist_in / hist_out: [s-1][nloc], newest first (N_{k-1} ...);
 * halo hist ghosts [s-1][width].  scratch: s*nloc doubles. */
int lmep_step_etds(const lmep_grid *grid, const lmep_weights *w, const lmep_bc *bc,
                   const lmep_halo *halo, int nl_kind, int order, double delta_t,
                   const double *u_in, const double *hist_in, double *u_out, double *hist_out,
                   double *scratch, int64_t steps, int32_t flags, const lmep_tuning *tuning,
                   int32_t *nonfinite, void *stream);

/* Plain banded mat-vec out[i] = sum_j w[i][j] * u[members(i, j)] with the
 * grid's window rule (kernels.py:23-29, harvest.apply at harvest.py:213-222). */
int lmep_banded_matvec(const lmep_grid *grid, const lmep_weights *w, const lmep_halo *halo,
                       const double *u, double *out, int32_t flags, void *stream);

/* Chooses the launch shape the library would use (for reporting/tests).
 * scheme: 0 linear, 1 etdrk4, 2 etd2; weight_mode: LMEP_W_*. */
int lmep_plan(const lmep_grid *grid, int scheme, int nl_kind, int weight_mode, int64_t steps,
              lmep_tuning *out);

/* Transpose (N, n) row-major per-node rows into the SoA [n][N] layout. */
int lmep_rows_to_soa(const double *rows, int64_t N, int n, double *soa, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LMEP_H */
