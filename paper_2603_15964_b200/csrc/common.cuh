// common.cuh -- shared helpers of liblmep (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "lmep.h"

namespace lmep {

constexpr unsigned FULL = 0xffffffffu;

// Exact IEEE operations that the compiler may not contract into FMA.  They
// reproduce numpy / numba (no fastmath, kernels.py:8-9) roundings bit for bit.
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// acc + w*v, either with two roundings (EXACT, numba order) or one FMA.
template <bool EXACT>
__device__ __forceinline__ double macc(double acc, double w, double v)
{
    if constexpr (EXACT) return __dadd_rn(acc, __dmul_rn(w, v));
    else return fma(w, v, acc);
}

// Host-side error bookkeeping (capi.cu).  The last error is per host thread.
void set_last_error(const char *what, cudaError_t e);
void set_last_error_text(const char *what, const char *msg);   // non-CUDA failures (NCCL, IPC)
int launch_status(const char *what);
void count_launches(int64_t k);       // kernels replayed by a graph launch

// Device status reductions (rows.cu): *flag = 1 if any status[i] != LMEP_OK;
// dst[i] = src[i] where dst[i] == LMEP_OK.
int launch_status_or(const int32_t *status, int64_t B, int32_t *flag, cudaStream_t st);
int launch_status_merge(int32_t *dst, const int32_t *src, int64_t B, cudaStream_t st);

// Per-device library state (capi.cu).  One process may drive several GPUs
// (and several host threads may call in concurrently): nothing device-specific
// is cached process-wide.
constexpr int kMaxDevices = 64;
int current_device();                 // cudaGetDevice, clamped to [0, kMaxDevices)
int device_sm_count();                // SM count of the current device (cached per device)

// Method switches of lmep_set_harvest_method / lmep_set_ring_cluster, one set
// per device (the setter applies to the calling thread's current device).
struct DeviceSettings {
    std::atomic<int> harvest_method{0};   // 0 auto (expm-multiply for d <= 16), 1 Pade
    std::atomic<int> mv_lanes{0};         // block / per-item lanes override (0 = heuristic)
    std::atomic<int> mvc{1};              // constant-table kernel when eligible (2: without its polynomial kernel)
    std::atomic<int> ring_cluster{1};     // linear ring mode on a thread-block cluster
    std::atomic<int> pernode_kernel{2};   // TMA per-node steps: 1 registers, 0 window, 2 auto
    std::atomic<int> etd2_persistent{1};  // ETD2 on mid-size periodic grids: one cooperative launch
};
DeviceSettings &device_settings();

// "Done on this device" bitmask for one-time per-device setup (function
// attributes, pool thresholds).  The setup runs before the bit is published;
// two threads racing both run it, which is harmless for those idempotent calls.
inline bool done_on_device(const std::atomic<uint64_t> &mask, int dev)
{
    return (mask.load(std::memory_order_acquire) >> dev) & 1ull;
}
inline void mark_device(std::atomic<uint64_t> &mask, int dev)
{
    mask.fetch_or(1ull << dev, std::memory_order_release);
}

enum { SCH_LIN = 0, SCH_ETDRK4 = 1, SCH_ETD2 = 2 };

// One stepping request of the host layer (step_host.cu): what the lmep_step_*
// entry points and the sharded chunk driver (comm.cu) hand to run_steps.
struct StepCall {
    int sch;
    int etds = 2;
    const lmep_grid *grid;
    const lmep_weights *w;
    const lmep_bc *bc;
    const lmep_halo *halo;
    int nl;
    double dt;
    const double *u_in, *q_in;
    double *u_out, *q_out, *scratch;
    int64_t steps;
    int32_t flags;
    const lmep_tuning *tuning;
    int32_t *nonfinite;
    double *nl0_out;
    cudaStream_t stream;
    // lmep_step_linear_host: the result also lands in host memory, the last launch
    // split into `parts` tile ranges whose copies overlap the remaining ranges
    double *host_out = nullptr;
    int parts = 1;
    cudaStream_t copy_stream = nullptr;
};

int run_steps(const StepCall &c);

}  // namespace lmep
