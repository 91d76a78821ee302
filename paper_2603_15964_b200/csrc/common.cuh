// common.cuh -- shared helpers of liblmep (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

// Host-side error bookkeeping (capi.cu).
void set_last_error(const char *what, cudaError_t e);
int launch_status(const char *what);

}  // namespace lmep
