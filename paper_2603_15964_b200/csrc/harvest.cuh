// harvest.cuh -- parameters shared by the harvest kernels.
#pragma once
#include "common.cuh"

namespace lmep {

struct HarvestParams {
    int mode;              // 0: expm of given matrices, 1: harvest (tables), 2: harvest (explicit L)
    int n, s, d, nterms;
    const double *tables;  // [ntab][nterms][n][n]
    const int32_t *table_idx;
    const double *coef;
    int64_t coef_stride;
    const double *c0;
    int64_t c0_stride;
    const double *L;       // [B][n][n]
    const double *Ain;     // expm mode: [B][d][d]
    double delta_t;
    const int32_t *rows;
    int row_default;
    const uint64_t *frozen;
    uint64_t frozen_default;
    int64_t B;
    int64_t out_ld;        // layout 1: leading dimension of out [s][n][out_ld] (>= B)
    int layout;
    double *out;
    int32_t *status;
    int32_t *ms;
    // row-scaled coefficients (lmep_harvest_mapped): local row i of item b
    // reads coef/c0 of node  map_node0 + b - row_b + i  (mod map_nnodes)
    int map_on, map_periodic;
    int64_t map_node0, map_nnodes;
    // optional (w_lin, raw dt/2 phi_1) rows at delta_t / 2, same layout as out
    // with s = 2 (lmep_harvest_ex half_out); only the per-item kernel emits them
    double *half_out;
    // constant-table kernels: work list between the polynomial kernel and the Taylor
    // kernel behind it (device: [0] = number of 128-item blocks handed back, then
    // their indices); null = every item
    int32_t *pending;
};

__device__ __forceinline__ int64_t coef_node(const HarvestParams &P, int64_t b, int row, int i)
{
    int64_t m = P.map_node0 + b - row + i;
    if (P.map_periodic) {
        m %= P.map_nnodes;
        if (m < 0) m += P.map_nnodes;
    }
    return m;
}

// expm-multiply harvest for d <= 16: the per-item kernel (harvest_mv.cuh,
// instantiated in harvest_mv_{a,b,c}.cu)
int launch_harvest_mv_a(const HarvestParams &P, cudaStream_t st);
int launch_harvest_mv_b(const HarvestParams &P, cudaStream_t st);
int launch_harvest_mv_c(const HarvestParams &P, cudaStream_t st);
inline int launch_harvest_mv(const HarvestParams &P, cudaStream_t st)
{
    if (P.d <= 8) return launch_harvest_mv_a(P, st);
    if (P.d <= 12) return launch_harvest_mv_b(P, st);
    return launch_harvest_mv_c(P, st);
}

// block-balanced fast path for large single-geometry per-node batches
// (harvest_mvb.cuh, instantiated in harvest_mvb_{a,b,c}.cu)
int launch_harvest_mvb_a(const HarvestParams &P, cudaStream_t st);
int launch_harvest_mvb_b(const HarvestParams &P, cudaStream_t st);
int launch_harvest_mvb_c(const HarvestParams &P, cudaStream_t st);
inline int launch_harvest_mvb(const HarvestParams &P, cudaStream_t st)
{
    if (P.d <= 10) return launch_harvest_mvb_a(P, st);
    if (P.d <= 13) return launch_harvest_mvb_b(P, st);
    return launch_harvest_mvb_c(P, st);
}
// same test as mvb_eligible (harvest_mvb.cuh), visible to harvest.cu
inline bool harvest_mvb_eligible(const HarvestParams &P)
{
    const int nt = P.nterms + (P.c0 ? 1 : 0);
    return P.mode == 1 && P.table_idx == nullptr && !P.map_on && P.rows == nullptr &&
           P.frozen == nullptr && P.frozen_default == 0 && P.nterms >= 1 && nt <= 3 &&
           P.d >= 5 && P.d <= 16 && P.B >= 4096;
}

// constant-table kernel for the largest single-geometry w_lin batches
// (harvest_mvc.cu: one item per lane, tables as constant-bank DFMA operands)
bool harvest_mvc_eligible(const HarvestParams &P);
int launch_harvest_mvc(const HarvestParams &P, cudaStream_t st);

}  // namespace lmep
