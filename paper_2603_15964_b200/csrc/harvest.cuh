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
    int layout;
    double *out;
    int32_t *status;
    int32_t *ms;
};

// expm-multiply harvest for d <= 16 (harvest_quad.cu)
int launch_harvest_quad(const HarvestParams &P, cudaStream_t st);
void set_lanes_per_item(int lpi);

}  // namespace lmep
