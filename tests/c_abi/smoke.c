/* A C program on the C ABI alone (include/lmep.h + liblmep.so + the CUDA runtime; no
 * Python, no torch): BASELINE config 1's path end to end -- Fornberg tables of the
 * upwind window, the harvest of the one shared weight row (harvest.py:73-79), 60 linear
 * steps (kernels.py:33-43) -- checked against the same loop on the host.  The row comes
 * back from the device, so the steps must agree BIT FOR BIT (LMEP_FLAG_EXACT).
 *   nvcc -Xcompiler -ffp-contract=off -I include tests/c_abi/smoke.c -L <lib> -llmep -o smoke */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lmep.h"

#define CHECK(call)                                                              \
    do {                                                                         \
        int rc_ = (call);                                                        \
        if (rc_ != 0) {                                                          \
            fprintf(stderr, "%s -> %d (%s) %s\n", #call, rc_, lmep_status_string(rc_), lmep_last_error()); \
            return 1;                                                            \
        }                                                                        \
    } while (0)
#define CUDA(call)                                                               \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_)); return 1; } \
    } while (0)

enum { N = 1024, n = 7, ROW = 6, STEPS = 60 };

int main(void)
{
    const double h = 2.0 * M_PI / N, dt = 3.5 * h, c = 1.0;
    double x[n], z[n];
    for (int j = 0; j < n; ++j) x[j] = z[j] = (j - ROW) * h;        /* window of the target node */

    /* D^(1) on the window: one Fornberg item per window node (shared node set, stride 0) */
    double *dx, *dz, *dtab, *dfull;
    CUDA(cudaMalloc((void **)&dx, sizeof x));
    CUDA(cudaMalloc((void **)&dz, sizeof z));
    CUDA(cudaMalloc((void **)&dfull, sizeof(double) * n * 2 * n));
    CUDA(cudaMalloc((void **)&dtab, sizeof(double) * n * n));
    CUDA(cudaMemcpy(dx, x, sizeof x, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dz, z, sizeof z, cudaMemcpyHostToDevice));
    CHECK(lmep_fornberg(dz, dx, 0, n, 1, n, dfull, NULL));
    double full[n][2][n], tab[n][n];
    CUDA(cudaMemcpy(full, dfull, sizeof full, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) tab[i][j] = full[i][1][j];       /* the first-derivative rows */
    CUDA(cudaMemcpy(dtab, tab, sizeof tab, cudaMemcpyHostToDevice));

    /* harvest: row ROW of exp(dt * (-c D^(1))), one item */
    double coef = -c, *dcoef, *dw;
    int32_t *dstatus, status = -1;
    CUDA(cudaMalloc((void **)&dcoef, sizeof coef));
    CUDA(cudaMalloc((void **)&dw, sizeof(double) * n));
    CUDA(cudaMalloc((void **)&dstatus, sizeof status));
    CUDA(cudaMemcpy(dcoef, &coef, sizeof coef, cudaMemcpyHostToDevice));
    CHECK(lmep_harvest(n, 1, 1, dtab, NULL, dcoef, 1, NULL, 0, NULL, dt, NULL, ROW, NULL, 0, 1, 0, dw,
                       dstatus, NULL, NULL));
    double w[n];
    CUDA(cudaMemcpy(w, dw, sizeof w, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(&status, dstatus, sizeof status, cudaMemcpyDeviceToHost));
    double sum = 0.0;
    for (int j = 0; j < n; ++j) sum += w[j];
    if (status != LMEP_OK || fabs(sum - 1.0) > 1e-12) {            /* a propagator row of a derivative sums to 1 */
        fprintf(stderr, "harvest: status %d, row sum %.17g\n", status, sum);
        return 1;
    }

    /* 60 steps on the device ... */
    static double u0[N], ua[N], ub[N], ud[N];
    for (int i = 0; i < N; ++i) u0[i] = sin(i * h) + 0.3 * cos(5 * i * h + 0.7);
    double *du, *dout;
    int32_t *dflag, flag = -1;
    CUDA(cudaMalloc((void **)&du, sizeof u0));
    CUDA(cudaMalloc((void **)&dout, sizeof u0));
    CUDA(cudaMalloc((void **)&dflag, sizeof flag));
    CUDA(cudaMemcpy(du, u0, sizeof u0, cudaMemcpyHostToDevice));
    lmep_grid g = {N, 0, N, n, ROW, 1, 0};
    lmep_weights W = {LMEP_W_SHARED, 1, 0, 0, w, NULL, NULL, 0};
    CHECK(lmep_step_linear(&g, &W, NULL, NULL, du, dout, NULL, STEPS, LMEP_FLAG_EXACT, NULL, dflag, NULL));
    CUDA(cudaMemcpy(ud, dout, sizeof ud, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(&flag, dflag, sizeof flag, cudaMemcpyDeviceToHost));

    /* ... and the reference loop on the host (kernels.py:23-43: ascending taps, a product
     * and a sum per tap, no contraction) */
    memcpy(ua, u0, sizeof u0);
    for (int s = 0; s < STEPS; ++s) {
        for (int i = 0; i < N; ++i) {
            double acc = 0.0;
            for (int j = 0; j < n; ++j) {
                volatile double prod = w[j] * ua[((i - ROW + j) % N + N) % N];
                acc = acc + prod;
            }
            ub[i] = acc;
        }
        memcpy(ua, ub, sizeof ua);
    }
    if (flag != 0 || memcmp(ua, ud, sizeof ua) != 0) {
        double worst = 0.0;
        for (int i = 0; i < N; ++i) worst = fmax(worst, fabs(ua[i] - ud[i]));
        fprintf(stderr, "steps differ: flag %d, max |diff| %.3g\n", flag, worst);
        return 1;
    }
    printf("c-abi smoke ok: row sum %.17g, %d steps bit-identical, %lld library launches\n", sum, STEPS,
           (long long)lmep_launch_count());
    return 0;
}
