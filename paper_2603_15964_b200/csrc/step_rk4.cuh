// step_rk4.cuh -- register-resident ETDRK4 passes for interior tiles (K4).
//
// Same arithmetic as the staged passes of step.cuh (kernels.py:62-132,
// run_etdrk4), reorganised so that far fewer values cross shared memory.
// The staged passes were bound by shared-memory wavefronts, not by the FP64
// pipe (ncu, profiles/r2a_c4_step_kernel.md: 2.4 wavefronts per node-step,
// FP64 pipe 47%): every banded product reloaded its window, every pointwise
// operand (whu, n0, n1) went through a slot, and b / c were stored although
// only the convective scheme reads them again.  Here every thread owns ONE
// chunk of P consecutive staged nodes for the whole launch, so
//
//   * values that are only consumed pointwise by the same node (whu = Wh u,
//     Wh a, the partial sum W u + alpha n0) stay in registers across the
//     barriers;
//   * products that share an operand share its window: Wh u, P1h N(u), W u and
//     alpha N(u) all come from one load of the u window (pointwise N is
//     recomputed on the window: 2 multiplies per element instead of a slot
//     round trip);
//   * u' overwrites u in place (u is last read before the first barrier).
//
// Pointwise N (cubic / none), per step:      windows  stores  barriers
//   A  whu, a = whu + P1h n0, n1 = N(a), t01    u       a, n1     1
//   B  b = whu + P1h n1, t2, s12               n1      t2, s12    1
//   C  c = Wh a + P1h t2, n3 = N(c)           a, t2      n3       1
//   D  u' = (t01 + beta s12) + gamma n3      s12, n3     u'       1
// 6 windows + 6 stores per node-step against 13 windows, 11 stores and 5
// pointwise loads before.  Convective N needs one more window per stage for
// D1 (n_i = -x D1 x): 9 windows + 9 stores in 8 passes.
//
// Nodes near the ends of the staged range read stale neighbours; as in
// fast_pass they are computed anyway and never stored.  EX instantiations
// keep every rounding of the reference order (bit-identical to numba).
#pragma once

namespace lmep {

// one banded product: output q of a chunk from its register window
template <int NS, bool EX>
__device__ __forceinline__ double band_reg(const double (&wrow)[LMEP_MAX_N], const double *win, int q)
{
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < NS; ++j) acc = macc<EX>(acc, wrow[j], win[q + j]);
    return acc;
}

// init + banded product.  EX: the product accumulated from zero and one
// separate addition (the reference's roundings); fused mode: the chain starts
// from init, which saves the addition.
template <int NS, bool EX>
__device__ __forceinline__ double band_add(double init, const double (&wrow)[LMEP_MAX_N],
                                           const double *win, int q)
{
    if constexpr (EX) return xadd(init, band_reg<NS, true>(wrow, win, q));
    else {
        double acc = init;
#pragma unroll
        for (int j = 0; j < NS; ++j) acc = fma(wrow[j], win[q + j], acc);
        return acc;
    }
}

template <int NS, int P, bool EX, int NLK>
__device__ __forceinline__ void etdrk4_regs_pointwise(const StepParams &p, double *sm, const int slen,
                                                      const int len, const int K, const int64_t O0,
                                                      const int64_t O1, const int64_t base)
{
    constexpr int W = P + NS - 1;
    const int eL = p.eL;
    double *XU = sm, *XA = sm + slen, *XN = sm + 2 * slen, *XT2 = sm + 3 * slen, *XS = sm + 4 * slen;
    const int l0 = eL + (int)threadIdx.x * P;             // this thread's chunk [l0, l0 + P)
    const bool act = l0 < len;
    auto sub2 = [](double n2, double n0) { return EX ? xsub(xmul(2.0, n2), n0) : 2.0 * n2 - n0; };
    for (int s = 0; s < K; ++s) {
        double whu[P], t01[P];
        if (act) {                                        // A: one window of u feeds four products
            double uw[W], nw[W];
            const double *x = XU + (l0 - eL);
#pragma unroll
            for (int i = 0; i < W; ++i) uw[i] = x[i];
#pragma unroll
            for (int i = 0; i < W; ++i) nw[i] = nlp<EX>(NLK, uw[i], 0.0);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                whu[q] = band_reg<NS, EX>(p.wi[LMEP_ROW_WHALF], uw, q);
                const double a = band_add<NS, EX>(whu[q], p.wi[LMEP_ROW_P1HALF], nw, q);
                t01[q] = band_add<NS, EX>(band_reg<NS, EX>(p.wi[LMEP_ROW_W], uw, q),
                                          p.wi[LMEP_ROW_ALPHA], nw, q);
                XA[l0 + q] = a;
                XN[l0 + q] = nlp<EX>(NLK, a, 0.0);
            }
            if (s == 0 && p.nl0_out) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int64_t g = base + l0 + q;
                    if (g >= O0 && g < O1) p.nl0_out[g - p.off] = nlp<EX>(NLK, XU[l0 + q], 0.0);
                }
            }
        }
        __syncthreads();
        // The a window of pass C is already final during B: it is loaded there and
        // held in registers across the barrier, so C starts on Wh a while its t2
        // window is in flight.  (Doing the same for s12 in D, or for wider stencils,
        // spills at 128 registers.)
        constexpr bool PRE = NS <= 7;
        double aw[W];
        if (act) {                                        // B: b from the n1 window; t2, s12
            double n1w[W], n0c[P], n1c[P];
            const double *x = XN + (l0 - eL), *xa = XA + (l0 - eL);
#pragma unroll
            for (int i = 0; i < W; ++i) n1w[i] = x[i];
#pragma unroll
            for (int q = 0; q < P; ++q) {                 // (a runtime index into the window would spill it)
                n0c[q] = XU[l0 + q];
                n1c[q] = XN[l0 + q];
            }
            if constexpr (PRE) {
#pragma unroll
                for (int i = 0; i < W; ++i) aw[i] = xa[i];
            }
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const double b = band_add<NS, EX>(whu[q], p.wi[LMEP_ROW_P1HALF], n1w, q);
                const double n2 = nlp<EX>(NLK, b, 0.0);
                XT2[l0 + q] = sub2(n2, nlp<EX>(NLK, n0c[q], 0.0));
                XS[l0 + q] = padd<EX>(n1c[q], n2);
            }
        }
        __syncthreads();
        if (act) {                                        // C: c = Wh a + P1h t2, n3 = N(c)
            double tw[W], wa[P];
            const double *xt = XT2 + (l0 - eL);
            if constexpr (!PRE) {
                const double *xa = XA + (l0 - eL);
#pragma unroll
                for (int i = 0; i < W; ++i) aw[i] = xa[i];
            }
#pragma unroll
            for (int i = 0; i < W; ++i) tw[i] = xt[i];
#pragma unroll
            for (int q = 0; q < P; ++q) wa[q] = band_reg<NS, EX>(p.wi[LMEP_ROW_WHALF], aw, q);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const double c = band_add<NS, EX>(wa[q], p.wi[LMEP_ROW_P1HALF], tw, q);
                XN[l0 + q] = nlp<EX>(NLK, c, 0.0);        // n1's slot: n1 was last read in B
            }
        }
        __syncthreads();
        if (act) {                                        // D: u' in place of u
            double sw[W], gw[W], bs[P];
            const double *xs = XS + (l0 - eL), *xg = XN + (l0 - eL);
#pragma unroll
            for (int i = 0; i < W; ++i) sw[i] = xs[i];
#pragma unroll
            for (int i = 0; i < W; ++i) gw[i] = xg[i];
#pragma unroll
            for (int q = 0; q < P; ++q) bs[q] = band_add<NS, EX>(t01[q], p.wi[LMEP_ROW_BETA], sw, q);
#pragma unroll
            for (int q = 0; q < P; ++q)
                XU[l0 + q] = band_add<NS, EX>(bs[q], p.wi[LMEP_ROW_GAMMA], gw, q);
        }
        __syncthreads();
    }
    bool bad = false;
    for (int64_t i = O0 + threadIdx.x; i < O1; i += blockDim.x) {
        const double v = XU[i - base];
        store_out(p, i - p.off, v);
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

template <int NS, int P, bool EX>
__device__ __forceinline__ void etdrk4_regs_convective(const StepParams &p, double *sm, const int slen,
                                                       const int len, const int K, const int64_t O0,
                                                       const int64_t O1, const int64_t base)
{
    constexpr int W = P + NS - 1;
    constexpr int NLK = LMEP_NL_CONVECTIVE;
    const int eL = p.eL;
    // slots: u | n0, later c | a, later b | n1, later n3 | t2 | s12
    double *XU = sm, *XN0 = sm + slen, *XA = sm + 2 * slen, *XN1 = sm + 3 * slen;
    double *XT2 = sm + 4 * slen, *XS = sm + 5 * slen;
    double *XC = XN0, *XB = XA, *XN3 = XN1;
    const int l0 = eL + (int)threadIdx.x * P;
    const bool act = l0 < len;
    auto sub2 = [](double n2, double n0) { return EX ? xsub(xmul(2.0, n2), n0) : 2.0 * n2 - n0; };
    auto load = [&](double (&w)[W], const double *X) {
        const double *x = X + (l0 - eL);
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] = x[i];
    };
    for (int s = 0; s < K; ++s) {
        double whu[P], t01[P], wha[P];
        if (act) {                                        // 0: n0 = -u D1 u; Wh u and W u off the same window
            double uw[W];
            load(uw, XU);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const double n0 = nlp<EX>(NLK, XU[l0 + q], band_reg<NS, EX>(p.wi[LMEP_ROW_D1], uw, q));
                whu[q] = band_reg<NS, EX>(p.wi[LMEP_ROW_WHALF], uw, q);
                t01[q] = band_reg<NS, EX>(p.wi[LMEP_ROW_W], uw, q);
                XN0[l0 + q] = n0;
                if (s == 0 && p.nl0_out) {
                    const int64_t g = base + l0 + q;
                    if (g >= O0 && g < O1) p.nl0_out[g - p.off] = n0;
                }
            }
        }
        __syncthreads();
        if (act) {                                        // A: a = whu + P1h n0; t01 = W u + alpha n0
            double nw[W];
            load(nw, XN0);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                XA[l0 + q] = band_add<NS, EX>(whu[q], p.wi[LMEP_ROW_P1HALF], nw, q);
                t01[q] = band_add<NS, EX>(t01[q], p.wi[LMEP_ROW_ALPHA], nw, q);
            }
        }
        __syncthreads();
        if (act) {                                        // A': n1 = -a D1 a; Wh a kept for c
            double aw[W];
            load(aw, XA);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                XN1[l0 + q] = nlp<EX>(NLK, XA[l0 + q], band_reg<NS, EX>(p.wi[LMEP_ROW_D1], aw, q));
                wha[q] = band_reg<NS, EX>(p.wi[LMEP_ROW_WHALF], aw, q);
            }
        }
        __syncthreads();
        if (act) {                                        // B: b = whu + P1h n1 (a's slot: a was last read in A')
            double nw[W];
            load(nw, XN1);
#pragma unroll
            for (int q = 0; q < P; ++q)
                XB[l0 + q] = band_add<NS, EX>(whu[q], p.wi[LMEP_ROW_P1HALF], nw, q);
        }
        __syncthreads();
        if (act) {                                        // B': n2 = -b D1 b; t2 = 2 n2 - n0; s12 = n1 + n2
            double bw[W];
            load(bw, XB);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const double n2 = nlp<EX>(NLK, XB[l0 + q], band_reg<NS, EX>(p.wi[LMEP_ROW_D1], bw, q));
                XT2[l0 + q] = sub2(n2, XN0[l0 + q]);
                XS[l0 + q] = padd<EX>(XN1[l0 + q], n2);
            }
        }
        __syncthreads();
        if (act) {                                        // C: c = Wh a + P1h t2 (n0's slot: n0 was last read in B')
            double tw[W];
            load(tw, XT2);
#pragma unroll
            for (int q = 0; q < P; ++q)
                XC[l0 + q] = band_add<NS, EX>(wha[q], p.wi[LMEP_ROW_P1HALF], tw, q);
        }
        __syncthreads();
        if (act) {                                        // C': n3 = -c D1 c (n1's slot)
            double cw[W];
            load(cw, XC);
#pragma unroll
            for (int q = 0; q < P; ++q)
                XN3[l0 + q] = nlp<EX>(NLK, XC[l0 + q], band_reg<NS, EX>(p.wi[LMEP_ROW_D1], cw, q));
        }
        __syncthreads();
        if (act) {                                        // D: u' in place of u
            double sw[W], gw[W];
            load(sw, XS);
            load(gw, XN3);
#pragma unroll
            for (int q = 0; q < P; ++q)
                XU[l0 + q] = band_add<NS, EX>(band_add<NS, EX>(t01[q], p.wi[LMEP_ROW_BETA], sw, q),
                                              p.wi[LMEP_ROW_GAMMA], gw, q);
        }
        __syncthreads();
    }
    bool bad = false;
    for (int64_t i = O0 + threadIdx.x; i < O1; i += blockDim.x) {
        const double v = XU[i - base];
        store_out(p, i - p.off, v);
        bad |= !isfinite(v);
    }
    if (bad) *p.flag = 1;
}

}  // namespace lmep
