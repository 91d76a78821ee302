// step_lin.cu -- instantiations of the linear step kernel.
#include "step.cuh"

namespace lmep {

int launch_scheme_lin(bool pernode, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (pernode) return launch_ns<SCH_LIN, true, 1, LMEP_NL_NONE, true>(p.n, p, grid, shm, st);
    return launch_ns<SCH_LIN, true, 5, LMEP_NL_NONE>(p.n, p, grid, shm, st);
}

}  // namespace lmep

namespace lmep {

// Per-node linear step without boundary closure (BASELINE config 5): a lean
// streaming kernel.  Each thread produces PPT outputs spaced blockDim apart
// (coalesced SoA weight loads, all PPT*n loads of a thread issued before the
// accumulations); u is read straight from global memory, where neighbouring
// threads' windows overlap in L1.  Arithmetic is the EXACT ascending order of
// kernels.py:23-29, so it is bit-identical to the generic engine.
template <int NS, int PPT>
__global__ void __launch_bounds__(256) lin_pernode_kernel(const __grid_constant__ StepParams p)
{
    const int n = NS > 0 ? NS : p.n;
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * PPT + threadIdx.x;
    const bool single = p.hl == nullptr && p.hr == nullptr;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int64_t li = base + (int64_t)k * blockDim.x;
        if (li >= p.nloc) break;
        const int64_t g = p.off + li;
        int64_t st = g - p.row;
        if (!p.periodic) st = st < 0 ? 0 : (st > p.N - n ? p.N - n : st);
        const double *w = p.wp + li;
        double acc = 0.0;
        if (single && p.periodic && st >= 0 && st + n <= p.N) {
            const double *u = p.u_in + st;
#pragma unroll
            for (int j = 0; j < (NS > 0 ? NS : 1); ++j) {
                if (NS == 0) break;
                acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.nloc), __ldg(u + j)));
            }
            if (NS == 0)
                for (int j = 0; j < n; ++j)
                    acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.nloc), __ldg(u + j)));
        } else {
            for (int j = 0; j < n; ++j)
                acc = xadd(acc, xmul(__ldcs(w + (int64_t)j * p.nloc),
                                     load_node(p, p.u_in, p.hl, p.hr, st + j)));
        }
        p.u_out[li] = acc;
        if (!isfinite(acc)) *p.flag = 1;
    }
}

int launch_lin_pernode(const StepParams &p, cudaStream_t st)
{
    constexpr int PPT = 4, TPB = 256;
    const int64_t blocks = (p.nloc + (int64_t)TPB * PPT - 1) / ((int64_t)TPB * PPT);
    if (p.n == 13) lin_pernode_kernel<13, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 7) lin_pernode_kernel<7, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 9) lin_pernode_kernel<9, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else if (p.n == 11) lin_pernode_kernel<11, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    else lin_pernode_kernel<0, PPT><<<(unsigned)blocks, TPB, 0, st>>>(p);
    return launch_status("lin_pernode_kernel");
}

}  // namespace lmep
