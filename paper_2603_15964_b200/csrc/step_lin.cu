// step_lin.cu -- instantiations of the linear step kernel.
#include "step.cuh"

namespace lmep {

int launch_scheme_lin(bool pernode, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (pernode) return launch_ns<SCH_LIN, true, 1, LMEP_NL_NONE, true>(p.n, p, grid, shm, st);
    return launch_ns<SCH_LIN, true, 5, LMEP_NL_NONE>(p.n, p, grid, shm, st);
}

}  // namespace lmep
