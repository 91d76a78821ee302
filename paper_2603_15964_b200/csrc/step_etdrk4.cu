// step_etdrk4.cu -- instantiations of the etdrk4 step kernel.
#include "step.cuh"

namespace lmep {

int launch_scheme_etdrk4(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (exact) return launch_ns<SCH_ETDRK4, true, 5>(p.n, p, grid, shm, st);
    return launch_ns<SCH_ETDRK4, false, 5>(p.n, p, grid, shm, st);
}

}  // namespace lmep
