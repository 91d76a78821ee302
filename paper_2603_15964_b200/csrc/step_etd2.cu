// step_etd2.cu -- instantiations of the etd2 step kernel.
#include "step.cuh"

namespace lmep {

int launch_scheme_etd2(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (exact) return launch_ns<SCH_ETD2, true, 5>(p.n, p, grid, shm, st);
    return launch_ns<SCH_ETD2, false, 5>(p.n, p, grid, shm, st);
}

}  // namespace lmep
