// step_etd2_convective.cu -- instantiations of the etd2 step kernel, N(u) kind convective.
#include "step.cuh"

namespace lmep {

int launch_scheme_etd2_convective(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (exact) return launch_ns<SCH_ETD2, true, STEP_P_ETD2, LMEP_NL_CONVECTIVE>(p.n, p, grid, shm, st);
    return launch_ns<SCH_ETD2, false, STEP_P_ETD2, LMEP_NL_CONVECTIVE>(p.n, p, grid, shm, st);
}

}  // namespace lmep
