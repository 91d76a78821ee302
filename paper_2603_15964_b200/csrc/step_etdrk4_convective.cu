// step_etdrk4_convective.cu -- instantiations of the etdrk4 step kernel, N(u) kind convective.
#include "step.cuh"

namespace lmep {

int launch_scheme_etdrk4_convective(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    if (exact) return launch_ns<SCH_ETDRK4, true, STEP_P_ETDRK4_CV, LMEP_NL_CONVECTIVE>(p.n, p, grid, shm, st);
    return launch_ns<SCH_ETDRK4, false, STEP_P_ETDRK4_CV, LMEP_NL_CONVECTIVE>(p.n, p, grid, shm, st);
}

}  // namespace lmep
