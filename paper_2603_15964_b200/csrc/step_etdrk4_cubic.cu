// step_etdrk4_cubic.cu -- instantiations of the etdrk4 step kernel, N(u) kind cubic.
#include "step.cuh"

namespace lmep {

int launch_scheme_etdrk4_cubic(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    // chunk size of the register-resident passes: step_p_etdrk4(nl, n)
    if (p.n == 7) {
        if (exact) return launch_ns<SCH_ETDRK4, true, STEP_P_ETDRK4, LMEP_NL_CUBIC>(p.n, p, grid, shm, st);
        return launch_ns<SCH_ETDRK4, false, STEP_P_ETDRK4, LMEP_NL_CUBIC>(p.n, p, grid, shm, st);
    }
    if (exact) return launch_ns<SCH_ETDRK4, true, STEP_P_ETDRK4_CV, LMEP_NL_CUBIC>(p.n, p, grid, shm, st);
    return launch_ns<SCH_ETDRK4, false, STEP_P_ETDRK4_CV, LMEP_NL_CUBIC>(p.n, p, grid, shm, st);
}

}  // namespace lmep
