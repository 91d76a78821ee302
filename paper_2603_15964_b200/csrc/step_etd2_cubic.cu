// step_etd2_cubic.cu -- instantiations of the etd2 step kernel, N(u) kind cubic.
#include "step.cuh"

namespace lmep {

int launch_scheme_etd2_cubic(bool exact, const StepParams &p, dim3 grid, size_t shm, cudaStream_t st)
{
    // exponential multistep order p.etds (1..5); order 2 has n-specialised kernels
#define ETDS_CASE(S_)                                                                             \
    case S_:                                                                                      \
        return exact ? launch_ns<SCH_ETD2, true, STEP_P_ETD2, LMEP_NL_CUBIC, false, S_>(p.n, p, grid, shm, st) \
                     : launch_ns<SCH_ETD2, false, STEP_P_ETD2, LMEP_NL_CUBIC, false, S_>(p.n, p, grid, shm, st);
    switch (p.etds) {
        ETDS_CASE(1)
        ETDS_CASE(2)
        ETDS_CASE(3)
        ETDS_CASE(4)
        ETDS_CASE(5)
    default: return LMEP_INVALID_CONFIG;
    }
#undef ETDS_CASE
}

}  // namespace lmep
