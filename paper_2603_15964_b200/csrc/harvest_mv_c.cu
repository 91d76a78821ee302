// harvest_mv_c.cu -- instantiations of harvest_mv.cuh for d = 13..16 (split for parallel builds).
#include "harvest_mv.cuh"

namespace lmep {

int launch_harvest_mv_c(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 13: return launch_mv<13>(P, st);
    case 14: return launch_mv<14>(P, st);
    case 15: return launch_mv<15>(P, st);
    case 16: return launch_mv<16>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
