// harvest_mv_b.cu -- instantiations of harvest_mv.cuh for d = 9..12 (split for parallel builds).
#include "harvest_mv.cuh"

namespace lmep {

int launch_harvest_mv_b(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 9: return launch_mv<9>(P, st);
    case 10: return launch_mv<10>(P, st);
    case 11: return launch_mv<11>(P, st);
    case 12: return launch_mv<12>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
