// harvest_mv_a.cu -- instantiations of harvest_mv.cuh for d = 2..8 (split for parallel builds).
#include "harvest_mv.cuh"

namespace lmep {

int launch_harvest_mv_a(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 2: return launch_mv<2>(P, st);
    case 3: return launch_mv<3>(P, st);
    case 4: return launch_mv<4>(P, st);
    case 5: return launch_mv<5>(P, st);
    case 6: return launch_mv<6>(P, st);
    case 7: return launch_mv<7>(P, st);
    case 8: return launch_mv<8>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
