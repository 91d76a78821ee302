// harvest_mvb_b.cu -- instantiations of harvest_mvb.cuh for d = 11..13 (split for parallel builds).
#include "harvest_mvb.cuh"

namespace lmep {

int launch_harvest_mvb_b(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 11: return launch_mvb<11>(P, st);
    case 12: return launch_mvb<12>(P, st);
    case 13: return launch_mvb<13>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
