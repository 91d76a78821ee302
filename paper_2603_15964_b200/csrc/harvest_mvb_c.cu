// harvest_mvb_c.cu -- instantiations of harvest_mvb.cuh for d = 14..16 (split for parallel builds).
#include "harvest_mvb.cuh"

namespace lmep {

int launch_harvest_mvb_c(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 14: return launch_mvb<14>(P, st);
    case 15: return launch_mvb<15>(P, st);
    case 16: return launch_mvb<16>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
