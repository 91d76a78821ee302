// harvest_mvb_a.cu -- instantiations of harvest_mvb.cuh for d = 5..10 (split for parallel builds).
#include "harvest_mvb.cuh"

namespace lmep {

int launch_harvest_mvb_a(const HarvestParams &P, cudaStream_t st)
{
    switch (P.d) {
    case 5: return launch_mvb<5>(P, st);
    case 6: return launch_mvb<6>(P, st);
    case 7: return launch_mvb<7>(P, st);
    case 8: return launch_mvb<8>(P, st);
    case 9: return launch_mvb<9>(P, st);
    case 10: return launch_mvb<10>(P, st);
    default: return LMEP_DIMENSION;
    }
}

}  // namespace lmep
