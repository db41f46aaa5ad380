// k_collide_19d.cu — D3Q19 double instantiations of the fused PSM stream-collide (k_collide.cuh)
#include "k_collide.cuh"

namespace psm {

cudaError_t launch_collide_19d(const CollideParams& p, int pat, bool force, bool dbg, int ntz,
                               cudaStream_t st) {
  return launch_t<19, double>(p, pat, force, dbg, ntz, st);
}

}  // namespace psm
