// k_collide_19f.cu — D3Q19 float instantiations of the fused PSM stream-collide (k_collide.cuh)
#include "k_collide.cuh"

namespace psm {

cudaError_t launch_collide_19f(const CollideParams& p, int pat, bool force, bool dbg, int ntz,
                               cudaStream_t st) {
  return launch_t<19, float>(p, pat, force, dbg, ntz, st);
}

}  // namespace psm
