// k_collide_27f.cu — D3Q27 float instantiations of the fused PSM stream-collide (k_collide.cuh)
#include "k_collide.cuh"

namespace psm {

cudaError_t launch_collide_27f(const CollideParams& p, int pat, bool force, bool dbg, int ntz,
                               cudaStream_t st) {
  return launch_t<27, float>(p, pat, force, dbg, ntz, st);
}

}  // namespace psm
