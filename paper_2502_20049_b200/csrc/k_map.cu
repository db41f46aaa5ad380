// k_map.cu — per-step fraction remap of moving rigid bodies (arXiv 2502.20049 §III,
// PAPER.md:310-321) for sm_100a.
//
// For every cell of the launched tiles (the swept bounding boxes of the bodies that moved) and
// every body whose conservative box contains it: eps_b = (#sub-samples inside) / 2^(3s), with
// the 2^(3s) sub-cell centres p of the world-fixed LBM cell mapped into the body frame,
// q = Q^T mi(p - t) (reading R1, A12; explicit fma order A14, so the integer count is
// bit-exact with the method definition).  Inside test: sphere q.q <= r^2; mesh: bit of the
// super-sampled geometry field (voxelised once) at floor((q - o) 2^s).
// The body with the largest eps wins (ties: lower id).  Output: one 32-bit word per cell,
// cnt | id << 16, and one "any solid" flag per tile, which gates the PSM path of the collide
// kernel.  Early-outs (exact): a sphere cell whose centre is farther than
// sqrt(3)/2 + margin from the surface is decided without sampling; a mesh cell whose centre
// lands in a geometry brick flagged "dilated all-in/all-out" is decided by that flag (every
// sub-sample lies within one brick of the centre's brick).
#include "psm_device.cuh"
#include "psm_internal.h"
#include "psm_map_common.cuh"

namespace psm {

// Remap of one 32x4x2 tile per block; grid = the box's tiles (blockIdx = tile offset in the box).
// Each warp owns one 32-cell x-row and decides it without block barriers: (1) lanes 0..3 decide
// the row's four 8-cell segments (fp64, reach kSubReach bricks) and broadcast them by shuffles,
// (2) per cell in fp32 (dilated-by-one brick flags), (3) the narrow-band cells' sub-samples are
// packed across the 32 lanes (lane -> (cell, sample)) and counted with ballots — exact fp64 per
// sample (A14).
__global__ void __launch_bounds__(kTileCells, 6) k_map(const __grid_constant__ MapParams p) {
  const Geom& G = p.g;
  const int tid = threadIdx.x + kTileX * (threadIdx.y + kTileY * threadIdx.z);
  const int lane = threadIdx.x;
  const MapBox& bx = p.box[0];
  const int tx = bx.t0[0] + (int)blockIdx.x;
  const int ty = bx.t0[1] + (int)blockIdx.y;
  const int tz = bx.t0[2] + (int)blockIdx.z;
  // The tile flag says whether any word of this tile is nonzero now; if it is 0, writing a
  // zero word is redundant, so warps far from every body store nothing.
  const int flag_old = p.tile_flag[(tz * G.gy + ty) * G.gx + tx];
  const int x = tx * kTileX + lane;
  const int y = ty * kTileY + threadIdx.y;
  const int z = tz * kTileZ + threadIdx.z;
  const bool row_ok = y < G.ny && z < G.nzl;
  const bool act = row_ok && x < G.nx;
  const int zg = G.z0 + z;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  int best = 0, bestcnt = 0;
  double beste = 0.0;
  for (uint32_t msk = bx.bodymask; msk; msk &= msk - 1) {  // warp-uniform loop
    const int id = __ffs(msk) - 1;
    const BodyGeo& b = p.bodies[id];
    const int s = b.s;
    // (1) segment decisions: lane k < 4 evaluates segment k of this row
    // (segments clamped to the grid; sd = 3: the segment straddles a periodic seam, so its
    // cells transform their own centres)
    int sd = 0;
    float q0 = 0.f, q1 = 0.f, q2 = 0.f;
    const int sx0 = tx * kTileX + lane * kSubX;
    if (lane < kTileX / kSubX && row_ok && sx0 < G.nx) {
      const int sx1 = min(sx0 + kSubX, G.nx);
      const double ps[3] = {0.5 * (sx0 + sx1), y + 0.5, zg + 0.5};
      const double half[3] = {0.5 * (sx1 - sx0), 0.5, 0.5};
      double qs[3];
      sd = tile_decision<kSubReach, 16, 32>(b, ps, half, L, G.wall, qs);
      if (p.stats) atomicAdd(p.stats + sd, 1ull);
      if (sd == 2 && region_straddles(b, ps, half, L, G.wall, 0)) sd = 3;
      q0 = (float)qs[0];
      q1 = (float)qs[1];
      q2 = (float)qs[2];
    }
    const int seg = lane / kSubX;
    const int sdec = __shfl_sync(0xFFFFFFFFu, sd, seg);
    // (2) per-cell fp32 decision from the segment-centre transform
    int cd = sdec;
    const unsigned need = __ballot_sync(0xFFFFFFFFu, sdec >= 2);
    if (need) {
      const float qs0 = __shfl_sync(0xFFFFFFFFu, q0, seg);
      const float qs1 = __shfl_sync(0xFFFFFFFFu, q1, seg);
      const float qs2 = __shfl_sync(0xFFFFFFFFu, q2, seg);
      if (sdec == 2) {
        const int s0 = tx * kTileX + seg * kSubX;
        const float off = (float)x + 0.5f - 0.5f * (float)(s0 + min(s0 + kSubX, G.nx));
        const float qc[3] = {qs0 + (float)b.Q[0] * off, qs1 + (float)b.Q[1] * off,
                             qs2 + (float)b.Q[2] * off};
        cd = cell_decision(b, qc);
      } else if (sdec == 3) {
        cd = act ? cell_decision_own(b, x, y, zg, L, G.wall) : 0;
      }
    }
    if (!act) cd = 0;
    int cnt = (cd == 1) ? (1 << (3 * s)) : 0;
    // (3) narrow band: pack (cell, sample) pairs of the warp's band cells over the lanes
    if (b.mapping == 1 && cd == 2) {  // R2: one centre-only block count per band cell
      cnt = r2_count(b, x, y, zg, L, G.wall);
      cd = 3;
    }
    const unsigned band = __ballot_sync(0xFFFFFFFFu, cd == 2);
    if (band) {
      const int ls = 3 * s;
      const int nsamp = 1 << ls;
      const int nband = __popc(band);
      const int items = nband << ls;
      for (int base = 0; base < items; base += 32) {
        const int it = base + lane;
        int c = -1;
        if (it < items) {
          c = (int)__fns(band, 0, (it >> ls) + 1);  // (it >> ls)-th set bit of `band`
        }
        const int inside =
            (c >= 0) ? sample_inside(b, tx * kTileX + c, y, zg, it & (nsamp - 1), L, G.wall)
                     : 0;
        const unsigned vote = __ballot_sync(0xFFFFFFFFu, inside);
        // lanes carrying samples of MY cell: it in [base, base + 32) with (it >> ls) == my rank
        if (cd == 2) {
          const int rank = __popc(band & ((1u << lane) - 1));
          const int first = (rank << ls) - base, last = first + nsamp;  // lane range
          const int l0 = max(first, 0), l1 = min(last, 32);
          if (l1 > l0) {
            const unsigned sel = (l1 - l0 == 32) ? 0xFFFFFFFFu
                                                 : (((1u << (l1 - l0)) - 1u) << l0);
            cnt += __popc(vote & sel);
          }
        }
      }
    }
    if (p.stats && act) atomicAdd(p.stats + 3 + (cd == 3 ? 2 : cd), 1ull);
    const double e = ldexp((double)cnt, -3 * s);
    if (cnt > 0 && e > beste) {
      best = id;
      bestcnt = cnt;
      beste = e;
    }
  }
  uint32_t word = 0;
  if (best) word = (uint32_t)bestcnt | ((uint32_t)best << 16);
  if (act && (word != 0 || flag_old != 0)) p.word[((long long)z * G.ny + y) * G.nx + x] = word;
  const int any = __syncthreads_or(word != 0);
  if (tid == 0) p.tile_flag[(tz * G.gy + ty) * G.gx + tx] = (uint8_t)(any ? 1 : 0);
}

cudaError_t launch_map(const MapParams& p, cudaStream_t st) {
  // one launch per box: blockIdx is the tile offset inside box[0]
  if (p.nbox != 1) return cudaErrorInvalidValue;
  const MapBox& b = p.box[0];
  if (b.n[0] <= 0 || b.n[1] <= 0 || b.n[2] <= 0) return cudaSuccess;
  k_map<<<dim3(b.n[0], b.n[1], b.n[2]), dim3(kTileX, kTileY, kTileZ), 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace psm
