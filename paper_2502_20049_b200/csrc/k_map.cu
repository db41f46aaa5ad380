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

namespace psm {

__device__ __forceinline__ void body_frame(const BodyGeo& b, const double p[3], const double L[3],
                                           const int wall[3], double q[3]) {
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = min_image(__dsub_rn(p[a], b.t[a]), L[a], !wall[a]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    q[a] = __fma_rn(b.Q[6 + a], d[2], __fma_rn(b.Q[3 + a], d[1], __dmul_rn(b.Q[a], d[0])));
}

__device__ __forceinline__ int mesh_bit(const BodyGeo& b, const double q[3]) {
  const double hs = ldexp(1.0, b.s);
  int g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = floor(__dmul_rn(__dsub_rn(q[a], b.o[a]), hs));
    if (!(x >= 0.0) || x >= (double)(b.dims_b[a] << b.s)) return 0;
    g[a] = (int)x;
  }
  const int n = 1 << b.s, msk = n - 1;
  const long long brick =
      ((long long)(g[2] >> b.s) * b.dims_b[1] + (g[1] >> b.s)) * b.dims_b[0] + (g[0] >> b.s);
  const int bit = (((g[2] & msk) * n) + (g[1] & msk)) * n + (g[0] & msk);
  const unsigned long long w = __ldg(b.bits + brick * b.words + (bit >> 6));
  return (int)((w >> (bit & 63)) & 1ull);
}

// number of inside sub-samples of cell (x, y, zg) for body b
__device__ int count_inside(const BodyGeo& b, int x, int y, int zg, const double L[3],
                            const int wall[3]) {
  const int n = 1 << b.s;
  const int full = n * n * n;
  const double h = ldexp(1.0, -b.s);
  // exact early-out from the cell centre
  {
    const double pc[3] = {x + 0.5, y + 0.5, zg + 0.5};
    double qc[3];
    body_frame(b, pc, L, wall, qc);
    if (b.kind == 0) {
      const double dist = sqrt(qc[0] * qc[0] + qc[1] * qc[1] + qc[2] * qc[2]);
      const double r = sqrt(b.r2);
      const double reach = 0.8660254037844387 + 1e-6;  // >= max |sample - centre|
      if (dist + reach < r) return full;
      if (dist - reach > r) return 0;
    } else {
      int bc[3];
      bool outside = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double xb = floor(qc[a] - b.o[a]);
        if (xb < -1.0 || xb > (double)b.dims_b[a]) outside = true;
        bc[a] = (int)fmax(-2.0, fmin(xb, (double)b.dims_b[a] + 1.0));
      }
      if (outside) return 0;
      if (bc[0] >= 0 && bc[1] >= 0 && bc[2] >= 0 && bc[0] < b.dims_b[0] &&
          bc[1] < b.dims_b[1] && bc[2] < b.dims_b[2]) {
        const uint8_t m =
            __ldg(b.mask + ((long long)bc[2] * b.dims_b[1] + bc[1]) * b.dims_b[0] + bc[0]);
        if (m == 1) return full;
        if (m == 2) return 0;
      }
    }
  }
  int cnt = 0;
  for (int gz = 0; gz < n; ++gz)
    for (int gy = 0; gy < n; ++gy)
      for (int gx = 0; gx < n; ++gx) {
        const double p[3] = {(double)x + (gx + 0.5) * h, (double)y + (gy + 0.5) * h,
                             (double)zg + (gz + 0.5) * h};
        double q[3];
        body_frame(b, p, L, wall, q);
        if (b.kind == 0) {
          const double d2 = __fma_rn(q[2], q[2], __fma_rn(q[1], q[1], __dmul_rn(q[0], q[0])));
          cnt += (d2 <= b.r2);
        } else {
          cnt += mesh_bit(b, q);
        }
      }
  return cnt;
}

__global__ void __launch_bounds__(kTileCells) k_map(const __grid_constant__ MapParams p) {
  const Geom& G = p.g;
  int k = 0;
  while (k + 1 < p.nbox && p.box[k + 1].first <= (int)blockIdx.x) ++k;
  const MapBox& bx = p.box[k];
  const int li = blockIdx.x - bx.first;
  const int tx = bx.t0[0] + li % bx.n[0];
  const int ty = bx.t0[1] + (li / bx.n[0]) % bx.n[1];
  const int tz = bx.t0[2] + li / (bx.n[0] * bx.n[1]);
  const int x = tx * kTileX + threadIdx.x;
  const int y = ty * kTileY + threadIdx.y;
  const int z = tz * kTileZ + threadIdx.z;
  const bool act = x < G.nx && y < G.ny && z < G.nzl;
  uint32_t word = 0;
  if (act) {
    const int zg = G.z0 + z;
    const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
    const double xc[3] = {x + 0.5, y + 0.5, zg + 0.5};
    int best = 0, bestcnt = 0;
    double beste = 0.0;
    for (int id = 1; id <= kMaxBodies; ++id) {
      const BodyGeo& b = p.bodies[id];
      if (!b.present) continue;
      bool in = true;
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (fabs(min_image(xc[a] - b.t[a], L[a], !G.wall[a])) > b.rb1) in = false;
      if (!in) continue;
      const int cnt = count_inside(b, x, y, zg, L, G.wall);
      const double e = ldexp((double)cnt, -3 * b.s);
      if (cnt > 0 && e > beste) {
        best = id;
        bestcnt = cnt;
        beste = e;
      }
    }
    if (best) word = (uint32_t)bestcnt | ((uint32_t)best << 16);
    p.word[((long long)z * G.ny + y) * G.nx + x] = word;
  }
  const int any = __syncthreads_or(word != 0);
  if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0)
    p.tile_flag[(tz * G.gy + ty) * G.gx + tx] = (uint8_t)(any ? 1 : 0);
}

cudaError_t launch_map(const MapParams& p, cudaStream_t st) {
  if (p.ntiles <= 0) return cudaSuccess;
  k_map<<<p.ntiles, dim3(kTileX, kTileY, kTileZ), 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace psm
