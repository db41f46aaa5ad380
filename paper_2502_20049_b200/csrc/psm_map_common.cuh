// psm_map_common.cuh — device helpers of the fraction remap (k_map.cu, k_remap.cu):
// body-frame transform with the A14 fma order, geometry-field bit lookup, exact sub-sample test,
// and the conservative region decisions (tile / segment / cell) built on the brick flags.
#pragma once
#include "psm_device.cuh"

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

// word index and bit of sub-sample `si` of cell (x, y, zg) in a mesh body's geometry field
// (wi = -1: outside the field, i.e. outside the body); same arithmetic as sample_inside
__device__ __forceinline__ void mesh_word_index(const BodyGeo& b, int x, int y, int zg, int si,
                                                const double L[3], const int wall[3],
                                                long long& wi, int& bitpos) {
  const int n = 1 << b.s;
  const double h = ldexp(1.0, -b.s);
  const int gx = si & (n - 1), gy = (si >> b.s) & (n - 1), gz = si >> (2 * b.s);
  const double p[3] = {(double)x + (gx + 0.5) * h, (double)y + (gy + 0.5) * h,
                       (double)zg + (gz + 0.5) * h};
  double q[3];
  body_frame(b, p, L, wall, q);
  const double hs = ldexp(1.0, b.s);
  int g[3];
  wi = -1;
  bitpos = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double xx = floor(__dmul_rn(__dsub_rn(q[a], b.o[a]), hs));
    if (!(xx >= 0.0) || xx >= (double)(b.dims_b[a] << b.s)) return;
    g[a] = (int)xx;
  }
  const int msk = n - 1;
  const long long brick =
      ((long long)(g[2] >> b.s) * b.dims_b[1] + (g[1] >> b.s)) * b.dims_b[0] + (g[0] >> b.s);
  const int bit = (((g[2] & msk) * n) + (g[1] & msk)) * n + (g[0] & msk);
  const long long gb = (brick << (3 * b.s)) + bit;  // linear bit index (psm_device.cuh)
  wi = gb >> 6;
  bitpos = (int)(gb & 63);
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
  const long long gb = (brick << (3 * b.s)) + ((((g[2] & msk) * n) + (g[1] & msk)) * n +
                                                (g[0] & msk));
  return (int)((__ldg(b.bits + (gb >> 6)) >> (gb & 63)) & 1ull);
}

// geometry bit g (in field range) of a mesh body
__device__ __forceinline__ int field_bit(const BodyGeo& b, int gx, int gy, int gz) {
  const int n = 1 << b.s, msk = n - 1;
  const long long brick =
      ((long long)(gz >> b.s) * b.dims_b[1] + (gy >> b.s)) * b.dims_b[0] + (gx >> b.s);
  const long long gb = (brick << (3 * b.s)) + ((((gz & msk) * n) + (gy & msk)) * n + (gx & msk));
  return (int)((__ldg(b.bits + (gb >> 6)) >> (gb & 63)) & 1ull);
}

// R2 (paper-literal): only the cell centre is transformed (A14 arithmetic); the
// count is the number of set geometry cells in the 2^s-cube block whose lower corner is
// g0 = floor((q_c - o) 2^s - 2^(s-1) + 1/2); cells beyond the field count 0.
static __device__ __noinline__ int r2_count(const BodyGeo& b, int x, int y, int zg, const double L[3],
                                     const int wall[3]) {
  const double pc[3] = {x + 0.5, y + 0.5, zg + 0.5};
  double q[3];
  body_frame(b, pc, L, wall, q);
  const int n = 1 << b.s;
  const double hs = ldexp(1.0, b.s), half = ldexp(1.0, b.s - 1);
  long long g0[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    g0[a] = (long long)floor(__dadd_rn(__dsub_rn(__dmul_rn(__dsub_rn(q[a], b.o[a]), hs), half),
                                       0.5));
  int cnt = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const long long gx = g0[0] + i, gy = g0[1] + j, gz = g0[2] + k;
        if (gx < 0 || gy < 0 || gz < 0 || gx >= ((long long)b.dims_b[0] << b.s) ||
            gy >= ((long long)b.dims_b[1] << b.s) || gz >= ((long long)b.dims_b[2] << b.s))
          continue;
        cnt += field_bit(b, (int)gx, (int)gy, (int)gz);
      }
  return cnt;
}

// exact inside test of sub-sample `si` (0 .. 8^s - 1) of cell (x, y, zg) for body b (reading R1,
// A14 arithmetic: dyadic sample point, q = Q^T mi(p - t) with the fixed fma order)
__device__ __forceinline__ int sample_inside(const BodyGeo& b, int x, int y, int zg, int si,
                                             const double L[3], const int wall[3]) {
  const int n = 1 << b.s;
  const double h = ldexp(1.0, -b.s);
  const int gx = si & (n - 1), gy = (si >> b.s) & (n - 1), gz = si >> (2 * b.s);
  const double p[3] = {(double)x + (gx + 0.5) * h, (double)y + (gy + 0.5) * h,
                       (double)zg + (gz + 0.5) * h};
  double q[3];
  body_frame(b, p, L, wall, q);
  if (b.kind == 0) {
    const double d2 = __fma_rn(q[2], q[2], __fma_rn(q[1], q[1], __dmul_rn(q[0], q[0])));
    return d2 <= b.r2;
  }
  return mesh_bit(b, q);
}

// Periodic seam guard.  A region (tile, segment or cell) is the box pc +- half (clamped to the
// grid, so a ragged last tile is described by the cells it really holds).  On a periodic axis the
// method maps each sample with its own minimum image (mi(p - t), A14), so a region whose
// displacement range reaches the cut at +-L/2 holds samples of two different images and its
// centre transform says nothing about them.  Such a region is never decided as a whole; with
// margin = 1 (cached band) the range is widened by the one cell the body may still move.
__device__ __forceinline__ bool region_straddles(const BodyGeo& b, const double pc[3],
                                                 const double half[3], const double L[3],
                                                 const int wall[3], int margin) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (wall[a]) continue;
    const double d = min_image(pc[a] - b.t[a], L[a], true);
    if (fabs(d) + half[a] + (double)margin >= 0.5 * L[a] - 1e-6) return true;
  }
  return false;
}

// Whole-region decision: 0 = every sub-sample of the region is outside, 1 = every sub-sample is
// inside, 2 = decide per cell.  pt = centre of the region clamped to the grid, half = its half
// extents; every sub-sample lies within REACH - 1 bricks of the centre's brick (REACH is sized
// for the unclamped region, which contains the clamped one).  qt = body-frame region centre
// (used as the base of the per-cell fp32 decisions).  Regions straddling a periodic seam are
// always 2 (region_straddles).
// margin = 1: valid for poses within one cell of this one (the brick reaches keep >= 1.84 cells
// of slack for meshes; the sphere test widens by the margin).
template <int REACH, int BIT_OUT, int BIT_IN>
__device__ __forceinline__ int tile_decision(const BodyGeo& b, const double pt[3],
                                             const double half[3], const double L[3],
                                             const int wall[3], double qt[3], int margin = 0) {
  constexpr int kTileReach = REACH;  // brick reach of the region's sub-samples + 1
  body_frame(b, pt, L, wall, qt);
  if (region_straddles(b, pt, half, L, wall, margin)) return 2;
  if (b.kind != 1) {
    const double dist = sqrt(qt[0] * qt[0] + qt[1] * qt[1] + qt[2] * qt[2]);
    const double r = sqrt(b.r2);
    if (dist - (double)(kTileReach - 1 + margin) > r) return 0;
    if (dist + (double)(kTileReach - 1 + margin) < r) return 1;
    return 2;
  }
  int bc[3];
  bool in_field = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double xb = floor(qt[a] - b.o[a]);
    if (xb < -(double)kTileReach || xb > (double)(b.dims_b[a] - 1 + kTileReach)) return 0;
    if (xb < 0.0 || xb > (double)(b.dims_b[a] - 1)) in_field = false;
    bc[a] = (int)xb;
  }
  if (!in_field) return 2;
  const uint8_t m =
      __ldg(b.mask + ((long long)bc[2] * b.dims_b[1] + bc[1]) * b.dims_b[0] + bc[0]);
  if (m & BIT_OUT) return 0;
  if (m & BIT_IN) return 1;
  return 2;
}

// Conservative per-cell decision in fp32 from the tile-centre transform (error << 0.1 cell):
// 0 outside, 1 inside, 2 needs exact sampling.  Sub-samples lie within sqrt(3)/2 of the centre.
// margin = 1: the decision must also hold after the body moves by up to one cell (every body
// point displaced by < 1): radius-2 brick flags, bounding box and reach widened by one — the
// cached narrow band of the remap.
__device__ __forceinline__ int cell_decision(const BodyGeo& b, const float qc[3],
                                             int margin = 0) {
  constexpr float kEps = 0.01f;  // >> fp32 error of qc
  const float M = (float)margin;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (qc[a] < (float)b.lo1[a] - M - kEps || qc[a] > (float)b.hi1[a] + M + kEps) return 0;
  if (b.kind == 0) {
    const float dist = sqrtf(qc[0] * qc[0] + qc[1] * qc[1] + qc[2] * qc[2]);
    const float r = sqrtf((float)b.r2);
    const float reach = 0.8660254f + M + kEps;
    if (dist + reach < r) return 1;
    if (dist - reach > r) return 0;
    return 2;
  }
  int bc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float xb = floorf(qc[a] - (float)b.o[a]);
    // every sample (plus the margin) beyond the field
    if (xb < -1.0f - M || xb > (float)b.dims_b[a] + M) return 0;
    bc[a] = (int)xb;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (bc[a] < 0 || bc[a] >= b.dims_b[a]) return 2;
  const uint8_t m =
      __ldg(b.mask + ((long long)bc[2] * b.dims_b[1] + bc[1]) * b.dims_b[0] + bc[0]);
  if (m & (margin ? 128 : 2)) return 1;
  if (m & (margin ? 64 : 1)) return 0;
  return 2;
}

// Per-cell decision of a cell of a region that straddles a periodic seam: the cell's own centre
// is transformed exactly (its own minimum image); a cell that itself straddles the cut is sampled.
__device__ __forceinline__ int cell_decision_own(const BodyGeo& b, int x, int y, int zg,
                                                 const double L[3], const int wall[3],
                                                 int margin = 0) {
  const double pc[3] = {x + 0.5, y + 0.5, zg + 0.5};
  const double half[3] = {0.5, 0.5, 0.5};
  if (region_straddles(b, pc, half, L, wall, margin)) return 2;
  double q[3];
  body_frame(b, pc, L, wall, q);
  const float qc[3] = {(float)q[0], (float)q[1], (float)q[2]};
  return cell_decision(b, qc, margin);
}

// Warp-centric remap of one 32x4x2 tile per block: each warp owns one 32-cell x-row and decides
// it without block barriers: (1) per 8-cell segment (reach kSubReach bricks), (2) per cell in
// fp32 (dilated-by-one brick flags), (3) the narrow-band cells' sub-samples packed across the 32
// lanes (lane -> (cell, sample) pairs) and counted with ballots — exact fp64 per sample.
// exact count of a cell for body b (R1: all sub-samples; R2: the centre block)
__device__ __forceinline__ int exact_count(const BodyGeo& b, int x, int y, int zg,
                                           const double L[3], const int wall[3]) {
  if (b.mapping == 1) return r2_count(b, x, y, zg, L, wall);
  int cnt = 0;
  for (int si = 0; si < (1 << (3 * b.s)); ++si) cnt += sample_inside(b, x, y, zg, si, L, wall);
  return cnt;
}

// Inside count of 8 consecutive sub-samples (si0 .. si0+7, same cell, si0 % 8 == 0) of a mesh
// body.  Sample si0 is transformed with the exact A14 arithmetic; the others by adding the
// rotated sub-sample offsets (error ~1e-13 cells).  A sample whose scaled coordinate lies within
// 1e-9 of a geometry-cell face is recomputed exactly, so every floor() equals the exact one and
// the count is bit-identical to mesh_word_index() per sample.  Each sample's geometry word is
// loaded as soon as its index is known, U samples in flight: few live registers, so more warps
// hide the load latency (measured faster than eight batched 64-bit indices).
#ifndef PSM_REMAP_U
#define PSM_REMAP_U 1
#endif
constexpr int kRemapU = PSM_REMAP_U;
__device__ __forceinline__ int mesh_count8(const BodyGeo& b, int x, int y, int zg, int si0,
                                           const double L[3], const int wall[3]) {
  const int n = 1 << b.s, msk = n - 1;
  const double h = ldexp(1.0, -b.s), hs = ldexp(1.0, b.s);
  const int gx0 = si0 & msk, gy0 = (si0 >> b.s) & msk, gz0 = si0 >> (2 * b.s);
  const double p0[3] = {(double)x + (gx0 + 0.5) * h, (double)y + (gy0 + 0.5) * h,
                        (double)zg + (gz0 + 0.5) * h};
  double q0[3];
  body_frame(b, p0, L, wall, q0);
  int cnt = 0;
#pragma unroll kRemapU
  for (int j = 0; j < 8; ++j) {
    const int si = si0 + j;
    const int gx = si & msk, gy = (si >> b.s) & msk, gz = si >> (2 * b.s);
    const double dx = (gx - gx0) * h, dy = (gy - gy0) * h, dz = (gz - gz0) * h;
    double f[3];
    bool safe = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double qa = q0[a] + (b.Q[a] * dx + b.Q[3 + a] * dy + b.Q[6 + a] * dz);
      f[a] = (qa - b.o[a]) * hs;
      const double fr = f[a] - floor(f[a]);
      if (fr < 1e-9 || fr > 1.0 - 1e-9) safe = false;
    }
    long long wi;
    int bit;
    if (!safe) {
      mesh_word_index(b, x, y, zg, si, L, wall, wi, bit);
    } else {
      int g[3];
      bool in = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double xx = floor(f[a]);
        if (!(xx >= 0.0) || xx >= (double)(b.dims_b[a] << b.s)) in = false;
        g[a] = (int)xx;
      }
      wi = -1;
      bit = 0;
      if (in) {
        const long long brick = ((long long)(g[2] >> b.s) * b.dims_b[1] + (g[1] >> b.s)) *
                                    b.dims_b[0] + (g[0] >> b.s);
        const long long gb = (brick << (3 * b.s)) + ((((g[2] & msk) * n) + (g[1] & msk)) * n +
                                                      (g[0] & msk));
        wi = gb >> 6;
        bit = (int)(gb & 63);
      }
    }
    if (wi >= 0) cnt += (int)((__ldg(b.bits + wi) >> bit) & 1ull);
  }
  return cnt;
}

}  // namespace psm
