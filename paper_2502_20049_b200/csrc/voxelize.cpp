// voxelize.cpp — one-time voxelisation of a closed triangle mesh into the super-sampled binary
// geometry field (arXiv 2502.20049 §III: "voxelizing the geometry onto the
// geometry field once as a pre-processing step"), plus the brick packing the GPU lookup uses.
//
// Inside test (reading A15, exact, no floating point after snapping): vertices are
// snapped to the fixed-point grid 2^-(s+12) relative to the field origin o_G (integer, mesh bbox
// - 2 cells, A17); the centre of geometry cell g is g*4096 + 2048 per axis.  A +x ray from each
// centre counts the triangles whose (y,z) projection contains it (2D edge functions, top-left
// tie rule on the counter-clockwise projection) and whose crossing lies strictly at x > x0 (exact
// int128 comparison).  Odd count = inside.  Implementation: triangles are binned by the z rows
// of their projected bounding box; each row of samples receives one prefix toggle per crossing
// (the crossing position is converted to the first sample index it does not cover), followed by
// a suffix XOR — O(rows touched + samples) instead of O(samples x triangles).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "psm_host.h"
#include "psm_device.cuh"

namespace psm {

typedef __int128 i128;

static inline bool tl_inside(int64_t ay, int64_t az, int64_t by, int64_t bz, int64_t py,
                             int64_t pz) {
  const i128 e = (i128)(by - ay) * (i128)(pz - az) - (i128)(bz - az) * (i128)(py - ay);
  if (e != 0) return e > 0;
  const int64_t dy = by - ay, dz = bz - az;
  return (dz == 0 && dy < 0) || dz < 0;  // top or left edge owns its boundary points
}

static inline i128 ceil_div(i128 a, i128 b) {  // b > 0
  if (a >= 0) return (a + b - 1) / b;
  return -((-a) / b);
}

int check_mesh(const double* verts, int64_t nv, const int32_t* tris, int64_t nt,
               std::string* why) {
  if (nv < 4 || nt < 4) {
    *why = "mesh needs at least 4 vertices and 4 triangles";
    return -1;
  }
  for (int64_t k = 0; k < 3 * nv; ++k)
    if (!std::isfinite(verts[k])) {
      *why = "non-finite vertex coordinate";
      return -1;
    }
  std::unordered_map<uint64_t, int> edges;
  edges.reserve((size_t)(3 * nt));
  for (int64_t t = 0; t < nt; ++t)
    for (int e = 0; e < 3; ++e) {
      const int64_t a = tris[3 * t + e], b = tris[3 * t + (e + 1) % 3];
      if (a < 0 || a >= nv || b < 0 || b >= nv) {
        *why = "triangle " + std::to_string(t) + " has a vertex index out of range";
        return -1;
      }
      const uint64_t lo = (uint64_t)std::min(a, b), hi = (uint64_t)std::max(a, b);
      edges[(lo << 32) | hi] += 1;
    }
  for (const auto& kv : edges)
    if (kv.second != 2) {
      *why = "mesh is not watertight: edge (" + std::to_string(kv.first >> 32) + "," +
             std::to_string(kv.first & 0xFFFFFFFFu) + ") is shared by " +
             std::to_string(kv.second) + " triangles";
      return -1;
    }
  return 0;
}

void geometry_extent(const double* verts, int64_t nv, int s, double origin[3],
                     int64_t dims_cells[3]) {
  for (int a = 0; a < 3; ++a) {
    double lo = verts[a], hi = verts[a];
    for (int64_t k = 1; k < nv; ++k) {
      lo = std::min(lo, verts[3 * k + a]);
      hi = std::max(hi, verts[3 * k + a]);
    }
    origin[a] = std::floor(lo) - 2.0;
    dims_cells[a] = (int64_t)(std::ceil(hi) + 2.0 - origin[a]);
  }
  (void)s;
}

// bits: one byte per geometry cell, [gz][gy][gx], dims = dims_cells << s
void voxelize_mesh(const double* verts, int64_t nv, const int32_t* tris, int64_t nt, int s,
                   const double origin[3], const int64_t dims_cells[3],
                   std::vector<uint8_t>& bits) {
  const int64_t NX = dims_cells[0] << s, NY = dims_cells[1] << s, NZ = dims_cells[2] << s;
  bits.assign((size_t)(NX * NY * NZ), 0);
  std::vector<int64_t> V((size_t)(3 * nv));
  const double sc = std::ldexp(1.0, s + 12);
  for (int64_t k = 0; k < nv; ++k)
    for (int a = 0; a < 3; ++a) V[3 * k + a] = std::llround((verts[3 * k + a] - origin[a]) * sc);

  // bin triangles by the z rows their projection can touch
  std::vector<std::vector<int64_t>> zbin((size_t)NZ);
  auto row_range = [](int64_t lo, int64_t hi, int64_t n, int64_t& r0, int64_t& r1) {
    // rows g with lo <= g*4096 + 2048 <= hi
    r0 = std::max<int64_t>(0, (int64_t)ceil_div((i128)lo - 2048, 4096));
    i128 t = (i128)hi - 2048;
    int64_t f = (int64_t)(t >= 0 ? t / 4096 : -((-t + 4095) / 4096));
    r1 = std::min<int64_t>(n - 1, f);
  };
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t* A = &V[3 * (int64_t)tris[3 * t]];
    const int64_t* B = &V[3 * (int64_t)tris[3 * t + 1]];
    const int64_t* C = &V[3 * (int64_t)tris[3 * t + 2]];
    int64_t z0, z1;
    row_range(std::min({A[2], B[2], C[2]}), std::max({A[2], B[2], C[2]}), NZ, z0, z1);
    for (int64_t gz = z0; gz <= z1; ++gz) zbin[(size_t)gz].push_back(t);
  }

#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t gz = 0; gz < NZ; ++gz) {
    const int64_t Z0 = gz * 4096 + 2048;
    std::vector<uint8_t> tog((size_t)((NX + 1) * NY), 0);
    bool any = false;
    for (int64_t t : zbin[(size_t)gz]) {
      const int64_t* A = &V[3 * (int64_t)tris[3 * t]];
      const int64_t* B = &V[3 * (int64_t)tris[3 * t + 1]];
      const int64_t* C = &V[3 * (int64_t)tris[3 * t + 2]];
      const i128 area = (i128)(B[1] - A[1]) * (i128)(C[2] - A[2]) -
                        (i128)(B[2] - A[2]) * (i128)(C[1] - A[1]);
      if (area == 0) continue;  // projection degenerate: the ray never enters it
      const int64_t *P0 = A, *P1 = (area > 0) ? B : C, *P2 = (area > 0) ? C : B;
      // plane normal of the ORIGINAL orientation; sign handled below
      const i128 e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
      const i128 e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
      const i128 n0 = e1[1] * e2[2] - e1[2] * e2[1];
      const i128 n1 = e1[2] * e2[0] - e1[0] * e2[2];
      const i128 n2 = e1[0] * e2[1] - e1[1] * e2[0];
      int64_t y0, y1;
      row_range(std::min({A[1], B[1], C[1]}), std::max({A[1], B[1], C[1]}), NY, y0, y1);
      for (int64_t gy = y0; gy <= y1; ++gy) {
        const int64_t Y0 = gy * 4096 + 2048;
        if (!tl_inside(P0[1], P0[2], P1[1], P1[2], Y0, Z0)) continue;
        if (!tl_inside(P1[1], P1[2], P2[1], P2[2], Y0, Z0)) continue;
        if (!tl_inside(P2[1], P2[2], P0[1], P0[2], Y0, Z0)) continue;
        // crossing counts for sample X0 iff M*X0 < Nn (strictly right of the sample)
        const i128 K = n1 * (i128)(A[1] - Y0) + n2 * (i128)(A[2] - Z0);
        const i128 Nraw = n0 * (i128)A[0] + K;
        const i128 M = n0 > 0 ? n0 : -n0;
        const i128 Nn = n0 > 0 ? Nraw : -Nraw;
        // samples gx < (Nn - 2048 M) / (4096 M) are covered
        i128 kmax = ceil_div(Nn - 2048 * M, 4096 * M);
        if (kmax <= 0) continue;
        if (kmax > NX) kmax = NX;
        tog[(size_t)(gy * (NX + 1) + (int64_t)kmax)] ^= 1;
        any = true;
      }
    }
    if (!any) continue;
    uint8_t* dst = &bits[(size_t)(gz * NY * NX)];
    for (int64_t gy = 0; gy < NY; ++gy) {
      uint8_t acc = 0;
      const uint8_t* tg = &tog[(size_t)(gy * (NX + 1))];
      for (int64_t gx = NX - 1; gx >= 0; --gx) {
        acc ^= tg[gx + 1];
        dst[gy * NX + gx] = acc;
      }
    }
  }
}

// Pack into LBM-cell bricks of (2^s)^3 bits (linear bit index (brick << 3s) + bit, so bricks
// share uint64 words at s = 0, 1) and build the
// per-brick flags the remap kernel's exact early-outs use (cells beyond the field count as
// all-outside):
//   bit0: the brick and its 26 neighbours are all-outside   (one cell's sub-samples)
//   bit1: the brick and its 26 neighbours are all-inside
//   bit2: every brick within Chebyshev distance kTileReach is all-outside (a whole tile)
//   bit3: every brick within Chebyshev distance kTileReach is all-inside
//   bit4/bit5: the same within kSubReach (an 8x4x2 sub-tile)
//   bit6/bit7: the same within 2 (one cell's sub-samples after a pose change of up to one cell:
//              the remap's cached narrow band)
static void box_or(std::vector<uint8_t>& v, int64_t bx, int64_t by, int64_t bz, int r) {
  // in place: v := OR of v over the L-infinity ball of radius r (separable running counts);
  // cells beyond the grid contribute 0
  std::vector<uint8_t> tmp(v.size());
  auto pass = [&](int64_t n, int64_t stride, int64_t lines, auto line_base) {
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < lines; ++l) {
      const int64_t b0 = line_base(l);
      int cnt = 0;
      for (int64_t i = 0; i < std::min<int64_t>(n, r); ++i) cnt += v[(size_t)(b0 + i * stride)];
      for (int64_t i = 0; i < n; ++i) {
        if (i + r < n) cnt += v[(size_t)(b0 + (i + r) * stride)];
        if (i - r - 1 >= 0) cnt -= v[(size_t)(b0 + (i - r - 1) * stride)];
        tmp[(size_t)(b0 + i * stride)] = cnt > 0;
      }
    }
    v.swap(tmp);
  };
  pass(bx, 1, by * bz, [&](int64_t l) { return l * bx; });
  pass(by, bx, bx * bz, [&](int64_t l) { return (l / bx) * bx * by + (l % bx); });
  pass(bz, bx * by, bx * by, [&](int64_t l) { return l; });
}

void pack_bricks(const std::vector<uint8_t>& bits, int s, const int64_t dims_cells[3],
                 std::vector<unsigned long long>& words, std::vector<uint8_t>& mask,
                 int* total_words) {
  const int n = 1 << s;
  const int64_t bx = dims_cells[0], by = dims_cells[1], bz = dims_cells[2];
  const int64_t NX = bx << s, NY = by << s;
  const int64_t nb = bx * by * bz;
  // linear bit index (b << 3s) + bit: bricks share words at s = 0, 1
  const int64_t W = ((nb << (3 * s)) + 63) / 64;
  *total_words = (int)W;
  words.assign((size_t)W, 0ull);
  std::vector<uint8_t> any_in((size_t)nb, 0), any_out((size_t)nb, 0);
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t ix = b % bx, iy = (b / bx) % by, iz = b / (bx * by);
    int ones = 0;
    for (int sz = 0; sz < n; ++sz)
      for (int sy = 0; sy < n; ++sy)
        for (int sx = 0; sx < n; ++sx) {
          const int64_t g = ((iz * n + sz) * NY + (iy * n + sy)) * NX + (ix * n + sx);
          if (bits[(size_t)g]) {
            const int bit = (sz * n + sy) * n + sx;
            const int64_t gb = (b << (3 * s)) + bit;
#pragma omp atomic
            words[(size_t)(gb >> 6)] |= 1ull << (gb & 63);
            ++ones;
          }
        }
    any_in[(size_t)b] = ones > 0;
    any_out[(size_t)b] = ones < n * n * n;
  }
  // "beyond the field" is outside: any_out must be 1 there, which box_or cannot see, so the
  // all-inside flags additionally require the whole ball to lie inside the field
  std::vector<uint8_t> in1 = any_in, out1 = any_out, inK = any_in, outK = any_out;
  std::vector<uint8_t> inS = any_in, outS = any_out, in2 = any_in, out2 = any_out;
  box_or(in2, bx, by, bz, 2);
  box_or(out2, bx, by, bz, 2);
  box_or(in1, bx, by, bz, 1);
  box_or(out1, bx, by, bz, 1);
  box_or(inK, bx, by, bz, kTileReach);
  box_or(outK, bx, by, bz, kTileReach);
  box_or(inS, bx, by, bz, kSubReach);
  box_or(outS, bx, by, bz, kSubReach);
  mask.assign((size_t)nb, 0);
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t ix = b % bx, iy = (b / bx) % by, iz = b / (bx * by);
    auto inside_field = [&](int r) {
      return ix - r >= 0 && iy - r >= 0 && iz - r >= 0 && ix + r < bx && iy + r < by &&
             iz + r < bz;
    };
    uint8_t m = 0;
    if (!in1[(size_t)b]) m |= 1;
    if (!out1[(size_t)b] && inside_field(1)) m |= 2;
    if (!inK[(size_t)b]) m |= 4;
    if (!outK[(size_t)b] && inside_field(kTileReach)) m |= 8;
    if (!inS[(size_t)b]) m |= 16;
    if (!outS[(size_t)b] && inside_field(kSubReach)) m |= 32;
    if (!in2[(size_t)b]) m |= 64;
    if (!out2[(size_t)b] && inside_field(2)) m |= 128;
    mask[(size_t)b] = m;
  }
}

}  // namespace psm
