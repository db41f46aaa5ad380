// psm_device.cuh — device-side definitions of the B200 PSM hot path (arXiv 2502.20049).
//
// Stencils, storage layout and kernel parameter blocks shared by the .cu files of the product
// library.  Nothing here is shared with oracle/ (which has its own tables and arithmetic).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace psm {

constexpr int kMaxBodies = 16;   // PSM_MAX_BODIES
constexpr int kTileX = 32;       // one warp along x (coalesced SoA rows)
constexpr int kTileY = 4;
constexpr int kTileZ = 2;
constexpr int kTileCells = kTileX * kTileY * kTileZ;  // 256 threads = one collide/map block
constexpr int kMaxBoxes = 1;     // remap boxes per launch (one launch per box)
// Chebyshev reach (in LBM cells) of a tile's sub-samples from the tile centre, plus one:
// half-diagonal of a 32x4x2 tile = sqrt(16^2 + 2^2 + 1^2) = 16.16 -> brick offset <= 17
constexpr int kTileReach = 18;
// second level: 8x4x2 sub-tiles (half-diagonal sqrt(4^2 + 2^2 + 1^2) = 4.58 -> offset <= 5)
constexpr int kSubX = 8;
constexpr int kSubReach = 6;
constexpr int kSlotVals = 12;    // F/T partial: m[3], (x_c-R) x m [3], |m| [3], |(x_c-R) x m| [3]

// ------------------------------------------------------------------------------ stencils ----
// Direction order of DESIGN.md §2.1 (lbmpy/waLBerla convention; PAPER.md:233 names the sets).
__host__ __device__ constexpr int stc_x(int i) {
  constexpr int t[27] = {0, 0, 0, -1, 1, 0, 0, -1, 1, -1, 1, 0, 0, -1, 1, 0, 0, -1, 1,
                         1, -1, 1, -1, 1, -1, 1, -1};
  return t[i];
}
__host__ __device__ constexpr int stc_y(int i) {
  constexpr int t[27] = {0, 1, -1, 0, 0, 0, 0, 1, 1, -1, -1, 1, -1, 0, 0, 1, -1, 0, 0,
                         1, 1, -1, -1, 1, 1, -1, -1};
  return t[i];
}
__host__ __device__ constexpr int stc_z(int i) {
  constexpr int t[27] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, 1, 1, 1, -1, -1, -1, -1,
                         1, 1, 1, 1, -1, -1, -1, -1};
  return t[i];
}
// opposite direction index (c_opp = -c)
__host__ __device__ constexpr int stc_opp(int i) {
  constexpr int t[27] = {0, 2, 1, 4, 3, 6, 5, 10, 9, 8, 7, 16, 15, 18, 17, 12, 11, 14, 13,
                         26, 25, 24, 23, 22, 21, 20, 19};
  return t[i];
}
// weights: D3Q19 1/3, 1/18, 1/36; D3Q27 8/27, 2/27, 1/54, 1/216
template <int Q>
__host__ __device__ constexpr double stc_w(int i) {
  int n = (stc_x(i) != 0) + (stc_y(i) != 0) + (stc_z(i) != 0);
  if (Q == 19) return n == 0 ? 1.0 / 3.0 : (n == 1 ? 1.0 / 18.0 : 1.0 / 36.0);
  return n == 0 ? 8.0 / 27.0 : (n == 1 ? 2.0 / 27.0 : (n == 2 ? 1.0 / 54.0 : 1.0 / 216.0));
}

// ------------------------------------------------------------------------- body tables -----
// What the collide kernel needs per body: rigid velocity u_s = v + w x mi(x_c - t) and the
// fraction weighting (s, tau-weighted or direct).
struct BodyKin {
  double t[3], v[3], w[3];
  int s;        // super-sampling exponent (eps = cnt * 2^-3s)
  int present;
};

// What the mapping kernel needs per body.
struct BodyGeo {
  double Q[9];      // body -> world, row major; sample maps to q = Q^T mi(p - t)
  double t[3];
  double lo1[3];    // body-frame AABB - 1: a cell whose centre maps outside [lo1, hi1] has
  double hi1[3];    // every sub-sample outside the body (samples lie within sqrt(3)/2)
  double r2;        // sphere: r*r
  double o[3];      // mesh: geometry-field origin (body frame, integer valued)
  int dims_b[3];    // mesh: field extent in bricks (LBM cells)
  int kind;         // 0 sphere, 1 mesh
  int s;
  int words;        // uint64 words of the whole field
  int present;
  int mapping;      // 0 R1 (per sub-sample), 1 R2 (centre-only block average), meshes only
  int pad_;
  // geometry bits packed linearly: bit (brick << 3s) + ((gz&m)*n + (gy&m))*n + (gx&m) of the
  // uint64 array (a brick = the (2^s)^3 geometry cells of one LBM cell; at s = 0, 1 several
  // bricks share a word instead of one word per brick, so the field stays cache-sized)
  const unsigned long long* bits;
  const uint8_t* mask;             // [brick] flag bits, see pack_bricks (voxelize.cpp)
};

// ---------------------------------------------------------------------- launch params -----
// unsigned division by a run-time constant d >= 1: n / d = (umulhi(n, m) + n) >> l for every
// 32-bit n (Granlund-Montgomery round-up multiplier, 33-bit sum in 64 bits); replaces the ~20
// instruction integer division in the remap's list decoding
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
  return FastDiv{d, (uint32_t)m, l};
}
#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t fast_div(uint32_t n, const FastDiv& f) {
  return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.l);
}
#endif

struct Geom {
  int nx, ny, nzl;        // local extents
  int nz_global;
  int z0;                 // global z of local plane 0
  int zghost;             // 1: ghost planes at local z = -1 and nzl (world > 1)
  int wall[3];            // 1 = not periodic: half-way bounce-back wall on this axis
  int open_x;             // x faces are inflow (x = 0) / outflow (x = nx-1), reading A30
  long long qstride;      // elements between consecutive direction planes
  int gx, gy, gz;         // tile grid
};

struct CollideParams {
  Geom g;
  const void* src;        // two-array: read array;   AA: the single array
  void* dst;              // two-array: write array;  AA: same as src
  const uint32_t* word;   // solid word per local cell: cnt | id << 16 (0 = fluid)
  const uint8_t* tile_flag;
  double* partial;        // [tile][2 slots][1 + kSlotVals] (slot id stored as double)
  double* overflow;       // [kMaxBodies+1][kSlotVals] atomics for a 3rd+ body in a tile
  unsigned long long* err;  // first (step, cell) with rho <= 0 or non-finite
  int hiocc;              // host: launch the higher-occupancy instantiation (fp64 D3Q19)
  const double* dbg_B;    // DBG: B [cell]
  const double* dbg_us;   // DBG: u_s [3][cell]
  const uint8_t* dbg_id;  // DBG: id [cell]
  double tau, omega;      // omega = 1/tau (symmetric rate w+)
  double omega_m;         // antisymmetric rate w- (TRT; == omega for SRT)
  int trt;                // fluid operator: 0 SRT (Eq.(2)), 1 TRT, 2 cumulant (D3Q27)
  double gforce[3];       // test-only Guo force
  double u_in[3];         // A30 inflow velocity (g.open_x)
  double rho_out;         // A30 outflow density (g.open_x)
  int sc;                 // 1, 2, 3
  int bmode;              // 0 direct, 1 weighted
  long long step;         // for the error word
  int tz0;                // first tile layer (z) of this launch: blockIdx.z + tz0
  BodyKin bodies[kMaxBodies + 1];
  // per-direction plane bases src + q * qstride and dst + q * qstride (filled by the launcher):
  // each access is then one 32-bit-offset LEA off a constant-bank pointer instead of a 64-bit
  // q * qstride + offset product per load/store
  const void* srcq[27];
  void* dstq[27];
  // fused halo (world > 1, peer memory over NVLink): plane bases of the neighbours' ghost planes
  // in THEIR destination array, per direction (c_z = +1: upper neighbour's plane below its slab;
  // c_z = -1: lower neighbour's plane above its slab); null where there is no such neighbour
  int p2p;
  void* gup[27];
  void* gdn[27];
};

struct MapBox {
  int t0[3];          // first tile (local tile coords)
  int n[3];           // tiles per axis
  int first;          // prefix sum of tiles before this box
  uint32_t bodymask;  // bit id: body id's current box overlaps this box
};

struct MapParams {
  Geom g;
  uint32_t* word;
  uint8_t* tile_flag;
  unsigned long long* stats;  // optional diagnostics (PSM_MAP_STATS): tiles by decision, cells
                              // by decision, sub-samples evaluated
  int nbox;
  int ntiles;
  MapBox box[kMaxBoxes];
  BodyGeo bodies[kMaxBodies + 1];
};

// single-body narrow-band remap (k_remap.cu)
struct RemapParams {
  Geom g;
  MapBox box;
  BodyGeo body;
  int id;
  uint32_t* word;
  uint8_t* tile_flag;
  int* counters;        // [0] tiles, [1] segments, [2] band cells
  int* tiles;           // listed tiles
  uint32_t* segs;       // listed segments: tile << 5 | segment
  float4* segq;         // body-frame segment centres
  uint32_t* band;       // narrow-band cells: tile << 8 | cell-in-tile
  int* bandcnt;         // their inside counts (s >= 2 chunked path)
  int* bandn;           // number of band cells (counters + 2, or a cached band's count)
  int seg_cap, band_cap;
  int margin;           // 1: decisions valid for any pose within one cell (cached band)
  FastDiv fgx, fgxy;    // division by g.gx and g.gx * g.gy (tile index -> tile coordinates)
  int fused12;          // L1 and L2 in one warp-cooperative launch (k_remap_l12)
};

#if defined(__CUDACC__)
// minimum image on a periodic axis (same tie rule as the method definition)
__device__ __forceinline__ double min_image(double d, double L, bool periodic) {
  if (!periodic) return d;
  if (d >= 0.5 * L)
    d = __dsub_rn(d, L);
  else if (d < -0.5 * L)
    d = __dadd_rn(d, L);
  return d;
}
#endif

}  // namespace psm
