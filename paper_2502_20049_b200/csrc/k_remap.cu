// k_remap.cu — narrow-band fraction remap for a box holding a single body (the common case:
// every moving body in its own bounding box), arXiv 2502.20049 §III.
//
// The count of a cell changes only near the body surface, so the work is organised as a flat
// pipeline of barrier-free kernels over compacted device lists, each level deciding exactly what
// it can and passing the rest on:
//   L0  one thread per tile of the box     : tile-centre test with reach kTileReach bricks
//   L1  one thread per 8-cell segment      : segment-centre test with reach kSubReach
//   L2  one thread per cell                : fp32 centre test against dilated-by-one bricks
//   L3  one thread per narrow-band cell    : exact fp64 inside test of each sub-sample
//                                            (reading R1, A14 order), count -> word
// Cached band (margin = 1): L0-L2 decide with one cell of slack (radius-2 brick flags, widened
// reaches), so their decisions hold for every pose within one cell of the build pose; until the
// body has moved that far, a step re-runs only L3 over the cached band list.
// Every early decision is conservative (it only claims "all sub-samples outside/inside" when the
// brick flags prove it), so the words equal the brute-force counts bit for bit.  Tile flags ("any word nonzero") are
// reset for every tile that reaches L1 and set by whichever level writes a nonzero word.
#include <cassert>

#include "psm_device.cuh"
#include "psm_internal.h"
#include "psm_map_common.cuh"

namespace psm {

namespace {

constexpr int kSegPerTile = (kTileX / kSubX) * kTileY * kTileZ;  // 32

__device__ __forceinline__ void tile_coords(int t, const RemapParams& r, int& tx, int& ty,
                                            int& tz) {
  const Geom& G = r.g;
  const uint32_t u = (uint32_t)t, q = fast_div(u, r.fgx), z = fast_div(u, r.fgxy);
  tx = (int)(u - q * (uint32_t)G.gx);
  ty = (int)(q - z * (uint32_t)G.gy);
  tz = (int)z;
}

// the cells a tile really holds (a ragged last tile is clamped to the grid): centre, half extents
__device__ __forceinline__ void region_of_tile(const Geom& G, int tx, int ty, int tz, double pc[3],
                                               double half[3]) {
  const int lo[3] = {tx * kTileX, ty * kTileY, tz * kTileZ};
  const int hi[3] = {min(lo[0] + kTileX, G.nx), min(lo[1] + kTileY, G.ny),
                     min(lo[2] + kTileZ, G.nzl)};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    pc[a] = 0.5 * (lo[a] + hi[a]);
    half[a] = 0.5 * (hi[a] - lo[a]);
  }
  pc[2] += G.z0;
}

__device__ __forceinline__ void put_word(const RemapParams& r, int x, int y, int z, uint32_t w,
                                         int tile) {
#if defined(PSM_BOUNDS_CHECK)
  assert(x >= 0 && x < r.g.nx && y >= 0 && y < r.g.ny && z >= 0 && z < r.g.nzl);
  assert(tile >= 0 && tile < r.g.gx * r.g.gy * r.g.gz);
#endif
  r.word[((long long)z * r.g.ny + y) * r.g.nx + x] = w;
  if (w) r.tile_flag[tile] = 1;
}

// L0: one thread per tile of the box
__global__ void k_remap_l0(const __grid_constant__ RemapParams r) {
  const MapBox& bx = r.box;
  const int ntile = bx.n[0] * bx.n[1] * bx.n[2];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntile) return;
  const int tx = bx.t0[0] + i % bx.n[0];
  const int ty = bx.t0[1] + (i / bx.n[0]) % bx.n[1];
  const int tz = bx.t0[2] + i / (bx.n[0] * bx.n[1]);
  const Geom& G = r.g;
  const int tile = (tz * G.gy + ty) * G.gx + tx;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  double pt[3], half[3];
  region_of_tile(G, tx, ty, tz, pt, half);
  double qt[3];
  const int dec = tile_decision<kTileReach, 4, 8>(r.body, pt, half, L, G.wall, qt, r.margin);
  if (dec == 0 && r.tile_flag[tile] == 0) return;  // far outside and already all zero
  r.tile_flag[tile] = 0;
  const int k = atomicAdd(r.counters + 0, 1);
  r.tiles[k] = tile;
}

// L1: one thread per segment of the listed tiles
__global__ void k_remap_l1(const __grid_constant__ RemapParams r) {
  const Geom& G = r.g;
  const int nseg = r.counters[0] * kSegPerTile;  // tiles list never overflows (<= box tiles)
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  const BodyGeo& b = r.body;
  const uint32_t full = ((uint32_t)1 << (3 * b.s)) | ((uint32_t)r.id << 16);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nseg; i += gridDim.x * blockDim.x) {
    const int tile = r.tiles[i / kSegPerTile];
    const int sg = i % kSegPerTile;
    int tx, ty, tz;
    tile_coords(tile, r, tx, ty, tz);
    const int sx = sg % (kTileX / kSubX), row = sg / (kTileX / kSubX);
    const int y = ty * kTileY + row % kTileY, z = tz * kTileZ + row / kTileY;
    if (y >= G.ny || z >= G.nzl) continue;
    const int x0 = tx * kTileX + sx * kSubX;
    if (x0 >= G.nx) continue;
    const int x1 = min(x0 + kSubX, G.nx);  // ragged last segment: clamped to the grid
    const double ps[3] = {0.5 * (x0 + x1), y + 0.5, G.z0 + z + 0.5};
    const double half[3] = {0.5 * (x1 - x0), 0.5, 0.5};
    double qs[3];
    const int dec = tile_decision<kSubReach, 16, 32>(b, ps, half, L, G.wall, qs, r.margin);
    if (dec == 2) {
      // straddling segments (seam): every cell transforms its own centre in L2 (segq.w = 1)
      const bool own = region_straddles(b, ps, half, L, G.wall, r.margin);
      const int k = atomicAdd(r.counters + 1, 1);
      if (k < r.seg_cap) {
        r.segs[k] = ((uint32_t)tile << 5) | (uint32_t)sg;
        r.segq[k] = make_float4((float)qs[0], (float)qs[1], (float)qs[2], own ? 1.f : 0.f);
        continue;
      }
      // list full: finish the segment here (exact, serial; a cached band gets its cells)
      for (int c = 0; c < x1 - x0; ++c) {
        const float off = (float)(x0 + c) + 0.5f - (float)ps[0];
        const float qc[3] = {(float)qs[0] + (float)b.Q[0] * off, (float)qs[1] + (float)b.Q[1] * off,
                             (float)qs[2] + (float)b.Q[2] * off};
        const int cd = own ? cell_decision_own(b, x0 + c, y, G.z0 + z, L, G.wall, r.margin)
                           : cell_decision(b, qc, r.margin);
        if (cd == 2 && r.margin) {  // the cached band holds every cell of the box: no overflow
          const int k = atomicAdd(r.bandn, 1);
          r.band[k] = ((uint32_t)tile << 8) | (uint32_t)(row * kTileX + sx * kSubX + c);
          r.bandcnt[k] = 0;
          continue;
        }
        int cnt = cd == 1 ? (1 << (3 * b.s)) : 0;
        if (cd == 2) cnt = exact_count(b, x0 + c, y, G.z0 + z, L, G.wall);
        put_word(r, x0 + c, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
      }
      continue;
    }
    const uint32_t w = dec == 1 ? full : 0u;
    for (int c = 0; c < kSubX; ++c)
      if (x0 + c < G.nx) put_word(r, x0 + c, y, z, w, tile);
  }
}

// L2: one thread per cell of the listed segments: fp32 centre test against the dilated-by-one
// brick flags; decided cells are written, narrow-band cells appended to the band list.
__global__ void k_remap_l2(const __grid_constant__ RemapParams r) {
  const Geom& G = r.g;
  const int ncell = min(r.counters[1], r.seg_cap) * kSubX;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  const BodyGeo& b = r.body;
  const uint32_t full = ((uint32_t)1 << (3 * b.s)) | ((uint32_t)r.id << 16);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncell; i += gridDim.x * blockDim.x) {
    const int si = i / kSubX, c = i % kSubX;
    const uint32_t sgw = r.segs[si];
    const int tile = (int)(sgw >> 5), sg = (int)(sgw & 31u);
    int tx, ty, tz;
    tile_coords(tile, r, tx, ty, tz);
    const int sx = sg % (kTileX / kSubX), row = sg / (kTileX / kSubX);
    const int y = ty * kTileY + row % kTileY, z = tz * kTileZ + row / kTileY;
    const int x = tx * kTileX + sx * kSubX + c;
    if (x >= G.nx) continue;
    const float4 q = r.segq[si];
    const int x0 = tx * kTileX + sx * kSubX;
    const float off = (float)x + 0.5f - 0.5f * (float)(x0 + min(x0 + kSubX, G.nx));
    const float qc[3] = {q.x + (float)b.Q[0] * off, q.y + (float)b.Q[1] * off,
                         q.z + (float)b.Q[2] * off};
    const int cd = q.w != 0.f ? cell_decision_own(b, x, y, G.z0 + z, L, G.wall, r.margin)
                              : cell_decision(b, qc, r.margin);
    if (cd == 2) {
      const int k = atomicAdd(r.bandn, 1);
      if (k < r.band_cap) {
        r.band[k] = ((uint32_t)tile << 8) | (uint32_t)(row * kTileX + sx * kSubX + c);
        r.bandcnt[k] = 0;
        continue;
      }
      const int cnt = exact_count(b, x, y, G.z0 + z, L, G.wall);  // list full: count here
      put_word(r, x, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
      continue;
    }
    put_word(r, x, y, z, cd == 1 ? full : 0u, tile);
  }
}

// L1 + L2 fused: one thread per segment takes the L1 decision; the warp then decides the cells
// of its undecided segments together, four segments (eight lanes each) per pass, instead of
// listing them for a separate L2 launch.  Same decisions and writes as k_remap_l1/k_remap_l2
// (whose segment list is bounded by seg_cap; here there is no segment list to overflow).
__global__ void k_remap_l12(const __grid_constant__ RemapParams r) {
  const Geom& G = r.g;
  const int nseg = r.counters[0] * kSegPerTile;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  const BodyGeo& b = r.body;
  const uint32_t full = ((uint32_t)1 << (3 * b.s)) | ((uint32_t)r.id << 16);
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * blockDim.x;
  // warp-uniform loop bound: the ballots and shuffles below need every lane
  for (int wb = blockIdx.x * blockDim.x + (threadIdx.x & ~31); wb < nseg; wb += stride) {
    const int i = wb + lane;
    bool und = false;
    int tile = 0, sg = 0, y = 0, z = 0, x0 = 0, x1 = 0;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < nseg) {
      tile = r.tiles[i / kSegPerTile];
      sg = i % kSegPerTile;
      int tx, ty, tz;
      tile_coords(tile, r, tx, ty, tz);
      const int sx = sg % (kTileX / kSubX), row = sg / (kTileX / kSubX);
      y = ty * kTileY + row % kTileY;
      z = tz * kTileZ + row / kTileY;
      x0 = tx * kTileX + sx * kSubX;
      if (y < G.ny && z < G.nzl && x0 < G.nx) {
        x1 = min(x0 + kSubX, G.nx);  // ragged last segment: clamped to the grid
        const double ps[3] = {0.5 * (x0 + x1), y + 0.5, G.z0 + z + 0.5};
        const double half[3] = {0.5 * (x1 - x0), 0.5, 0.5};
        double qs[3];
        const int dec = tile_decision<kSubReach, 16, 32>(b, ps, half, L, G.wall, qs, r.margin);
        if (dec == 2) {
          // straddling segments (seam): every cell transforms its own centre (q.w = 1)
          const bool own = region_straddles(b, ps, half, L, G.wall, r.margin);
          q = make_float4((float)qs[0], (float)qs[1], (float)qs[2], own ? 1.f : 0.f);
          und = true;
        } else {
          const uint32_t w = dec == 1 ? full : 0u;
          for (int c = 0; c < x1 - x0; ++c) put_word(r, x0 + c, y, z, w, tile);
        }
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, und);
    while (m) {
      const int slot = lane >> 3, c = lane & 7;
      unsigned mm = m;  // the (slot + 1)-th undecided segment of the warp
      for (int k = 0; k < slot && mm; ++k) mm &= mm - 1;
      const int src = mm ? __ffs(mm) - 1 : 0;
      const bool have = mm != 0u;
      const int t_ = __shfl_sync(0xffffffffu, tile, src);
      const int sg_ = __shfl_sync(0xffffffffu, sg, src);
      const int y_ = __shfl_sync(0xffffffffu, y, src);
      const int z_ = __shfl_sync(0xffffffffu, z, src);
      const int x0_ = __shfl_sync(0xffffffffu, x0, src);
      const int x1_ = __shfl_sync(0xffffffffu, x1, src);
      const float qx = __shfl_sync(0xffffffffu, q.x, src), qy = __shfl_sync(0xffffffffu, q.y, src);
      const float qz = __shfl_sync(0xffffffffu, q.z, src), qw = __shfl_sync(0xffffffffu, q.w, src);
      const int x = x0_ + c;
      if (have && x < x1_) {
        const float off = (float)x + 0.5f - 0.5f * (float)(x0_ + x1_);
        const float qc[3] = {qx + (float)b.Q[0] * off, qy + (float)b.Q[1] * off,
                             qz + (float)b.Q[2] * off};
        const int cd = qw != 0.f ? cell_decision_own(b, x, y_, G.z0 + z_, L, G.wall, r.margin)
                                 : cell_decision(b, qc, r.margin);
        if (cd == 2) {
          const int k = atomicAdd(r.bandn, 1);
          if (k < r.band_cap) {
            const int sx = sg_ % (kTileX / kSubX), row = sg_ / (kTileX / kSubX);
            r.band[k] = ((uint32_t)t_ << 8) | (uint32_t)(row * kTileX + sx * kSubX + c);
            r.bandcnt[k] = 0;
          } else {  // list full: count here
            const int cnt = exact_count(b, x, y_, G.z0 + z_, L, G.wall);
            put_word(r, x, y_, z_, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, t_);
          }
        } else {
          put_word(r, x, y_, z_, cd == 1 ? full : 0u, t_);
        }
      }
      for (int k = 0; k < 4 && m; ++k) m &= m - 1;  // the four segments just done
    }
  }
}

__device__ __forceinline__ void band_cell(const RemapParams& r, uint32_t e, int& x, int& y,
                                          int& z, int& tile) {
  tile = (int)(e >> 8);
  const int c = (int)(e & 255u);
  int tx, ty, tz;
  tile_coords(tile, r, tx, ty, tz);
  x = tx * kTileX + c % kTileX;
  y = ty * kTileY + (c / kTileX) % kTileY;
  z = tz * kTileZ + c / (kTileX * kTileY);
}

// L3: one thread per narrow-band cell: all its sub-samples with the exact fp64 test (A14),
// geometry-bit loads issued 8 at a time, and the word written directly.
// the exact sample kernels at four blocks per SM (64 registers, one sample load in flight per
// thread, more threads): measured faster than the 118-register batched-load form
#ifndef PSM_REMAP_MINB
#define PSM_REMAP_MINB 4
#endif
__global__ void __launch_bounds__(256, PSM_REMAP_MINB) k_remap_l3(const __grid_constant__ RemapParams r) {
  const Geom& G = r.g;
  const BodyGeo& b = r.body;
  const int n = min(*r.bandn, r.band_cap);
  const int nsamp = 1 << (3 * b.s);
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int x, y, z, tile;
    band_cell(r, r.band[k], x, y, z, tile);
    const int zg = G.z0 + z;
    int cnt = 0;
    if (b.mapping == 1) {  // R2: centre-only block count
      cnt = r2_count(b, x, y, zg, L, G.wall);
      put_word(r, x, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
      continue;
    }
    for (int s0 = 0; s0 < nsamp; s0 += 8) {
      const int m = min(8, nsamp - s0);
      if (b.kind == 0) {
        for (int j = 0; j < m; ++j) cnt += sample_inside(b, x, y, zg, s0 + j, L, G.wall);
        continue;
      }
      // mesh at s = 0 (s >= 1 meshes run k_remap_l3_mesh): the single sample
      for (int j = 0; j < m; ++j) {
        long long wi;
        int bit;
        mesh_word_index(b, x, y, zg, s0 + j, L, G.wall, wi, bit);
        if (wi >= 0) cnt += (int)((__ldg(b.bits + wi) >> bit) & 1ull);
      }
    }
    put_word(r, x, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
  }
}

// L3 for spheres at s >= 2 (64 or 512 sub-samples per cell): one thread per (band cell, 8-sample
// chunk), integer atomics into the cell's count (order-independent); L4
// writes the words.
__global__ void __launch_bounds__(256, PSM_REMAP_MINB) k_remap_l3_chunks(const __grid_constant__ RemapParams r) {
  const Geom& G = r.g;
  const BodyGeo& b = r.body;
  const int n = min(*r.bandn, r.band_cap);
  const int lch = 3 * b.s - 3;  // log2(chunks per cell)
  const long long items = (long long)n << lch;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(it >> lch), ch = (int)(it & ((1ll << lch) - 1));
    int x, y, z, tile;
    band_cell(r, r.band[k], x, y, z, tile);
    const int zg = G.z0 + z;
    int cnt = 0;
    for (int j = 0; j < 8; ++j) cnt += sample_inside(b, x, y, zg, ch * 8 + j, L, G.wall);
    if (cnt) atomicAdd(r.bandcnt + k, cnt);
  }
}

// L3 for mesh bodies with R1 at s = 1..3 (S compile-time): G lanes per band cell (8 at s >= 2,
// one 8-sample chunk each at s = 2, eight at s = 3; 1 at s = 1), mesh_count8_t per chunk, the
// lanes' counts summed with shuffles and the word written by the cell's first lane (no count
// atomics, no L4).  Warps iterate together (warp-uniform loop bound) so the full-mask shuffles
// are legal; items = cells * G with G | 32, so a cell's lanes are all active or all idle.
template <int S>
__global__ void __launch_bounds__(256, PSM_REMAP_MINB) k_remap_l3_mesh(const __grid_constant__ RemapParams r) {
  constexpr int kLanes = S >= 2 ? 8 : 1;
  constexpr int C = S >= 2 ? (1 << (3 * S - 3)) / kLanes : 1;  // 8-sample chunks per lane
  const Geom& G = r.g;
  const BodyGeo& b = r.body;
  const int n = min(*r.bandn, r.band_cap);
  const long long items = (long long)n * kLanes;
  const double L[3] = {(double)G.nx, (double)G.ny, (double)G.nz_global};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (long long wb = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); wb < items;
       wb += stride) {
    const long long it = wb + lane;
    const bool act = it < items;
    const int k = (int)(it / kLanes), ch = (int)(it % kLanes);
    int x = 0, y = 0, z = 0, tile = 0, cnt = 0;
    if (act) {
      band_cell(r, r.band[k], x, y, z, tile);
#pragma unroll 1
      for (int c = 0; c < C; ++c)
        cnt += mesh_count8_t<S>(b, x, y, G.z0 + z, (ch * C + c) * 8, L, G.wall);
    }
    if (kLanes > 1) {
#pragma unroll
      for (int o = 1; o < kLanes; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (act && ch == 0)
      put_word(r, x, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
  }
}

__global__ void k_remap_l4(const __grid_constant__ RemapParams r) {
  const int n = min(*r.bandn, r.band_cap);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    int x, y, z, tile;
    band_cell(r, r.band[k], x, y, z, tile);
    const int cnt = r.bandcnt[k];
    r.bandcnt[k] = 0;  // ready for the next pass over a cached band
    put_word(r, x, y, z, cnt ? ((uint32_t)cnt | ((uint32_t)r.id << 16)) : 0u, tile);
  }
}

// the exact (L3) stage for body r.body over the band list
void launch_l3(const RemapParams& r, int blocks, cudaStream_t st, int threads) {
  const BodyGeo& b = r.body;
  if (b.kind == 1 && b.mapping == 0 && b.s >= 1) {
    if (b.s == 1) k_remap_l3_mesh<1><<<blocks, threads, 0, st>>>(r);
    else if (b.s == 2) k_remap_l3_mesh<2><<<blocks, threads, 0, st>>>(r);
    else k_remap_l3_mesh<3><<<blocks, threads, 0, st>>>(r);
  } else if (b.s >= 2 && b.mapping == 0) {
    k_remap_l3_chunks<<<blocks, threads, 0, st>>>(r);
    k_remap_l4<<<blocks, threads, 0, st>>>(r);
  } else {
    k_remap_l3<<<blocks, threads, 0, st>>>(r);
  }
}

}  // namespace

int remap_l3_kernels(const BodyGeo& b) {
  return (b.kind != 1 && b.s >= 2 && b.mapping == 0) ? 2 : 1;
}

int remap_single_kernels(const RemapParams& r) {
  return (r.fused12 ? 2 : 3) + remap_l3_kernels(r.body);
}

// the exact pass alone over a cached band (poses within one cell of the band's build pose)
cudaError_t launch_remap_band(const RemapParams& r, int persistent_blocks, cudaStream_t st,
                              int threads) {
  launch_l3(r, persistent_blocks, st, threads);
  return cudaGetLastError();
}

cudaError_t launch_remap_single(const RemapParams& r, int persistent_blocks, cudaStream_t st,
                                int threads) {
  const int ntile = r.box.n[0] * r.box.n[1] * r.box.n[2];
  if (ntile <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(r.counters, 0, 4 * sizeof(int), st);
  if (e != cudaSuccess) return e;
  // (a cached band's count is reset by the host once per rebuild, before the body's first box)
  k_remap_l0<<<(ntile + 255) / 256, 256, 0, st>>>(r);
  if (r.fused12) {
    k_remap_l12<<<persistent_blocks, threads, 0, st>>>(r);
  } else {
    k_remap_l1<<<persistent_blocks, threads, 0, st>>>(r);
    k_remap_l2<<<persistent_blocks, threads, 0, st>>>(r);
  }
  launch_l3(r, persistent_blocks, st, threads);
  return cudaGetLastError();
}

}  // namespace psm
