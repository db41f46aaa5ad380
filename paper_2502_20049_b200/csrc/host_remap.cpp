// host_remap.cpp — fraction-remap planning (swept boxes, single-body narrow band vs general
// boxes), cached narrow bands, double-buffered solid words and the remap-ahead pipeline
// (DESIGN.md §1, §6.2).
#include "psm_ctx.h"

namespace psm {

// Persistent remap blocks when the remap overlaps the collide (remap-ahead): one per SM, two at
// s >= 2 where the 64-register chunked sample kernel fits twice into the registers one collide
// block frees (measured: c3 scenario A at s = 2, 9963 -> 10183 MLUPS; one per SM is better for
// the s = 1 band of c5w).  PSM_AHEAD_BLOCKS overrides.
// the cached band pays off while its exact pass is cheap: R1 up to s = 1 (8 sub-samples per
// cell; at s >= 2 the radius-2 band's 64/512 samples per cell cost more than the L0-L2
// pipeline), R2 at every s (one block popcount per cell: c3 scenario A at s = 2, 1.014 ->
// 0.924 ms per step)
static bool cache_pays(const psm_ctx* c, const Body& b) {
  return b.mapping == 1 ? b.s <= c->cache_max_s_r2 : b.s <= c->cache_max_s;
}

static int ahead_blocks(const psm_ctx* c, int s) {
  if (c->ahead_blocks_env > 0) return c->ahead_blocks_env;
  return s >= 2 ? 2 * 148 : 148;
}

psm_status run_map(psm_ctx* c, const std::vector<Box>& boxes) {
  MapParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.g = c->geom;
  mp.word = c->word;
  mp.tile_flag = c->tile_flag;
  for (int id = 1; id <= kMaxBodies; ++id) {
    const Body& b = c->bodies[id];
    BodyGeo& g = mp.bodies[id];
    if (!b.present) continue;
    std::memcpy(g.Q, b.ms.Qc, sizeof(g.Q));
    std::memcpy(g.t, b.ms.tc, sizeof(g.t));
    for (int a = 0; a < 3; ++a) {
      g.lo1[a] = b.bmin[a] - 1.0;
      g.hi1[a] = b.bmax[a] + 1.0;
    }
    g.r2 = b.radius * b.radius;
    for (int a = 0; a < 3; ++a) {
      g.o[a] = b.o[a];
      g.dims_b[a] = (int)b.dims[a];
    }
    g.kind = b.kind;
    g.s = b.s;
    g.words = b.words;
    g.present = 1;
    g.mapping = b.mapping;
    g.bits = b.d_bits;
    g.mask = b.d_mask;
  }
  // boxes -> local tile boxes, launched in batches of kMaxBoxes
  std::vector<MapBox> tb;
  for (const Box& b : boxes) {
    const int64_t zlo = std::max<int64_t>(b.lo[2], c->z0) - c->z0;
    const int64_t zhi = std::min<int64_t>(b.hi[2], c->z0 + c->nzl) - c->z0;
    if (zhi <= zlo || b.hi[0] <= b.lo[0] || b.hi[1] <= b.lo[1]) continue;
    MapBox m;
    m.t0[0] = (int)(b.lo[0] / kTileX);
    m.n[0] = (int)((b.hi[0] - 1) / kTileX + 1 - m.t0[0]);
    m.t0[1] = (int)(b.lo[1] / kTileY);
    m.n[1] = (int)((b.hi[1] - 1) / kTileY + 1 - m.t0[1]);
    m.t0[2] = (int)(zlo / kTileZ);
    m.n[2] = (int)((zhi - 1) / kTileZ + 1 - m.t0[2]);
    m.first = 0;
    // bodies whose current box overlaps the TILE-ALIGNED extent of this box (the kernels
    // rewrite whole tiles, so every body that can own a cell of those tiles must be evaluated)
    const int64_t tlo[3] = {(int64_t)m.t0[0] * kTileX, (int64_t)m.t0[1] * kTileY,
                            (int64_t)m.t0[2] * kTileZ + c->z0};
    const int64_t thi[3] = {tlo[0] + (int64_t)m.n[0] * kTileX, tlo[1] + (int64_t)m.n[1] * kTileY,
                            tlo[2] + (int64_t)m.n[2] * kTileZ};
    m.bodymask = 0;
    for (int id = 1; id <= kMaxBodies; ++id) {
      const Body& bd = c->bodies[id];
      if (!bd.present || !bd.ms.has_box) continue;
      std::vector<Box> pieces;
      add_box(c, bd.ms.box_lo, bd.ms.box_hi, pieces);
      for (const Box& pc : pieces) {
        bool ov = true;
        for (int a = 0; a < 3; ++a)
          if (pc.hi[a] <= tlo[a] || pc.lo[a] >= thi[a]) ov = false;
        if (ov) {
          m.bodymask |= 1u << id;
          break;
        }
      }
    }
    if (!m.bodymask) {
      // nothing can be inside: still launched so the words/flags of the box are cleared
    }
    tb.push_back(m);
  }
  static const bool stats_on = std::getenv("PSM_MAP_STATS") != nullptr;
  unsigned long long* dstats = nullptr;
  if (stats_on) {
    CUDA_TRY(c, cudaMalloc(&dstats, 8 * 8));
    CUDA_TRY(c, cudaMemsetAsync(dstats, 0, 8 * 8, c->mst));
  }
  mp.stats = dstats;
  if (record(c, 0, 0, c->mst) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
  const bool force_general = c->force_general;
  // cached bands: bodies rebuilt in single-body boxes only; capacity = every cell of their boxes
  size_t need[kMaxBodies + 1] = {};
  int nsingle[kMaxBodies + 1] = {}, ngeneral[kMaxBodies + 1] = {};
  for (size_t i = 0; i < tb.size(); ++i) {
    const int pc = __builtin_popcount(tb[i].bodymask);
    if (pc == 1 && !force_general) {
      const int id = __builtin_ctz(tb[i].bodymask);
      need[id] += (size_t)tb[i].n[0] * tb[i].n[1] * tb[i].n[2] * kTileCells;
      nsingle[id] += 1;
    } else {
      for (int id = 1; id <= kMaxBodies; ++id)
        if (tb[i].bodymask & (1u << id)) ngeneral[id] += 1;
    }
  }
  for (int id = 1; id <= kMaxBodies; ++id) {
    Body& bd = c->bodies[id];
    if (ngeneral[id]) bd.ms.cache = false;  // shares a box with another body: no band cache
    if (!bd.want_cache || ngeneral[id] || !nsingle[id]) {
      bd.want_cache = false;
      continue;
    }
    const int sl = bd.ms.slot;
    if (bd.ccap[sl] < need[id]) {
      // stream-ordered (no device-wide sync in the middle of a pipelined step), with headroom
      // so that the slowly changing box of a moving body rarely regrows it
      const size_t cap = need[id] + need[id] / 4;
      if (bd.cband[sl]) CUDA_TRY(c, cudaFreeAsync(bd.cband[sl], c->mst));
      if (bd.ccnt[sl]) CUDA_TRY(c, cudaFreeAsync(bd.ccnt[sl], c->mst));
      bd.cband[sl] = nullptr;
      bd.ccnt[sl] = nullptr;
      bd.ccap[sl] = 0;
      CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&bd.cband[sl]), cap * 4, c->mst));
      CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&bd.ccnt[sl]), cap * 4, c->mst));
      bd.ccap[sl] = cap;
    }
    if (!bd.cn[sl]) CUDA_TRY(c, cudaMallocAsync(reinterpret_cast<void**>(&bd.cn[sl]), sizeof(int), c->mst));
    CUDA_TRY(c, cudaMemsetAsync(bd.cn[sl], 0, sizeof(int), c->mst));
  }
  for (size_t i = 0; i < tb.size(); ++i) {
    if (__builtin_popcount(tb[i].bodymask) == 1 && !force_general) {
      // one body in the box: narrow-band pipeline (k_remap.cu)
      RemapParams r;
      std::memset(&r, 0, sizeof(r));
      r.g = c->geom;
      r.fgx = make_fastdiv((uint32_t)r.g.gx);
      r.fgxy = make_fastdiv((uint32_t)r.g.gx * (uint32_t)r.g.gy);
      r.fused12 = c->remap_fused12;
      r.box = tb[i];
      r.id = __builtin_ctz(tb[i].bodymask);
      r.body = mp.bodies[r.id];
      r.word = c->word;
      r.tile_flag = c->tile_flag;
      r.counters = c->r_counters;
      r.tiles = c->r_tiles;
      r.segs = c->r_segs;
      r.segq = c->r_segq;
      r.band = c->r_band;
      r.bandcnt = c->r_bandcnt;
      r.bandn = c->r_counters + 2;
      r.seg_cap = c->seg_cap;
      r.band_cap = c->band_cap;
      Body& bd = c->bodies[r.id];
      if (bd.want_cache) {  // build the body's cached band (decisions with one cell of slack)
        const int sl = bd.ms.slot;
        r.margin = 1;
        r.band = bd.cband[sl];
        r.bandcnt = bd.ccnt[sl];
        r.bandn = bd.cn[sl];
        r.band_cap = (int)std::min<size_t>(bd.ccap[sl], (size_t)INT32_MAX);
      }
      CUDA_TRY(c, launch_remap_single(r, c->mst == c->st ? 148 * 8 : ahead_blocks(c, r.body.s), c->mst,
                                      c->mst == c->st ? 256 : c->ahead_threads));
      c->launches += remap_single_kernels(r);
      continue;
    }
    // general box (several bodies may cover its cells): one launch, 3D grid of its tiles
    mp.box[0] = tb[i];
    mp.nbox = 1;
    mp.ntiles = tb[i].n[0] * tb[i].n[1] * tb[i].n[2];
    CUDA_TRY(c, launch_map(mp, c->mst));
    c->launches += 1;
  }
  for (int id = 1; id <= kMaxBodies; ++id) {
    Body& bd = c->bodies[id];
    if (!bd.want_cache) continue;
    bd.want_cache = false;
    bd.ms.cache = true;
    std::memcpy(bd.ms.Qrb, bd.ms.Qc, sizeof(bd.ms.Qrb));
    std::memcpy(bd.ms.trb, bd.ms.tc, sizeof(bd.ms.trb));
  }
  if (record(c, 0, 1, c->mst) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
  if (dstats) {
    unsigned long long h[8];
    CUDA_TRY(c, cudaMemcpyAsync(h, dstats, sizeof(h), cudaMemcpyDeviceToHost, c->mst));
    CUDA_TRY(c, cudaStreamSynchronize(c->mst));
    cudaFree(dstats);
    std::fprintf(stderr,
                 "[psm map] boxes %zu  8-cell segments: out %llu in %llu cell %llu | "
                 "cells: out %llu in %llu band %llu | tiles skipped %llu\n",
                 tb.size(), h[0], h[1], h[2], h[3], h[4], h[5], h[7]);
  }
  return PSM_OK;
}

// the active and spare solid-word buffers trade places (with every body's mapping state)
void swap_buffers(psm_ctx* c) {
  std::swap(c->word, c->word_alt);
  std::swap(c->tile_flag, c->tile_flag_alt);
  for (int id = 1; id <= kMaxBodies; ++id) std::swap(c->bodies[id].ms, c->bodies[id].alt);
}

psm_status ensure_pipeline(psm_ctx* c) {
  if (c->map_st) return PSM_OK;
  int lo_prio = 0, hi_prio = 0;
  CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  // highest priority: measured 40.7k vs 40.0k MLUPS (c5w) against the default priority, which
  // lets the remap start only as the collide drains
  CUDA_TRY(c, cudaStreamCreateWithPriority(&c->map_st, cudaStreamNonBlocking, hi_prio));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_map, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_coll, cudaEventDisableTiming));
  return PSM_OK;
}

// Upper bound on how far any point of body b moves between the band's build pose and (Q, t):
// |mi(t - t_rb)| + r_bound * |Q - Q_rb|_F / sqrt(2)  (the chord of a rotation by theta is
// 2 r sin(theta/2) = r |Q - Q_rb|_F / sqrt(2)).
double band_displacement(const psm_ctx* c, const Body& b, const double Q[9],
                                 const double t[3]) {
  double dt2 = 0.0, dq2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    double d = t[a] - b.ms.trb[a];
    if (c->grid.bc[a] == PSM_PERIODIC) {
      const double L = extent(c, a);
      d -= L * std::nearbyint(d / L);
    }
    dt2 += d * d;
  }
  for (int k = 0; k < 9; ++k) dq2 += (Q[k] - b.ms.Qrb[k]) * (Q[k] - b.ms.Qrb[k]);
  return std::sqrt(dt2) + b.rbound * std::sqrt(dq2 * 0.5);
}

bool boxes_overlap(const psm_ctx* c, const Body& b, const std::vector<Box>& boxes) {
  std::vector<Box> mine;
  add_box(c, b.ms.box_lo, b.ms.box_hi, mine);
  for (const Box& m : mine)
    for (const Box& o : boxes) {
      bool ov = true;
      for (int a = 0; a < 3; ++a)
        if (m.hi[a] <= o.lo[a] || m.lo[a] >= o.hi[a]) ov = false;
      if (ov) return true;
    }
  return false;
}

// remap the given bodies at the pose of `step` (or all present bodies if ids empty).  A body with
// a valid cached band that has moved less than one cell since the band was built (and whose box
// no other remapped body touches) only re-runs the exact pass over its band.
psm_status remap(psm_ctx* c, const std::vector<int>& ids, int64_t step) {
  const bool no_cache = c->no_cache;
  std::vector<Box> boxes;
  std::vector<int> incr;
  for (int id : ids) {
    Body& b = c->bodies[id];
    if (!b.present) continue;
    double Q[9], t[3];
    if (b.dynamic) {
      std::memcpy(Q, b.Qd, sizeof(Q));
      std::memcpy(t, b.td, sizeof(t));
    } else if (b.moving) {
      pose_at(c, b, step, Q, t);
    } else {
      std::memcpy(Q, b.Q0, sizeof(Q));
      std::memcpy(t, b.t0, sizeof(t));
    }
    std::memcpy(b.ms.Qc, Q, sizeof(Q));
    std::memcpy(b.ms.tc, t, sizeof(t));
    b.ms.mapped_step = step;
    if (!no_cache && !c->dbg && b.ms.cache && b.ms.has_box &&
        band_displacement(c, b, Q, t) < 1.0 - 1e-6) {
      incr.push_back(id);
      continue;
    }
    b.ms.cache = false;
    b.want_cache = !no_cache && !c->dbg && cache_pays(c, b);
    remap_region(c, b, Q, t, boxes);
  }
  // an incremental body whose (build) box meets a box remapped now goes the full way
  for (bool changed = true; changed;) {
    changed = false;
    for (size_t k = 0; k < incr.size(); ++k) {
      Body& b = c->bodies[incr[k]];
      if (!boxes_overlap(c, b, boxes)) continue;
      b.ms.cache = false;
      b.want_cache = cache_pays(c, b);
      remap_region(c, b, b.ms.Qc, b.ms.tc, boxes);
      incr.erase(incr.begin() + (long)k);
      changed = true;
      break;
    }
  }
  if (c->dbg && !boxes.empty()) {  // leaving the debug field mode: the words are authoritative
    c->dbg = false;
    CUDA_TRY(c, cudaMemsetAsync(c->tile_flag, 0, (size_t)c->ntiles, c->mst));
    std::vector<Box> all;
    for (int id = 1; id <= kMaxBodies; ++id)
      if (c->bodies[id].present && c->bodies[id].ms.has_box)
        add_box(c, c->bodies[id].ms.box_lo, c->bodies[id].ms.box_hi, all);
    CUDA_TRY(c, cudaMemsetAsync(c->word, 0, (size_t)c->ncell_local * 4, c->mst));
    psm_status s = run_map(c, all);
    if (s != PSM_OK) return s;
  }
  if (!boxes.empty()) {
    psm_status s = run_map(c, boxes);
    if (s != PSM_OK) return s;
  }
  if (!incr.empty() && record(c, 0, 0, c->mst) != cudaSuccess)
    FAIL(c, PSM_E_CUDA, "event record failed");
  for (int id : incr) {
    Body& b = c->bodies[id];
    const int sl = b.ms.slot;
    RemapParams r;
    std::memset(&r, 0, sizeof(r));
    r.g = c->geom;
    r.fgx = make_fastdiv((uint32_t)r.g.gx);
    r.fgxy = make_fastdiv((uint32_t)r.g.gx * (uint32_t)r.g.gy);
    r.id = id;
    BodyGeo& g = r.body;
    std::memcpy(g.Q, b.ms.Qc, sizeof(g.Q));
    std::memcpy(g.t, b.ms.tc, sizeof(g.t));
    for (int a = 0; a < 3; ++a) {
      g.lo1[a] = b.bmin[a] - 1.0;
      g.hi1[a] = b.bmax[a] + 1.0;
      g.o[a] = b.o[a];
      g.dims_b[a] = (int)b.dims[a];
    }
    g.r2 = b.radius * b.radius;
    g.kind = b.kind;
    g.s = b.s;
    g.words = b.words;
    g.present = 1;
    g.mapping = b.mapping;
    g.bits = b.d_bits;
    g.mask = b.d_mask;
    r.word = c->word;
    r.tile_flag = c->tile_flag;
    r.band = b.cband[sl];
    r.bandcnt = b.ccnt[sl];
    r.bandn = b.cn[sl];
    r.band_cap = (int)std::min<size_t>(b.ccap[sl], (size_t)INT32_MAX);
    r.margin = 1;
    CUDA_TRY(c, launch_remap_band(r, c->mst == c->st ? 148 * 8 : ahead_blocks(c, b.s), c->mst,
                                  c->mst == c->st ? 256 : c->ahead_threads));
    c->launches += remap_l3_kernels(r.body);
  }
  if (!incr.empty() && record(c, 0, 1, c->mst) != cudaSuccess)
    FAIL(c, PSM_E_CUDA, "event record failed");
  return PSM_OK;
}

// Remap-ahead (prescribed motion only): enqueue the remap for step `next` into the spare buffer
// on map_st, after the collide that last read that buffer (ev_coll); ev_map marks completion.
// The remap is latency/ALU-bound and the collide HBM-bound, so the two overlap.
psm_status remap_ahead(psm_ctx* c, int64_t next) {
  CUDA_TRY(c, cudaStreamWaitEvent(c->map_st, c->ev_coll, 0));
  swap_buffers(c);
  c->mst = c->map_st;
  std::vector<int> ids;
  if (!c->alt_valid) {  // start the spare buffer from scratch: every body mapped afresh
    CUDA_TRY(c, cudaMemsetAsync(c->word, 0, (size_t)c->ncell_local * 4, c->mst));
    CUDA_TRY(c, cudaMemsetAsync(c->tile_flag, 0, (size_t)c->ntiles, c->mst));
    for (int id = 1; id <= kMaxBodies; ++id) {
      const int sl = c->bodies[id].ms.slot;
      c->bodies[id].ms = MapState();
      c->bodies[id].ms.slot = sl;
      if (c->bodies[id].present) ids.push_back(id);
    }
    c->alt_valid = true;
  } else {
    for (int id = 1; id <= kMaxBodies; ++id) {
      const Body& b = c->bodies[id];
      if (b.present && b.ms.mapped_step != next &&
          (b.moving || b.ms.mapped_step < 0))
        ids.push_back(id);
    }
  }
  psm_status st = PSM_OK;
  if (!ids.empty()) st = remap(c, ids, next);
  c->mst = c->st;
  swap_buffers(c);
  if (st != PSM_OK) return st;
  CUDA_TRY(c, cudaEventRecord(c->ev_map, c->map_st));
  return PSM_OK;
}

}  // namespace psm
