// psm_api.cpp — C ABI of the B200 PSM hot path (include/psm.h).  Host orchestration only:
// validation, memory layout, closed-form pose advance (host fp64 libm, reading A13),
// remap-box planning, the per-step launch sequence, NCCL halo exchange and force/torque
// allreduce.  Every arithmetic step of the method runs in the sm_100a kernels (k_*.cu).
#include "psm.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "psm_device.cuh"
#include "psm_host.h"
#include "psm_internal.h"

using namespace psm;

namespace {

constexpr int kFtChunks = 296;           // 2 x 148 SMs, pass-1 blocks of the F/T reduction
constexpr size_t kStageBudget = 256ull << 20;
constexpr size_t kGeomCapBytes = 1ull << 30;

struct MapState {
  double Qc[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, tc[3] = {0, 0, 0};  // pose of the mapping
  int64_t mapped_step = -1;
  bool has_box = false;
  int64_t box_lo[3] = {0, 0, 0}, box_hi[3] = {0, 0, 0};  // mapped box (global, unwrapped)
  // cached narrow band (k_remap.cu, margin 1): valid for poses within one cell of (Qrb, trb)
  int slot = 0;        // which of the body's two band stores belongs to this word buffer
  bool cache = false;
  double Qrb[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, trb[3] = {0, 0, 0};
};

struct Body {
  bool present = false;
  int kind = 0, s = 0, mapping = 0;
  double radius = 0, rbound = 0;
  double bmin[3] = {0, 0, 0}, bmax[3] = {0, 0, 0};  // body-frame AABB of the shape
  // mesh geometry field (device)
  double o[3] = {0, 0, 0};
  int64_t dims[3] = {0, 0, 0};
  int words = 1;
  unsigned long long* d_bits = nullptr;
  uint8_t* d_mask = nullptr;
  // prescribed motion: pose at step0, closed-form advance
  double Q0[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t0[3] = {0, 0, 0};
  double v[3] = {0, 0, 0}, w[3] = {0, 0, 0};
  int64_t step0 = 0;
  bool moving = false;
  // mapping state of the active solid-word buffer (ms) and of the spare one (alt, used by the
  // remap-ahead pipeline of psm_step; swapped together with the buffers)
  MapState ms, alt;
  // band stores (device), indexed by MapState::slot; capacity in cells
  uint32_t* cband[2] = {nullptr, nullptr};
  int* ccnt[2] = {nullptr, nullptr};
  int* cn[2] = {nullptr, nullptr};
  size_t ccap[2] = {0, 0};
  bool want_cache = false;  // transient: the current remap rebuilds this body's band
  Body() { alt.slot = 1; }
  // two-way coupling: state advanced by the host integrator after every step
  bool dynamic = false;
  double mass = 0, Ib[9] = {0}, fext[3] = {0, 0, 0}, text[3] = {0, 0, 0};
  double Ma = 0, Ia[9] = {0};                    // virtual mass / inertia (A28)
  double dv[3] = {0, 0, 0}, dw[3] = {0, 0, 0};   // last velocity increments (world frame)
  double Qd[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, td[3] = {0, 0, 0}, vd[3] = {0, 0, 0},
         wd[3] = {0, 0, 0};
};

struct Box {
  int64_t lo[3], hi[3];  // global cells, [lo, hi), already wrapped into the domain
};

}  // namespace

struct psm_ctx {
  psm_grid grid{};
  int Q = 19;
  double tau = 0.8;
  psm_options opt{};
  double u_in[3] = {0.0, 0.0, 0.0};  // A30 open boundaries (bc[0] == PSM_INOUT)
  double rho_out = 1.0;
  int rank = 0, world = 1;
  int64_t z0 = 0, nzl = 0;
  Geom geom{};
  int64_t ncell_local = 0, ntiles = 0;
  size_t S = 8;
  // device memory
  void* mem = nullptr;
  size_t mem_bytes = 0;
  bool own_mem = false, bound = false;
  void* A[2] = {nullptr, nullptr};
  int cur = 0;
  uint32_t* word = nullptr;          // active solid-word buffer (read by the next collide)
  uint8_t* tile_flag = nullptr;
  uint32_t* word_alt = nullptr;      // spare buffer: the remap of step n+1 runs into it while
  uint8_t* tile_flag_alt = nullptr;  // the collide of step n reads the active one
  bool alt_valid = false;            // the spare buffer's words match every body's alt state
  cudaStream_t mst = nullptr;        // stream the remap launches go to (st, or map_st ahead)
  cudaStream_t map_st = nullptr;     // remap-ahead stream (high priority)
  cudaEvent_t ev_map = nullptr, ev_coll = nullptr;
  int ahead_blocks = 148;            // persistent remap blocks when overlapped with the collide
  int ahead_threads = 256;
  double* partial = nullptr;
  double* overflow = nullptr;
  unsigned long long* err = nullptr;
  double* ft_scratch = nullptr;
  double* ft_out = nullptr;
  int* ft_ids = nullptr;
  double* stage = nullptr;
  size_t stage_bytes = 0;
  // narrow-band remap lists
  int* r_counters = nullptr;
  int* r_tiles = nullptr;
  uint32_t* r_segs = nullptr;
  float4* r_segq = nullptr;
  uint32_t* r_band = nullptr;
  int* r_bandcnt = nullptr;
  int seg_cap = 0, band_cap = 0;
  double* pinned = nullptr;  // host staging (ft + err)
  // test-only dense fields
  double *dbg_B = nullptr, *dbg_us = nullptr;
  uint8_t* dbg_id = nullptr;
  bool dbg = false;
  Body bodies[kMaxBodies + 1];
  int64_t step = 0;
  double ft[kMaxBodies + 1][kSlotVals] = {};
  bool ft_valid = false;
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_st = nullptr;     // halo stream (overlaps the interior collide)
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;
  // fused peer-store halo (psm_halo_mode 2)
  bool p2p_checked = false, p2p = false;
  bool has_up = false, has_dn = false;
  void* ipc_up = nullptr;            // opened IPC base of the upper / lower neighbour's memory
  void* ipc_dn = nullptr;
  char* up_A[2] = {nullptr, nullptr};
  char* dn_A[2] = {nullptr, nullptr};
  int64_t up_qs = 0, dn_qs = 0, dn_nzl = 0;
  unsigned long long* up_flag = nullptr;  // the upper neighbour's "from below" flag word
  unsigned long long* dn_flag = nullptr;  // the lower neighbour's "from above" flag word
  unsigned long long* flags = nullptr;    // mine: [0] from below, [1] from above, [2] hs error
  unsigned long long epoch = 0;
  unsigned char nccl_id[128] = {};
  std::string err_msg;
  int64_t launches = 0;
  bool prof = false;
  std::vector<std::array<cudaEvent_t, 2>> ev[PSM_NUM_PHASES];
  double prof_ms[PSM_NUM_PHASES] = {};
  int64_t prof_cnt[PSM_NUM_PHASES] = {};
};

static std::string g_last_error;

#define FAIL(ctx, code, msg)                  \
  do {                                        \
    std::string _m = (msg);                   \
    if (ctx) (ctx)->err_msg = _m;             \
    g_last_error = _m;                        \
    return (code);                            \
  } while (0)

#define CUDA_TRY(ctx, expr)                                                             \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      FAIL(ctx, PSM_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                             \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      FAIL(ctx, PSM_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));        \
  } while (0)

// ---------------------------------------------------------------------------- helpers ------
static void free_bands(Body& b) {  // callers have synchronised the streams
  for (int k = 0; k < 2; ++k) {
    if (b.cband[k]) cudaFreeAsync(b.cband[k], 0);
    if (b.ccnt[k]) cudaFreeAsync(b.ccnt[k], 0);
    if (b.cn[k]) cudaFreeAsync(b.cn[k], 0);
    b.cband[k] = nullptr;
    b.ccnt[k] = nullptr;
    b.cn[k] = nullptr;
    b.ccap[k] = 0;
  }
}

static void rodrigues(const double w[3], double n, const double Q0[9], double out[9]) {
  // Q_n = Rot(w/|w|, n|w|) Q_0 (A13: host libm sin/cos)
  const double wn = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (wn > 0.0) {
    const double k[3] = {w[0] / wn, w[1] / wn, w[2] / wn};
    const double th = n * wn, s = std::sin(th), c = 1.0 - std::cos(th);
    const double K[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double k2 = 0.0;
        for (int l = 0; l < 3; ++l) k2 += K[3 * r + l] * K[3 * l + cc];
        R[3 * r + cc] += s * K[3 * r + cc] + c * k2;
      }
  }
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) {
      double acc = 0.0;
      for (int l = 0; l < 3; ++l) acc += R[3 * r + l] * Q0[3 * l + cc];
      out[3 * r + cc] = acc;
    }
}

static double extent(const psm_ctx* c, int a) {
  return (double)(a == 0 ? c->grid.nx : (a == 1 ? c->grid.ny : c->grid.nz));
}

static void pose_at(const psm_ctx* c, const Body& b, int64_t step, double Q[9], double t[3]) {
  const double n = (double)(step - b.step0);
  for (int a = 0; a < 3; ++a) {
    double x = b.t0[a] + n * b.v[a];
    if (c->grid.bc[a] == PSM_PERIODIC) {
      const double L = extent(c, a);
      x = x - L * std::floor(x / L);
    }
    t[a] = x;
  }
  rodrigues(b.w, n, b.Q0, Q);
}

// world box of the cells the body can touch at pose (Q, t): AABB of the rotated body-frame
// AABB, dilated by one cell (the kernel's per-cell filter uses the same +-1 margin)
static void body_box(const psm_ctx* c, const Body& b, const double Q[9], const double t[3],
                     int64_t lo[3], int64_t hi[3]) {
  (void)c;
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int k = 0; k < 8; ++k) {
    const double p[3] = {(k & 1) ? b.bmax[0] : b.bmin[0], (k & 2) ? b.bmax[1] : b.bmin[1],
                         (k & 4) ? b.bmax[2] : b.bmin[2]};
    for (int a = 0; a < 3; ++a) {
      const double w = Q[3 * a] * p[0] + Q[3 * a + 1] * p[1] + Q[3 * a + 2] * p[2];
      mn[a] = std::min(mn[a], w);
      mx[a] = std::max(mx[a], w);
    }
  }
  for (int a = 0; a < 3; ++a) {
    // +2: one cell for the kernel filter margin, one for rounding of the corner transform
    lo[a] = (int64_t)std::floor(t[a] + mn[a] - 2.0);
    hi[a] = (int64_t)std::floor(t[a] + mx[a] + 2.0) + 1;
  }
}

// split [lo, hi) on axis a into in-domain pieces
static int axis_pieces(const psm_ctx* c, int a, int64_t lo, int64_t hi, int64_t out[2][2]) {
  const int64_t L = (int64_t)extent(c, a);
  if (c->grid.bc[a] != PSM_PERIODIC) {
    lo = std::max<int64_t>(lo, 0);
    hi = std::min<int64_t>(hi, L);
    if (hi <= lo) return 0;
    out[0][0] = lo;
    out[0][1] = hi;
    return 1;
  }
  if (hi - lo >= L) {
    out[0][0] = 0;
    out[0][1] = L;
    return 1;
  }
  int64_t l = ((lo % L) + L) % L, len = hi - lo;
  if (l + len <= L) {
    out[0][0] = l;
    out[0][1] = l + len;
    return 1;
  }
  out[0][0] = l;
  out[0][1] = L;
  out[1][0] = 0;
  out[1][1] = l + len - L;
  return 2;
}

static void add_box(const psm_ctx* c, const int64_t lo[3], const int64_t hi[3],
                    std::vector<Box>& boxes) {
  int64_t px[2][2], py[2][2], pz[2][2];
  const int nxp = axis_pieces(c, 0, lo[0], hi[0], px);
  const int nyp = axis_pieces(c, 1, lo[1], hi[1], py);
  const int nzp = axis_pieces(c, 2, lo[2], hi[2], pz);
  for (int i = 0; i < nxp; ++i)
    for (int j = 0; j < nyp; ++j)
      for (int k = 0; k < nzp; ++k) {
        Box b;
        b.lo[0] = px[i][0]; b.hi[0] = px[i][1];
        b.lo[1] = py[j][0]; b.hi[1] = py[j][1];
        b.lo[2] = pz[k][0]; b.hi[2] = pz[k][1];
        boxes.push_back(b);
      }
}

// region to remap for body b moving to pose t: hull of the old and new boxes if they overlap
// (after the periodic shift that brings them closest), both boxes otherwise
static void remap_region(const psm_ctx* c, Body& b, const double Q[9], const double t[3],
                         std::vector<Box>& boxes) {
  int64_t lo[3], hi[3];
  body_box(c, b, Q, t, lo, hi);
  if (b.ms.has_box) {
    bool overlap = true;
    int64_t slo[3], shi[3];
    for (int a = 0; a < 3; ++a) {
      int64_t shift = 0;
      if (c->grid.bc[a] == PSM_PERIODIC) {
        const int64_t L = (int64_t)extent(c, a);
        const double dc = 0.5 * ((lo[a] + hi[a]) - (b.ms.box_lo[a] + b.ms.box_hi[a]));
        shift = -(int64_t)std::llround(dc / (double)L) * L;
      }
      slo[a] = lo[a] + shift;
      shi[a] = hi[a] + shift;
      if (slo[a] >= b.ms.box_hi[a] || shi[a] <= b.ms.box_lo[a]) overlap = false;
    }
    if (overlap) {
      int64_t ulo[3], uhi[3];
      for (int a = 0; a < 3; ++a) {
        ulo[a] = std::min(slo[a], b.ms.box_lo[a]);
        uhi[a] = std::max(shi[a], b.ms.box_hi[a]);
      }
      add_box(c, ulo, uhi, boxes);
    } else {
      add_box(c, b.ms.box_lo, b.ms.box_hi, boxes);
      add_box(c, lo, hi, boxes);
    }
  } else {
    add_box(c, lo, hi, boxes);
  }
  for (int a = 0; a < 3; ++a) {
    b.ms.box_lo[a] = lo[a];
    b.ms.box_hi[a] = hi[a];
  }
  b.ms.has_box = true;
}

static cudaError_t record(psm_ctx* c, int phase, int which, cudaStream_t s = nullptr) {
  if (!c->prof) return cudaSuccess;
  if (which == 0) {
    std::array<cudaEvent_t, 2> e{};
    cudaError_t r = cudaEventCreate(&e[0]);
    if (r != cudaSuccess) return r;
    r = cudaEventCreate(&e[1]);
    if (r != cudaSuccess) return r;
    c->ev[phase].push_back(e);
  }
  return cudaEventRecord(c->ev[phase].back()[which], s ? s : c->st);
}

// ------------------------------------------------------------------------- memory plan -----
struct Plan {
  size_t off_A0, off_A1, off_word, off_flag, off_word_alt, off_flag_alt, off_partial, off_overflow, off_err, off_scratch,
      off_ftout, off_ids, off_stage, off_flags, stage_bytes, total;
  size_t off_rcnt, off_rtiles, off_rsegs, off_rsegq, off_rband, off_rbandcnt;
  int seg_cap, band_cap;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static Plan make_plan(const psm_ctx* c) {
  Plan p{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  const size_t arr = (size_t)c->Q * (size_t)c->geom.qstride * c->S;
  p.off_A0 = take(arr);
  p.off_A1 = (c->opt.pattern == PSM_TWO_ARRAY) ? take(arr) : 0;
  p.off_word = take((size_t)c->ncell_local * 4);
  p.off_flag = take((size_t)c->ntiles);
  p.off_word_alt = take((size_t)c->ncell_local * 4);
  p.off_flag_alt = take((size_t)c->ntiles);
  p.off_partial = take((size_t)c->ntiles * 2 * (1 + kSlotVals) * 8);
  p.off_overflow = take((kMaxBodies + 1) * kSlotVals * 8);
  p.off_err = take(8);
  p.off_scratch = take((size_t)kFtChunks * kMaxBodies * kSlotVals * 8);
  p.off_ftout = take(kMaxBodies * kSlotVals * 8);
  p.off_ids = take(kMaxBodies * 4);
  p.off_flags = take(64);
  // narrow-band remap lists (k_remap.cu); overflow is handled in-kernel (serial fallback)
  p.seg_cap = (int)std::min<int64_t>(32 * c->ntiles, 1 << 22);
  p.band_cap = (int)std::min<int64_t>(c->ncell_local, 1 << 23);
  p.off_rcnt = take(4 * sizeof(int));
  p.off_rtiles = take((size_t)c->ntiles * 4);
  p.off_rsegs = take((size_t)p.seg_cap * 4);
  p.off_rsegq = take((size_t)p.seg_cap * 16);
  p.off_rband = take((size_t)p.band_cap * 4);
  p.off_rbandcnt = take((size_t)p.band_cap * 4);
  const size_t plane = (size_t)c->grid.nx * c->grid.ny * 8;
  const size_t per = plane * (size_t)c->Q;
  size_t planes = std::max<size_t>(3, kStageBudget / per);
  planes = std::min<size_t>(planes, (size_t)c->nzl + 2);
  p.stage_bytes = planes * per;
  p.off_stage = take(p.stage_bytes);
  p.total = off;
  return p;
}

static psm_status ensure_pinned(psm_ctx* c);

static psm_status ensure_comm(psm_ctx* c);

static psm_status bind(psm_ctx* c, void* mem, size_t bytes) {
  psm_status ps = ensure_pinned(c);
  if (ps != PSM_OK) return ps;
  ps = ensure_comm(c);
  if (ps != PSM_OK) return ps;
  Plan p = make_plan(c);
  if (bytes < p.total)
    FAIL(c, PSM_E_OOM, "bound buffer has " + std::to_string(bytes) + " bytes, need " +
                           std::to_string(p.total));
  char* m = static_cast<char*>(mem);
  c->mem = mem;
  c->mem_bytes = bytes;
  c->A[0] = m + p.off_A0;
  c->A[1] = (c->opt.pattern == PSM_TWO_ARRAY) ? (void*)(m + p.off_A1) : nullptr;
  c->word = reinterpret_cast<uint32_t*>(m + p.off_word);
  c->tile_flag = reinterpret_cast<uint8_t*>(m + p.off_flag);
  c->word_alt = reinterpret_cast<uint32_t*>(m + p.off_word_alt);
  c->tile_flag_alt = reinterpret_cast<uint8_t*>(m + p.off_flag_alt);
  c->alt_valid = false;
  c->partial = reinterpret_cast<double*>(m + p.off_partial);
  c->overflow = reinterpret_cast<double*>(m + p.off_overflow);
  c->err = reinterpret_cast<unsigned long long*>(m + p.off_err);
  c->ft_scratch = reinterpret_cast<double*>(m + p.off_scratch);
  c->ft_out = reinterpret_cast<double*>(m + p.off_ftout);
  c->ft_ids = reinterpret_cast<int*>(m + p.off_ids);
  c->flags = reinterpret_cast<unsigned long long*>(m + p.off_flags);
  c->stage = reinterpret_cast<double*>(m + p.off_stage);
  c->r_counters = reinterpret_cast<int*>(m + p.off_rcnt);
  c->r_tiles = reinterpret_cast<int*>(m + p.off_rtiles);
  c->r_segs = reinterpret_cast<uint32_t*>(m + p.off_rsegs);
  c->r_segq = reinterpret_cast<float4*>(m + p.off_rsegq);
  c->r_band = reinterpret_cast<uint32_t*>(m + p.off_rband);
  c->r_bandcnt = reinterpret_cast<int*>(m + p.off_rbandcnt);
  c->seg_cap = p.seg_cap;
  c->band_cap = p.band_cap;
  c->stage_bytes = p.stage_bytes;
  CUDA_TRY(c, cudaMemsetAsync(c->word, 0, (size_t)c->ncell_local * 4, c->st));
  CUDA_TRY(c, cudaMemsetAsync(c->tile_flag, 0, (size_t)c->ntiles, c->st));
  CUDA_TRY(c, cudaMemsetAsync(c->overflow, 0, (kMaxBodies + 1) * kSlotVals * 8, c->st));
  CUDA_TRY(c, cudaMemsetAsync(c->err, 0xFF, 8, c->st));
  CUDA_TRY(c, cudaMemsetAsync(c->flags, 0, 64, c->st));
  c->bound = true;
  return PSM_OK;
}

static psm_status ensure_pinned(psm_ctx* c) {
  if (c->pinned) return PSM_OK;
  if (cudaMallocHost(&c->pinned, (kMaxBodies + 2) * kSlotVals * 8) != cudaSuccess) {
    cudaGetLastError();
    c->pinned = nullptr;
    FAIL(c, PSM_E_OOM, "cudaMallocHost failed");
  }
  return PSM_OK;
}

static psm_status ensure_comm(psm_ctx* c) {
  // the communicator is created at the first device call, so psm_create stays host-only
  if (c->world == 1 || c->comm) return PSM_OK;
  ncclUniqueId id;
  static_assert(sizeof(id) == sizeof(c->nccl_id), "ncclUniqueId size");
  std::memcpy(&id, c->nccl_id, sizeof(id));
  NCCL_TRY(c, ncclCommInitRank(&c->comm, c->world, id, c->rank));
  // highest priority: NCCL's blocks are scheduled as soon as interior-collide blocks retire
  int lo_prio = 0, hi_prio = 0;
  CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  CUDA_TRY(c, cudaStreamCreateWithPriority(&c->comm_st, cudaStreamNonBlocking, hi_prio));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  return PSM_OK;
}

static psm_status ensure_mem(psm_ctx* c) {
  psm_status ps = ensure_pinned(c);
  if (ps != PSM_OK) return ps;
  ps = ensure_comm(c);
  if (ps != PSM_OK) return ps;
  if (c->bound) return PSM_OK;
  Plan p = make_plan(c);
  void* m = nullptr;
  if (cudaMalloc(&m, p.total) != cudaSuccess) {
    cudaGetLastError();
    FAIL(c, PSM_E_OOM, "cudaMalloc of " + std::to_string(p.total) + " bytes failed");
  }
  c->own_mem = true;
  return bind(c, m, p.total);
}

static psm_status halo(psm_ctx* c, void* arr, cudaStream_t hst) {
  // two-array pull: ship the c_z = +1 populations of the top plane up and the c_z = -1
  // populations of the bottom plane down, straight from/into the SoA planes (no packing)
  if (c->world == 1) return PSM_OK;
  const int P = c->world, r = c->rank;
  const bool zwall = c->grid.bc[2] == PSM_WALL;
  const int up = (r + 1) % P, down = (r - 1 + P) % P;
  const bool has_up = !(zwall && r == P - 1), has_down = !(zwall && r == 0);
  const size_t plane = (size_t)c->grid.nx * c->grid.ny;
  const ncclDataType_t dt = (c->opt.prec == PSM_F64) ? ncclFloat64 : ncclFloat32;
  char* base = static_cast<char*>(arr);
  auto ptr = [&](int q, int64_t zs) {
    return base + ((size_t)q * (size_t)c->geom.qstride + (size_t)zs * plane) * c->S;
  };
  NCCL_TRY(c, ncclGroupStart());
  for (int q = 0; q < c->Q; ++q) {
    const int cz = stc_z(q);
    if (cz > 0) {
      if (has_up) NCCL_TRY(c, ncclSend(ptr(q, c->nzl), plane, dt, up, c->comm, hst));
      if (has_down) NCCL_TRY(c, ncclRecv(ptr(q, 0), plane, dt, down, c->comm, hst));
    } else if (cz < 0) {
      if (has_down) NCCL_TRY(c, ncclSend(ptr(q, 1), plane, dt, down, c->comm, hst));
      if (has_up) NCCL_TRY(c, ncclRecv(ptr(q, c->nzl + 1), plane, dt, up, c->comm, hst));
    }
  }
  NCCL_TRY(c, ncclGroupEnd());
  return PSM_OK;
}

static void fill_kin(const psm_ctx* c, CollideParams& p, int64_t step) {
  for (int id = 0; id <= kMaxBodies; ++id) {
    BodyKin& k = p.bodies[id];
    std::memset(&k, 0, sizeof(k));
    const Body& b = c->bodies[id];
    if (!b.present) continue;
    double Q[9], t[3];
    pose_at(c, b, step, Q, t);
    (void)Q;
    (void)t;
    for (int a = 0; a < 3; ++a) {
      k.t[a] = b.ms.tc[a];  // pose of the current mapping (remapped before this collide)
      k.v[a] = b.dynamic ? b.vd[a] : b.v[a];
      k.w[a] = b.dynamic ? b.wd[a] : b.w[a];
    }
    k.s = b.s;
    k.present = 1;
  }
}

// Semi-implicit Euler step of a dynamic body with the force/torque ON it from the step just
// completed (the oracle implements the same formulas independently).
static void integrate_body(const psm_ctx* c, Body& b, const double F[3], const double T[3]) {
  for (int a = 0; a < 3; ++a) {
    b.dv[a] = (F[a] + b.fext[a] + b.Ma * b.dv[a]) / (b.mass + b.Ma);
    b.vd[a] = b.vd[a] + b.dv[a];
  }
  for (int a = 0; a < 3; ++a) {
    double x = b.td[a] + b.vd[a];
    if (c->grid.bc[a] == PSM_PERIODIC) {
      const double L = extent(c, a);
      x = x - L * std::floor(x / L);
    }
    b.td[a] = x;
  }
  // world-frame inertia I_w = Q I Q^T and virtual inertia A_w = Q I_a Q^T
  auto to_world = [&](const double* Ib, double* W) {
    double M[9];
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int l = 0; l < 3; ++l) acc += b.Qd[3 * r + l] * Ib[3 * l + cc];
        M[3 * r + cc] = acc;
      }
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int l = 0; l < 3; ++l) acc += M[3 * r + l] * b.Qd[3 * cc + l];
        W[3 * r + cc] = acc;
      }
  };
  double Iw[9], Aw[9];
  to_world(b.Ib, Iw);
  to_world(b.Ia, Aw);
  double Aw_dw[3];
  for (int r = 0; r < 3; ++r) {
    double acc = 0.0;
    for (int cc = 0; cc < 3; ++cc) acc += Aw[3 * r + cc] * b.dw[cc];
    Aw_dw[r] = acc;
  }
  for (int k = 0; k < 9; ++k) Iw[k] = Iw[k] + Aw[k];
  // dw = (I_w + A_w)^-1 (T + ext_torque + A_w dw_prev), by the adjugate
  const double A = Iw[0], B = Iw[1], C = Iw[2], D = Iw[3], E = Iw[4], Fm = Iw[5], G = Iw[6],
               H = Iw[7], I = Iw[8];
  const double adj[9] = {E * I - Fm * H, C * H - B * I, B * Fm - C * E,
                         Fm * G - D * I, A * I - C * G, C * D - A * Fm,
                         D * H - E * G, B * G - A * H, A * E - B * D};
  const double det = A * (E * I - Fm * H) - B * (D * I - Fm * G) + C * (D * H - E * G);
  const double tt[3] = {T[0] + b.text[0] + Aw_dw[0], T[1] + b.text[1] + Aw_dw[1],
                        T[2] + b.text[2] + Aw_dw[2]};
  for (int r = 0; r < 3; ++r) {
    double acc = 0.0;
    for (int cc = 0; cc < 3; ++cc) acc += adj[3 * r + cc] * tt[cc];
    b.dw[r] = acc / det;
  }
  for (int r = 0; r < 3; ++r) b.wd[r] = b.wd[r] + b.dw[r];
  double Qn[9];
  rodrigues(b.wd, 1.0, b.Qd, Qn);
  // Gram-Schmidt on the columns
  double c0[3] = {Qn[0], Qn[3], Qn[6]}, c1[3] = {Qn[1], Qn[4], Qn[7]};
  const double n0 = std::sqrt(c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2]);
  for (int a = 0; a < 3; ++a) c0[a] = c0[a] / n0;
  const double d01 = c0[0] * c1[0] + c0[1] * c1[1] + c0[2] * c1[2];
  for (int a = 0; a < 3; ++a) c1[a] = c1[a] - d01 * c0[a];
  const double n1 = std::sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
  for (int a = 0; a < 3; ++a) c1[a] = c1[a] / n1;
  const double c2[3] = {c0[1] * c1[2] - c0[2] * c1[1], c0[2] * c1[0] - c0[0] * c1[2],
                        c0[0] * c1[1] - c0[1] * c1[0]};
  for (int a = 0; a < 3; ++a) {
    b.Qd[3 * a + 0] = c0[a];
    b.Qd[3 * a + 1] = c1[a];
    b.Qd[3 * a + 2] = c2[a];
  }
}

static psm_status run_map(psm_ctx* c, const std::vector<Box>& boxes) {
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
  static const bool force_general = std::getenv("PSM_REMAP_GENERAL") != nullptr;
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
      CUDA_TRY(c, launch_remap_single(r, c->mst == c->st ? 148 * 8 : c->ahead_blocks, c->mst,
                                      c->mst == c->st ? 256 : c->ahead_threads));
      c->launches += 4;
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
static void swap_buffers(psm_ctx* c) {
  std::swap(c->word, c->word_alt);
  std::swap(c->tile_flag, c->tile_flag_alt);
  for (int id = 1; id <= kMaxBodies; ++id) std::swap(c->bodies[id].ms, c->bodies[id].alt);
}

static psm_status ensure_pipeline(psm_ctx* c) {
  if (c->map_st) return PSM_OK;
  int lo_prio = 0, hi_prio = 0;
  CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  CUDA_TRY(c, cudaStreamCreateWithPriority(&c->map_st, cudaStreamNonBlocking, hi_prio));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_map, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_coll, cudaEventDisableTiming));
  return PSM_OK;
}

// Upper bound on how far any point of body b moves between the band's build pose and (Q, t):
// |mi(t - t_rb)| + r_bound * |Q - Q_rb|_F / sqrt(2)  (the chord of a rotation by theta is
// 2 r sin(theta/2) = r |Q - Q_rb|_F / sqrt(2)).
static double band_displacement(const psm_ctx* c, const Body& b, const double Q[9],
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

static bool boxes_overlap(const psm_ctx* c, const Body& b, const std::vector<Box>& boxes) {
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
static psm_status remap(psm_ctx* c, const std::vector<int>& ids, int64_t step) {
  static const bool no_cache = [] {
    const char* e = std::getenv("PSM_BAND_CACHE");
    return e && std::strcmp(e, "0") == 0;
  }();
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
    // the cached band pays off while the exact pass is cheap (8 sub-samples per cell); at
    // s >= 2 the radius-2 band's 64/512 samples per cell cost more than the L0-L2 pipeline
    b.want_cache = !no_cache && !c->dbg && b.s <= 1;
    remap_region(c, b, Q, t, boxes);
  }
  // an incremental body whose (build) box meets a box remapped now goes the full way
  for (bool changed = true; changed;) {
    changed = false;
    for (size_t k = 0; k < incr.size(); ++k) {
      Body& b = c->bodies[incr[k]];
      if (!boxes_overlap(c, b, boxes)) continue;
      b.ms.cache = false;
      b.want_cache = b.s <= 1;
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
    CUDA_TRY(c, launch_remap_band(r, c->mst == c->st ? 148 * 8 : c->ahead_blocks, c->mst,
                                  c->mst == c->st ? 256 : c->ahead_threads));
    c->launches += (b.s >= 2 && b.mapping == 0) ? 2 : 1;
  }
  if (!incr.empty() && record(c, 0, 1, c->mst) != cudaSuccess)
    FAIL(c, PSM_E_CUDA, "event record failed");
  return PSM_OK;
}

static psm_status state_write(psm_ctx* c, const double* host, int mode) {
  // mode 0: f [Q][N] host; 1: rho/u host (rho or u may be NULL -> defaults); 2: uniform rest
  psm_status s = ensure_mem(c);
  if (s != PSM_OK) return s;
  const size_t plane = (size_t)c->grid.nx * c->grid.ny;
  const int nvals = mode == 0 ? c->Q : 4;
  const size_t per = plane * (size_t)nvals * 8;
  const int64_t cap = (int64_t)(c->stage_bytes / per);  // planes in staging
  const bool ghost = c->geom.zghost != 0;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(c->nzl, cap - 2));
  void* arr = c->A[c->opt.pattern == PSM_TWO_ARRAY ? c->cur : 0];
  std::vector<double> tmp;
  for (int64_t za = 0; za < c->nzl; za += chunk) {
    const int64_t zb = std::min<int64_t>(c->nzl, za + chunk);
    StateParams p{};
    p.g = c->geom;
    p.A = arr;
    p.stage = c->stage;
    p.za = (int)za;
    p.zb = (int)zb;
    p.pattern = c->opt.pattern == PSM_AA ? 1 : 0;
    p.mode = mode;
    p.ghosts = ghost ? 1 : 0;
    for (int a = 0; a < 3; ++a) p.u_in[a] = c->u_in[a];
    p.rho_out = c->rho_out;
    if (mode != 2) {
      // staging planes cover the readers of slots in [za, zb): local planes [za-1, zb+1)
      int64_t s0 = za - 1, s1 = zb + 1;
      if (ghost || c->opt.pattern == PSM_AA) {
        s0 = std::max<int64_t>(0, s0);
        s1 = std::min<int64_t>(c->nzl, s1);
      }
      if (!ghost && c->opt.pattern != PSM_AA && c->grid.bc[2] == PSM_WALL) {
        s0 = std::max<int64_t>(0, s0);
        s1 = std::min<int64_t>(c->nzl, s1);
      }
      int64_t ns = s1 - s0;
      if (ns > c->nzl) {  // small periodic grid: the whole slab once
        s0 = 0;
        ns = c->nzl;
      }
      p.stage_z0 = (int)s0;
      p.stage_nz = (int)ns;
      // gather host planes (wrapped) into a contiguous pinned-free host buffer, then H2D
      tmp.assign((size_t)(ns * plane * nvals), 0.0);
      const size_t N = (size_t)c->nzl * plane;
      if (mode == 0)
        for (int v = 0; v < nvals; ++v)
          for (int64_t k = 0; k < ns; ++k) {
            const int64_t zl = ((s0 + k) % c->nzl + c->nzl) % c->nzl;
            std::memcpy(&tmp[((size_t)v * ns + k) * plane], host + (size_t)v * N + (size_t)zl * plane,
                        plane * 8);
          }
      if (mode == 1) {
        // host points to a 2-element array {rho, u} packed by the caller
        const double* const* ru = reinterpret_cast<const double* const*>(host);
        for (int64_t k = 0; k < ns; ++k) {
          const int64_t zl = ((s0 + k) % c->nzl + c->nzl) % c->nzl;
          for (size_t i = 0; i < plane; ++i) {
            const size_t src = (size_t)zl * plane + i;
            tmp[((size_t)0 * ns + k) * plane + i] = ru[0] ? ru[0][src] : 1.0;
            for (int a = 0; a < 3; ++a)
              tmp[((size_t)(a + 1) * ns + k) * plane + i] = ru[1] ? ru[1][a * N + src] : 0.0;
          }
        }
      }
      CUDA_TRY(c, cudaMemcpyAsync(c->stage, tmp.data(), tmp.size() * 8, cudaMemcpyHostToDevice,
                                  c->st));
    }
    CUDA_TRY(c, launch_write_state(c->Q, c->opt.prec == PSM_F64, p, c->st));
    c->launches += 1;
    CUDA_TRY(c, cudaStreamSynchronize(c->st));  // tmp is reused by the next chunk
  }
  c->step = 0;
  c->ft_valid = false;
  return PSM_OK;
}

static psm_status state_read(psm_ctx* c, double* f, double* rho, double* u, int64_t zbeg = 0,
                             int64_t zend = -1) {
  psm_status s = ensure_mem(c);
  if (s != PSM_OK) return s;
  if (zend < 0) zend = c->nzl;
  const size_t plane = (size_t)c->grid.nx * c->grid.ny;
  const int mode = f ? 0 : 1;
  const int nvals = mode == 0 ? c->Q : 4;
  const size_t per = plane * (size_t)nvals * 8;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(c->nzl,
                                                              (int64_t)(c->stage_bytes / per)));
  const void* arr = (c->opt.pattern == PSM_TWO_ARRAY) ? c->A[c->cur] : c->A[0];
  const size_t N = (size_t)(zend - zbeg) * plane;
  std::vector<double> tmp;
  for (int64_t za = zbeg; za < zend; za += chunk) {
    const int64_t zb = std::min<int64_t>(zend, za + chunk);
    StateParams p{};
    p.g = c->geom;
    p.A = const_cast<void*>(arr);
    p.stage = c->stage;
    p.za = (int)za;
    p.zb = (int)zb;
    p.stage_z0 = (int)za;
    p.stage_nz = (int)(zb - za);
    for (int a = 0; a < 3; ++a) p.u_in[a] = c->u_in[a];
    p.rho_out = c->rho_out;
    p.pattern = c->opt.pattern == PSM_AA ? 1 : 0;
    p.odd = (int)(c->step & 1);
    p.mode = mode;
    CUDA_TRY(c, launch_read_state(c->Q, c->opt.prec == PSM_F64, p, c->st));
    c->launches += 1;
    const size_t nz = (size_t)(zb - za);
    tmp.resize(nz * plane * nvals);
    CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), c->stage, tmp.size() * 8, cudaMemcpyDeviceToHost,
                                c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    for (int v = 0; v < nvals; ++v) {
      const double* src = &tmp[(size_t)v * nz * plane];
      const size_t o = (size_t)(za - zbeg) * plane;
      if (mode == 0) {
        std::memcpy(f + (size_t)v * N + o, src, nz * plane * 8);
      } else if (v == 0) {
        if (rho) std::memcpy(rho + o, src, nz * plane * 8);
      } else if (u) {
        std::memcpy(u + (size_t)(v - 1) * N + o, src, nz * plane * 8);
      }
    }
  }
  return PSM_OK;
}

// ----------------------------------------------------------------------------- ABI --------
// Enqueue the per-body force/torque reduction of the step just collided (two deterministic
// passes, allreduce over ranks) and its D2H copy into the pinned buffer; ids receives the body
// order of the copied rows.  The caller synchronises.
static psm_status ft_enqueue(psm_ctx* c, std::vector<int>& ids) {
  ids.clear();
  for (int id = 1; id <= kMaxBodies; ++id)
    if (c->bodies[id].present || c->dbg) ids.push_back(id);
  const int nb = (int)ids.size();
  if (nb == 0) return PSM_OK;
  int* hid = reinterpret_cast<int*>(c->pinned + kMaxBodies * kSlotVals);
  for (int i = 0; i < nb; ++i) hid[i] = ids[i];
  CUDA_TRY(c, cudaMemcpyAsync(c->ft_ids, hid, nb * 4, cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(c, launch_ft_reduce(c->tile_flag, c->partial, (int)c->ntiles, c->overflow, c->ft_ids,
                               nb, c->ft_scratch, kFtChunks, c->ft_out, c->st));
  c->launches += 2;
  if (c->world > 1)
    NCCL_TRY(c, ncclAllReduce(c->ft_out, c->ft_out, (size_t)nb * kSlotVals, ncclFloat64, ncclSum,
                              c->comm, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(c->pinned, c->ft_out, (size_t)nb * kSlotVals * 8,
                              cudaMemcpyDeviceToHost, c->st));
  return PSM_OK;
}

static void ft_store(psm_ctx* c, const std::vector<int>& ids) {
  std::memset(c->ft, 0, sizeof(c->ft));
  for (size_t i = 0; i < ids.size(); ++i)
    std::memcpy(c->ft[ids[i]], c->pinned + i * kSlotVals, kSlotVals * 8);
  c->ft_valid = true;
}

extern "C" {

psm_status psm_create(const psm_grid* grid, psm_stencil stencil, double tau,
                      const psm_options* opt, psm_ctx** out) {
  if (!grid || !opt || !out) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  *out = nullptr;
  if (!(tau > 0.5) || !std::isfinite(tau))
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "tau must be finite and > 1/2 (Eq.(2): nu = (tau-1/2)/3)");
  if (stencil != PSM_D3Q19 && stencil != PSM_D3Q27)
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "stencil must be 19 or 27");
  if (grid->nx < 1 || grid->ny < 1 || grid->nz < 1)
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "grid extents must be >= 1");
  for (int a = 0; a < 3; ++a)
    if (grid->bc[a] != PSM_PERIODIC && grid->bc[a] != PSM_WALL && grid->bc[a] != PSM_INOUT)
      FAIL((psm_ctx*)nullptr, PSM_E_ARG, "bad boundary kind");
  if (grid->bc[1] == PSM_INOUT || grid->bc[2] == PSM_INOUT)
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED, "inflow/outflow boundaries are on the x axis only");
  if (grid->bc[0] == PSM_INOUT && (grid->nx < 3 || opt->pattern != PSM_TWO_ARRAY))
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED,
         "inflow/outflow boundaries need nx >= 3 and PSM_TWO_ARRAY");
  if ((opt->prec != PSM_F64 && opt->prec != PSM_F32) ||
      (opt->pattern != PSM_TWO_ARRAY && opt->pattern != PSM_AA) || opt->sc < 1 || opt->sc > 3 ||
      (opt->bmode != PSM_B_DIRECT && opt->bmode != PSM_B_WEIGHTED) ||
      (opt->collision != PSM_SRT && opt->collision != PSM_TRT && opt->collision != PSM_CUMULANT))
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "bad option enum");
  if (opt->collision == PSM_TRT && !(opt->trt_magic > 0.0 && std::isfinite(opt->trt_magic)))
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "TRT magic parameter must be finite and > 0");
  const int world = opt->world < 1 ? 1 : opt->world;
  if (opt->rank < 0 || opt->rank >= world) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "bad rank");
  if (grid->nz < world) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "nz < world");
  const bool force = opt->body_force[0] != 0.0 || opt->body_force[1] != 0.0 ||
                     opt->body_force[2] != 0.0;
  if (force && opt->pattern == PSM_AA)
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED, "body force needs PSM_TWO_ARRAY");
  if (world > 1 && opt->pattern == PSM_AA)
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED, "multi-rank runs need PSM_TWO_ARRAY");
  if (opt->collision == PSM_CUMULANT && (stencil != PSM_D3Q27 || force))
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED, "the cumulant operator needs D3Q27 and no body force");
  if (world > 1 && !opt->nccl_unique_id)
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "world > 1 needs an ncclUniqueId");
  psm_ctx* c = new (std::nothrow) psm_ctx();
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_OOM, "host allocation failed");
  c->grid = *grid;
  c->Q = (int)stencil;
  c->tau = tau;
  c->opt = *opt;
  c->rank = opt->rank;
  c->world = world;
  c->S = opt->prec == PSM_F64 ? 8 : 4;
  c->z0 = (grid->nz * c->rank) / world;
  c->nzl = (grid->nz * (c->rank + 1)) / world - c->z0;
  c->st = static_cast<cudaStream_t>(opt->cuda_stream);
  c->mst = c->st;
  if (const char* e = std::getenv("PSM_AHEAD_BLOCKS")) c->ahead_blocks = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PSM_AHEAD_THREADS"))
    c->ahead_threads = std::min(1024, std::max(32, std::atoi(e)));
  Geom& g = c->geom;
  g.nx = (int)grid->nx;
  g.ny = (int)grid->ny;
  g.nzl = (int)c->nzl;
  g.nz_global = (int)grid->nz;
  g.z0 = (int)c->z0;
  g.zghost = world > 1 ? 1 : 0;
  // wall[a]: the axis is not periodic (half-way bounce-back sources; A30 patches the x faces)
  for (int a = 0; a < 3; ++a) g.wall[a] = grid->bc[a] != PSM_PERIODIC;
  g.open_x = grid->bc[0] == PSM_INOUT;
  g.qstride = (long long)(c->nzl + 2 * g.zghost) * grid->ny * grid->nx;
  g.gx = (int)((grid->nx + kTileX - 1) / kTileX);
  g.gy = (int)((grid->ny + kTileY - 1) / kTileY);
  g.gz = (int)((c->nzl + kTileZ - 1) / kTileZ);
  if (g.qstride >= (1ll << 31) || grid->nx >= (1 << 30) || grid->ny > 65535 * kTileY ||
      c->nzl > 65535 * kTileZ) {
    delete c;
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "local slab too large for 32-bit in-plane indexing");
  }
  c->ncell_local = (int64_t)c->nzl * grid->ny * grid->nx;
  c->ntiles = (int64_t)g.gx * g.gy * g.gz;
  if (world > 1) std::memcpy(c->nccl_id, opt->nccl_unique_id, sizeof(c->nccl_id));
  *out = c;
  return PSM_OK;
}

psm_status psm_destroy(psm_ctx* c) {
  if (!c) return PSM_OK;
  cudaStreamSynchronize(c->st);
  if (c->map_st) cudaStreamSynchronize(c->map_st);
  for (int id = 0; id <= kMaxBodies; ++id) {
    cudaFree(c->bodies[id].d_bits);
    cudaFree(c->bodies[id].d_mask);
    free_bands(c->bodies[id]);
  }
  cudaFree(c->dbg_B);
  cudaFree(c->dbg_us);
  cudaFree(c->dbg_id);
  if (c->own_mem) cudaFree(c->mem);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (int ph = 0; ph < PSM_NUM_PHASES; ++ph)
    for (auto& e : c->ev[ph]) {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  if (c->ipc_up) cudaIpcCloseMemHandle(c->ipc_up);
  if (c->ipc_dn && c->ipc_dn != c->ipc_up) cudaIpcCloseMemHandle(c->ipc_dn);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_st) cudaStreamDestroy(c->comm_st);
  if (c->ev_bnd) cudaEventDestroy(c->ev_bnd);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->map_st) cudaStreamDestroy(c->map_st);
  if (c->ev_map) cudaEventDestroy(c->ev_map);
  if (c->ev_coll) cudaEventDestroy(c->ev_coll);
  delete c;
  return PSM_OK;
}

psm_status psm_required_bytes(const psm_ctx* c, size_t* bytes) {
  if (!c || !bytes) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  *bytes = make_plan(c).total;
  return PSM_OK;
}

psm_status psm_bind_memory(psm_ctx* c, void* dev_ptr, size_t bytes) {
  if (!c || !dev_ptr) FAIL(c, PSM_E_ARG, "null argument");
  if (c->bound) FAIL(c, PSM_E_STATE, "memory already bound");
  if (reinterpret_cast<uintptr_t>(dev_ptr) & 255) FAIL(c, PSM_E_ARG, "dev_ptr not 256-aligned");
  return bind(c, dev_ptr, bytes);
}

psm_status psm_local_extent(const psm_ctx* c, int64_t* z0, int64_t* nz_local) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (z0) *z0 = c->z0;
  if (nz_local) *nz_local = c->nzl;
  return PSM_OK;
}

psm_status psm_init_equilibrium(psm_ctx* c, const double* rho, const double* u) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (!rho && !u) return state_write(c, nullptr, 2);
  const double* ru[2] = {rho, u};
  return state_write(c, reinterpret_cast<const double*>(ru), 1);
}

psm_status psm_write_pdfs(psm_ctx* c, const double* f) {
  if (!c || !f) FAIL(c, PSM_E_ARG, "null argument");
  return state_write(c, f, 0);
}

psm_status psm_read_pdfs(psm_ctx* c, double* f) {
  if (!c || !f) FAIL(c, PSM_E_ARG, "null argument");
  return state_read(c, f, nullptr, nullptr);
}

psm_status psm_read_pdfs_planes(psm_ctx* c, int64_t z_begin, int64_t nz, double* f) {
  if (!c || !f) FAIL(c, PSM_E_ARG, "null argument");
  if (z_begin < 0 || nz < 1 || z_begin + nz > c->nzl) FAIL(c, PSM_E_ARG, "plane range outside the slab");
  return state_read(c, f, nullptr, nullptr, z_begin, z_begin + nz);
}

psm_status psm_read_velocity(psm_ctx* c, double* rho, double* u) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (!rho && !u) return PSM_OK;
  return state_read(c, nullptr, rho, u);
}

psm_status psm_set_body(psm_ctx* c, int32_t id, const psm_shape* shape, const psm_pose* pose,
                        const psm_velocity* vel) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (id < 1 || id > kMaxBodies) FAIL(c, PSM_E_ARG, "body id must be in 1..16");
  psm_status st = ensure_mem(c);
  if (st != PSM_OK) return st;
  Body& b = c->bodies[id];
  if (!shape && !b.present) FAIL(c, PSM_E_ARG, "new body needs a shape");
  if (!pose) FAIL(c, PSM_E_ARG, "pose required");
  // pose validation: orthonormal, det = +1
  const double* Q = pose->Q;
  double dev = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) {
      double acc = 0.0;
      for (int l = 0; l < 3; ++l) acc += Q[3 * l + r] * Q[3 * l + cc];
      dev = std::max(dev, std::fabs(acc - (r == cc ? 1.0 : 0.0)));
    }
  const double det = Q[0] * (Q[4] * Q[8] - Q[5] * Q[7]) - Q[1] * (Q[3] * Q[8] - Q[5] * Q[6]) +
                     Q[2] * (Q[3] * Q[7] - Q[4] * Q[6]);
  if (!(dev <= 1e-9) || !(det > 0.0)) FAIL(c, PSM_E_POSE, "pose matrix is not a rotation");
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(pose->t[a])) FAIL(c, PSM_E_POSE, "non-finite translation");
  if (shape) {
    if (shape->s < 0 || shape->s > 3) FAIL(c, PSM_E_ARG, "s must be in 0..3");
    Body nb;
    nb.kind = shape->kind;
    nb.s = shape->s;
    if (shape->mapping != PSM_MAP_R1 && shape->mapping != PSM_MAP_R2)
      FAIL(c, PSM_E_ARG, "unknown mapping mode");
    nb.mapping = shape->kind == PSM_MESH ? shape->mapping : PSM_MAP_R1;
    if (shape->kind == PSM_SPHERE) {
      if (!(shape->radius > 0.0) || !std::isfinite(shape->radius))
        FAIL(c, PSM_E_ARG, "sphere radius must be > 0");
      nb.radius = shape->radius;
      nb.rbound = shape->radius;
      for (int a = 0; a < 3; ++a) {
        nb.bmin[a] = -shape->radius;
        nb.bmax[a] = shape->radius;
      }
    } else if (shape->kind == PSM_MESH) {
      std::string why;
      if (!shape->verts || !shape->tris ||
          check_mesh(shape->verts, shape->nverts, shape->tris, shape->ntris, &why) != 0)
        FAIL(c, PSM_E_MESH, why.empty() ? std::string("null mesh arrays") : why);
      geometry_extent(shape->verts, shape->nverts, shape->s, nb.o, nb.dims);
      const double bits = (double)nb.dims[0] * nb.dims[1] * nb.dims[2] * std::ldexp(1.0, 3 * shape->s);
      if (bits / 8.0 > (double)kGeomCapBytes)
        FAIL(c, PSM_E_OOM, "geometry field exceeds the 1 GiB cap (reduce s)");
      double rb = 0.0;
      for (int a = 0; a < 3; ++a) {
        nb.bmin[a] = shape->verts[a];
        nb.bmax[a] = shape->verts[a];
      }
      for (int64_t k = 0; k < shape->nverts; ++k) {
        const double* v = shape->verts + 3 * k;
        rb = std::max(rb, std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]));
        for (int a = 0; a < 3; ++a) {
          nb.bmin[a] = std::min(nb.bmin[a], v[a]);
          nb.bmax[a] = std::max(nb.bmax[a], v[a]);
        }
      }
      nb.rbound = rb;
      // geometry field (reading A15/A17): GPU voxeliser by default (k_voxelize.cu); the host
      // implementation with PSM_VOXELIZE=host; PSM_VOXELIZE_CHECK=1 runs both and compares
      const int sl = shape->s, n = 1 << sl;
      const size_t nbk = (size_t)(nb.dims[0] * nb.dims[1] * nb.dims[2]);
      nb.words = std::max(1, (n * n * n) / 64);
      CUDA_TRY(c, cudaMalloc(&nb.d_bits, nbk * nb.words * 8));
      CUDA_TRY(c, cudaMalloc(&nb.d_mask, nbk));
      const char* vx = std::getenv("PSM_VOXELIZE");
      const bool host_vox = vx && std::strcmp(vx, "host") == 0;
      const bool check = std::getenv("PSM_VOXELIZE_CHECK") != nullptr;
      if (!host_vox) {
        std::vector<long long> V((size_t)(3 * shape->nverts));
        const double sc = std::ldexp(1.0, sl + 12);
        for (int64_t k = 0; k < shape->nverts; ++k)
          for (int a = 0; a < 3; ++a)
            V[3 * k + a] = std::llround((shape->verts[3 * k + a] - nb.o[a]) * sc);
        VoxParams vp;
        std::memset(&vp, 0, sizeof(vp));
        vp.nt = shape->ntris;
        vp.s = sl;
        vp.bx = nb.dims[0];
        vp.by = nb.dims[1];
        vp.bz = nb.dims[2];
        vp.NX = vp.bx << sl;
        vp.NY = vp.by << sl;
        vp.NZ = vp.bz << sl;
        vp.W = nb.words;
        vp.words = nb.d_bits;
        vp.wpr = (vp.NX + 1 + 31) / 32;
        long long* dV = nullptr;
        int* dT = nullptr;
        void* scratch = nullptr;
        const size_t sbytes = voxelize_scratch_bytes(vp);
        CUDA_TRY(c, cudaMalloc(&dV, V.size() * 8));
        CUDA_TRY(c, cudaMalloc(&dT, (size_t)shape->ntris * 12));
        CUDA_TRY(c, cudaMalloc(&scratch, sbytes));
        CUDA_TRY(c, cudaMemcpyAsync(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice, c->st));
        CUDA_TRY(c, cudaMemcpyAsync(dT, shape->tris, (size_t)shape->ntris * 12,
                                    cudaMemcpyHostToDevice, c->st));
        vp.V = dV;
        vp.tris = dT;
        CUDA_TRY(c, launch_voxelize(vp, scratch, nb.d_mask, c->st));
        c->launches += 6 + 18 + 1;
        CUDA_TRY(c, cudaStreamSynchronize(c->st));
        cudaFree(dV);
        cudaFree(dT);
        cudaFree(scratch);
      }
      if (host_vox || check) {
        std::vector<uint8_t> field, mask;
        std::vector<unsigned long long> words;
        voxelize_mesh(shape->verts, shape->nverts, shape->tris, shape->ntris, sl, nb.o,
                      nb.dims, field);
        int W = 0;
        pack_bricks(field, sl, nb.dims, words, mask, &W);
        if (host_vox) {
          CUDA_TRY(c, cudaMemcpy(nb.d_bits, words.data(), words.size() * 8,
                                 cudaMemcpyHostToDevice));
          CUDA_TRY(c, cudaMemcpy(nb.d_mask, mask.data(), mask.size(), cudaMemcpyHostToDevice));
        } else {
          std::vector<unsigned long long> gw(words.size());
          std::vector<uint8_t> gm(mask.size());
          CUDA_TRY(c, cudaMemcpy(gw.data(), nb.d_bits, gw.size() * 8, cudaMemcpyDeviceToHost));
          CUDA_TRY(c, cudaMemcpy(gm.data(), nb.d_mask, gm.size(), cudaMemcpyDeviceToHost));
          if (gw != words || gm != mask) {
            cudaFree(nb.d_bits);
            cudaFree(nb.d_mask);
            FAIL(c, PSM_E_STATE, "PSM_VOXELIZE_CHECK: GPU and host voxelisers differ");
          }
        }
      }
    } else {
      FAIL(c, PSM_E_ARG, "unknown shape kind");
    }
    for (int a = 0; a < 3; ++a)
      if (c->grid.bc[a] == PSM_PERIODIC && nb.rbound + 1.0 >= 0.5 * extent(c, a))
        FAIL(c, PSM_E_ARG, "body bounding radius + 1 must be < half a periodic extent");
    // keep the previous mapped box so the old footprint gets cleared
    nb.ms.has_box = b.ms.has_box;
    for (int a = 0; a < 3; ++a) {
      nb.ms.box_lo[a] = b.ms.box_lo[a];
      nb.ms.box_hi[a] = b.ms.box_hi[a];
    }
    cudaStreamSynchronize(c->st);
    cudaFree(b.d_bits);
    cudaFree(b.d_mask);
    free_bands(b);
    b = nb;
  }
  b.present = true;
  std::memcpy(b.Q0, pose->Q, sizeof(b.Q0));
  std::memcpy(b.t0, pose->t, sizeof(b.t0));
  for (int a = 0; a < 3; ++a) {
    b.v[a] = vel ? vel->v[a] : 0.0;
    b.w[a] = vel ? vel->omega[a] : 0.0;
  }
  b.moving = false;
  for (int a = 0; a < 3; ++a)
    if (b.v[a] != 0.0 || b.w[a] != 0.0) b.moving = true;
  b.step0 = c->step;
  if (b.dynamic) {  // new initial state of a dynamic body
    b.moving = true;
    for (int a = 0; a < 3; ++a) b.dv[a] = b.dw[a] = 0.0;
    std::memcpy(b.Qd, b.Q0, sizeof(b.Qd));
    std::memcpy(b.td, b.t0, sizeof(b.td));
    std::memcpy(b.vd, b.v, sizeof(b.vd));
    std::memcpy(b.wd, b.w, sizeof(b.wd));
  }
  c->ft_valid = false;
  c->alt_valid = false;  // the spare word buffer no longer matches the bodies
  // (a pose change keeps the cached band: remap() checks the displacement bound itself)
  return remap(c, std::vector<int>{id}, c->step);
}

psm_status psm_voxelize(const double* verts, int64_t nverts, const int32_t* tris, int64_t ntris,
                        int32_t s, double origin[3], int64_t dims[3], uint8_t* bits) {
  if (!verts || !tris || !origin || !dims) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  if (s < 0 || s > 3) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "s must be in 0..3");
  std::string why;
  if (check_mesh(verts, nverts, tris, ntris, &why) != 0) FAIL((psm_ctx*)nullptr, PSM_E_MESH, why);
  int64_t cells[3];
  geometry_extent(verts, nverts, s, origin, cells);
  for (int a = 0; a < 3; ++a) dims[a] = cells[a] << s;
  if (bits) {
    std::vector<uint8_t> field;
    voxelize_mesh(verts, nverts, tris, ntris, s, origin, cells, field);
    std::memcpy(bits, field.data(), field.size());
  }
  return PSM_OK;
}

psm_status psm_set_open_boundary(psm_ctx* c, const double u_in[3], double rho_out) {
  if (!c || !u_in) FAIL(c, PSM_E_ARG, "null argument");
  if (c->grid.bc[0] != PSM_INOUT) FAIL(c, PSM_E_UNSUPPORTED, "bc[0] is not PSM_INOUT");
  if (!(std::isfinite(rho_out) && rho_out > 0.0) || !std::isfinite(u_in[0]) ||
      !std::isfinite(u_in[1]) || !std::isfinite(u_in[2]))
    FAIL(c, PSM_E_ARG, "u_in must be finite, rho_out finite and > 0");
  for (int a = 0; a < 3; ++a) c->u_in[a] = u_in[a];
  c->rho_out = rho_out;
  return PSM_OK;
}

psm_status psm_set_dynamics(psm_ctx* c, int32_t id, const psm_dynamics* d) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (id < 1 || id > kMaxBodies || !c->bodies[id].present) FAIL(c, PSM_E_ARG, "unknown body");
  Body& b = c->bodies[id];
  if (!d) {  // back to prescribed motion from the current state
    if (b.dynamic) {
      std::memcpy(b.Q0, b.Qd, sizeof(b.Q0));
      std::memcpy(b.t0, b.td, sizeof(b.t0));
      std::memcpy(b.v, b.vd, sizeof(b.v));
      std::memcpy(b.w, b.wd, sizeof(b.w));
      b.step0 = c->step;
      b.dynamic = false;
      b.moving = false;
      for (int a = 0; a < 3; ++a)
        if (b.v[a] != 0.0 || b.w[a] != 0.0) b.moving = true;
    }
    return PSM_OK;
  }
  if (!(d->mass > 0.0) || !std::isfinite(d->mass)) FAIL(c, PSM_E_ARG, "mass must be > 0");
  const double* I = d->inertia;
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc)
      if (!std::isfinite(I[3 * r + cc]) || std::fabs(I[3 * r + cc] - I[3 * cc + r]) >
                                               1e-12 * (std::fabs(I[0]) + std::fabs(I[4]) + std::fabs(I[8])))
        FAIL(c, PSM_E_ARG, "inertia tensor must be symmetric and finite");
  const double m1 = I[0], m2 = I[0] * I[4] - I[1] * I[3];
  const double m3 = I[0] * (I[4] * I[8] - I[5] * I[7]) - I[1] * (I[3] * I[8] - I[5] * I[6]) +
                    I[2] * (I[3] * I[7] - I[4] * I[6]);
  if (!(m1 > 0 && m2 > 0 && m3 > 0)) FAIL(c, PSM_E_ARG, "inertia tensor must be positive definite");
  // current state becomes the initial dynamic state
  if (!b.dynamic) {
    double Q[9], t[3];
    if (b.moving) pose_at(c, b, c->step, Q, t);
    else {
      std::memcpy(Q, b.Q0, sizeof(Q));
      std::memcpy(t, b.t0, sizeof(t));
    }
    std::memcpy(b.Qd, Q, sizeof(Q));
    std::memcpy(b.td, t, sizeof(t));
    std::memcpy(b.vd, b.v, sizeof(b.vd));
    std::memcpy(b.wd, b.w, sizeof(b.wd));
    for (int a = 0; a < 3; ++a) b.dv[a] = b.dw[a] = 0.0;
  }
  if (!(d->added_mass >= 0.0) || !std::isfinite(d->added_mass))
    FAIL(c, PSM_E_ARG, "added mass must be finite and >= 0");
  for (int r = 0; r < 3; ++r) {
    if (!(d->added_inertia[4 * r] >= 0.0)) FAIL(c, PSM_E_ARG, "added inertia must be >= 0");
    for (int cc = 0; cc < 3; ++cc)
      if (!std::isfinite(d->added_inertia[3 * r + cc]) ||
          d->added_inertia[3 * r + cc] != d->added_inertia[3 * cc + r])
        FAIL(c, PSM_E_ARG, "added inertia must be symmetric and finite");
  }
  b.dynamic = true;
  b.moving = true;
  b.mass = d->mass;
  b.Ma = d->added_mass;
  std::memcpy(b.Ia, d->added_inertia, sizeof(b.Ia));
  std::memcpy(b.Ib, d->inertia, sizeof(b.Ib));
  std::memcpy(b.fext, d->ext_force, sizeof(b.fext));
  std::memcpy(b.text, d->ext_torque, sizeof(b.text));
  return PSM_OK;
}

psm_status psm_get_body_state(const psm_ctx* c, int32_t id, psm_pose* pose, psm_velocity* vel) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (id < 1 || id > kMaxBodies || !c->bodies[id].present)
    FAIL((psm_ctx*)nullptr, PSM_E_ARG, "unknown body");
  const Body& b = c->bodies[id];
  double Q[9], t[3], v[3], w[3];
  if (b.dynamic) {
    std::memcpy(Q, b.Qd, sizeof(Q));
    std::memcpy(t, b.td, sizeof(t));
    std::memcpy(v, b.vd, sizeof(v));
    std::memcpy(w, b.wd, sizeof(w));
  } else {
    if (b.moving) pose_at(c, b, c->step, Q, t);
    else {
      std::memcpy(Q, b.Q0, sizeof(Q));
      std::memcpy(t, b.t0, sizeof(t));
    }
    std::memcpy(v, b.v, sizeof(v));
    std::memcpy(w, b.w, sizeof(w));
  }
  if (pose) {
    std::memcpy(pose->Q, Q, sizeof(Q));
    std::memcpy(pose->t, t, sizeof(t));
  }
  if (vel) {
    std::memcpy(vel->v, v, sizeof(v));
    std::memcpy(vel->omega, w, sizeof(w));
  }
  return PSM_OK;
}

psm_status psm_remove_body(psm_ctx* c, int32_t id) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (id < 1 || id > kMaxBodies) FAIL(c, PSM_E_ARG, "body id must be in 1..16");
  Body& b = c->bodies[id];
  if (!b.present) return PSM_OK;
  std::vector<Box> boxes;
  if (b.ms.has_box) add_box(c, b.ms.box_lo, b.ms.box_hi, boxes);
  cudaStreamSynchronize(c->st);
  cudaFree(b.d_bits);
  cudaFree(b.d_mask);
  free_bands(b);
  b = Body();
  c->alt_valid = false;
  return run_map(c, boxes);
}

psm_status psm_map_fractions(psm_ctx* c) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  psm_status st = ensure_mem(c);
  if (st != PSM_OK) return st;
  std::vector<int> ids;
  for (int id = 1; id <= kMaxBodies; ++id)
    if (c->bodies[id].present) ids.push_back(id);
  return remap(c, ids, c->step);
}

// Fused halo setup (collective over the ranks, once): exchange CUDA IPC handles of every rank's
// device memory through NCCL, check peer access to both z neighbours on every rank, open the
// neighbours' memory.  Any failure anywhere keeps the NCCL send/recv halo on all ranks.
struct P2PInfo {
  cudaIpcMemHandle_t h;
  unsigned long long off_A0, off_A1, off_flags;
  long long nzl, qstride;
  int dev, ok;
};

static psm_status ensure_p2p(psm_ctx* c) {
  if (c->p2p_checked) return PSM_OK;
  c->p2p_checked = true;
  if (c->world == 1 || c->opt.pattern != PSM_TWO_ARRAY) return PSM_OK;
  const char* env = std::getenv("PSM_HALO");
  const bool want = !(env && std::strcmp(env, "nccl") == 0);
  const int P = c->world, r = c->rank;
  const bool zwall = c->grid.bc[2] == PSM_WALL;
  const int up = (r + 1) % P, dn = (r - 1 + P) % P;
  c->has_up = !(zwall && r == P - 1);
  c->has_dn = !(zwall && r == 0);
  P2PInfo mine;
  std::memset(&mine, 0, sizeof(mine));
  CUDA_TRY(c, cudaGetDevice(&mine.dev));
  // base of the allocation that holds the context memory (it may be a sub-block of a caller's
  // allocation, psm_bind_memory): driver cuMemGetAddressRange through the runtime entry point
  unsigned long long base = 0;
  size_t size = 0;
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (want && cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) ==
                  cudaSuccess && fn && q == cudaDriverEntryPointSuccess &&
      reinterpret_cast<GetRange>(fn)(&base, &size, (unsigned long long)c->mem) == 0 &&
      cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    const unsigned long long m = (unsigned long long)c->mem;
    mine.off_A0 = (unsigned long long)c->A[0] - base;
    mine.off_A1 = (unsigned long long)c->A[1] - base;
    mine.off_flags = (unsigned long long)c->flags - base;
    (void)m;
    mine.ok = 1;
  }
  cudaGetLastError();
  mine.nzl = c->nzl;
  mine.qstride = c->geom.qstride;
  std::vector<P2PInfo> all(P);
  char* d = nullptr;
  CUDA_TRY(c, cudaMalloc(&d, sizeof(P2PInfo) * (P + 1)));
  CUDA_TRY(c, cudaMemcpyAsync(d, &mine, sizeof(mine), cudaMemcpyHostToDevice, c->st));
  NCCL_TRY(c, ncclAllGather(d, d + sizeof(P2PInfo), sizeof(P2PInfo), ncclChar, c->comm, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(all.data(), d + sizeof(P2PInfo), sizeof(P2PInfo) * P,
                              cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  // every rank must be able to reach both its neighbours
  int ok = 1;
  for (int k = 0; k < P; ++k) ok &= all[k].ok;
  if (ok) {
    for (int nb : {up, dn}) {
      if (nb == r) continue;
      int can = 0;
      if (all[nb].dev == mine.dev) can = 1;  // same device (two ranks on one GPU): IPC works
      else if (cudaDeviceCanAccessPeer(&can, mine.dev, all[nb].dev) != cudaSuccess) can = 0;
      ok &= can;
    }
  }
  int* dok = reinterpret_cast<int*>(d);
  CUDA_TRY(c, cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, c->st));
  NCCL_TRY(c, ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  cudaFree(d);
  if (!ok || up == r) return PSM_OK;
  auto open = [&](int nb, void** out) -> bool {
    if (cudaIpcOpenMemHandle(out, all[nb].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      *out = nullptr;
      return false;
    }
    return true;
  };
  bool good = true;
  if (c->has_up) good &= open(up, &c->ipc_up);
  if (c->has_dn) {
    if (dn == up && c->has_up) c->ipc_dn = c->ipc_up;
    else good &= open(dn, &c->ipc_dn);
  }
  // all ranks must agree again (an open can fail)
  int g = good ? 1 : 0;
  CUDA_TRY(c, cudaMalloc(&dok, sizeof(int)));
  CUDA_TRY(c, cudaMemcpyAsync(dok, &g, sizeof(int), cudaMemcpyHostToDevice, c->st));
  NCCL_TRY(c, ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(&g, dok, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  cudaFree(dok);
  if (!g) return PSM_OK;  // (opened handles are closed in psm_destroy)
  if (c->has_up) {
    char* b = static_cast<char*>(c->ipc_up);
    c->up_A[0] = b + all[up].off_A0;
    c->up_A[1] = b + all[up].off_A1;
    c->up_qs = all[up].qstride;
    c->up_flag = reinterpret_cast<unsigned long long*>(b + all[up].off_flags) + 0;
  }
  if (c->has_dn) {
    char* b = static_cast<char*>(c->ipc_dn);
    c->dn_A[0] = b + all[dn].off_A0;
    c->dn_A[1] = b + all[dn].off_A1;
    c->dn_qs = all[dn].qstride;
    c->dn_nzl = all[dn].nzl;
    c->dn_flag = reinterpret_cast<unsigned long long*>(b + all[dn].off_flags) + 1;
  }
  c->p2p = true;
  return PSM_OK;
}

// Remap-ahead (prescribed motion only): enqueue the remap for step `next` into the spare buffer
// on map_st, after the collide that last read that buffer (ev_coll); ev_map marks completion.
// The remap is latency/ALU-bound and the collide HBM-bound, so the two overlap.
static psm_status remap_ahead(psm_ctx* c, int64_t next) {
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

psm_status psm_step(psm_ctx* c, int64_t n) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (n < 0) FAIL(c, PSM_E_ARG, "n < 0");
  psm_status st = ensure_mem(c);
  if (st != PSM_OK) return st;
  if (n == 0) return PSM_OK;
  const bool fp64 = c->opt.prec == PSM_F64;
  const bool force = c->opt.body_force[0] != 0.0 || c->opt.body_force[1] != 0.0 ||
                     c->opt.body_force[2] != 0.0;
  CollideParams p;
  std::memset(&p, 0, sizeof(p));
  p.g = c->geom;
  p.word = c->word;
  p.tile_flag = c->tile_flag;
  p.partial = c->partial;
  p.overflow = c->overflow;
  p.err = c->err;
  p.dbg_B = c->dbg_B;
  p.dbg_us = c->dbg_us;
  p.dbg_id = c->dbg_id;
  p.tau = c->tau;
  p.omega = 1.0 / c->tau;
  p.omega_m = (c->opt.collision == PSM_TRT)
                  ? 1.0 / (0.5 + c->opt.trt_magic / (c->tau - 0.5))
                  : p.omega;
  p.trt = c->opt.collision == PSM_TRT ? 1 : (c->opt.collision == PSM_CUMULANT ? 2 : 0);
  for (int a = 0; a < 3; ++a) p.gforce[a] = c->opt.body_force[a];
  for (int a = 0; a < 3; ++a) p.u_in[a] = c->u_in[a];
  p.rho_out = c->rho_out;
  p.sc = c->opt.sc;
  p.bmode = c->opt.bmode;
  CUDA_TRY(c, cudaMemsetAsync(c->overflow, 0, (kMaxBodies + 1) * kSlotVals * 8, c->st));
  // remap-ahead pipeline: several steps in this call, bodies in prescribed motion only
  bool any_moving = false, any_dynamic = false;
  int max_s = 0;
  for (int id = 1; id <= kMaxBodies; ++id) {
    const Body& b = c->bodies[id];
    if (!b.present) continue;
    any_moving |= b.moving;
    any_dynamic |= b.dynamic;
    if (b.moving) max_s = std::max(max_s, b.s);
  }
  if (c->world > 1) {
    st = ensure_p2p(c);
    if (st != PSM_OK) return st;
  }
  static const bool no_ahead = std::getenv("PSM_NO_REMAP_AHEAD") != nullptr;
  // (at s = 3 the remap is ALU-heavy enough to slow the collide more than it hides: measured
  // 12.4k vs 14.8k MLUPS on c5w, so it runs in series there)
  const bool ahead = n > 1 && any_moving && !any_dynamic && !c->dbg && !no_ahead && max_s <= 2;
  if (ahead) {
    st = ensure_pipeline(c);
    if (st != PSM_OK) return st;
  }
  for (int64_t k = 0; k < n; ++k) {
    // 1. closed-form pose advance + remap of the bodies that moved; in the
    // pipeline the remap for this step was enqueued during the previous one into the spare buffer
    if (ahead && k > 0) {
      swap_buffers(c);
      CUDA_TRY(c, cudaStreamWaitEvent(c->st, c->ev_map, 0));
    } else {
      std::vector<int> moved;
      for (int id = 1; id <= kMaxBodies; ++id) {
        const Body& b = c->bodies[id];
        if (b.present && b.moving && b.ms.mapped_step != c->step) moved.push_back(id);
      }
      if (!moved.empty() && !c->dbg) {
        st = remap(c, moved, c->step);
        if (st != PSM_OK) return st;
      }
      if (ahead) CUDA_TRY(c, cudaEventRecord(c->ev_coll, c->st));  // spare buffer is free
    }
    if (ahead && k + 1 < n) {
      st = remap_ahead(c, c->step + 1);
      if (st != PSM_OK) return st;
    }
    // 2. fused PSM stream-collide (Eq.(4)) + F/T partials
    bool any_dyn = false;
    for (int id = 1; id <= kMaxBodies; ++id)
      if (c->bodies[id].present && c->bodies[id].dynamic) any_dyn = true;
    if (k == n - 1 || any_dyn)
      CUDA_TRY(c, cudaMemsetAsync(c->overflow, 0, (kMaxBodies + 1) * kSlotVals * 8, c->st));
    fill_kin(c, p, c->step);
    p.word = c->word;  // the active buffer (the pipeline swaps buffers between steps)
    p.tile_flag = c->tile_flag;
    p.step = c->step;
    int pat = 0;
    if (c->opt.pattern == PSM_TWO_ARRAY) {
      p.src = c->A[c->cur];
      p.dst = c->A[c->cur ^ 1];
    } else {
      p.src = c->A[0];
      p.dst = c->A[0];
      pat = (c->step & 1) ? 2 : 1;
    }
    const int gz = c->geom.gz;
    if (c->p2p) {
      // fused halo: wait for both neighbours' previous step, one launch over all tile layers
      // whose z-boundary cells also store into the neighbours' ghost planes, then signal
      if (c->epoch > 0)
        CUDA_TRY(c, launch_p2p_wait(c->has_dn ? c->flags + 0 : nullptr,
                                    c->has_up ? c->flags + 1 : nullptr, c->epoch, c->flags + 2,
                                    c->st));
      const int d = c->cur ^ 1;
      const size_t plane = (size_t)c->grid.nx * c->grid.ny;
      p.p2p = 1;
      for (int q = 0; q < c->Q; ++q) {
        p.gup[q] = (stc_z(q) > 0 && c->has_up)
                       ? (void*)(c->up_A[d] + (size_t)q * c->up_qs * c->S) : nullptr;
        p.gdn[q] = (stc_z(q) < 0 && c->has_dn)
                       ? (void*)(c->dn_A[d] + ((size_t)q * c->dn_qs +
                                               (size_t)(c->dn_nzl + 1) * plane) * c->S)
                       : nullptr;
      }
      if (record(c, 1, 0) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      p.tz0 = 0;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, gz, c->st));
      if (record(c, 1, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      c->epoch += 1;
      CUDA_TRY(c, launch_p2p_signal(c->has_up ? c->up_flag : nullptr,
                                    c->has_dn ? c->dn_flag : nullptr, c->epoch, c->st));
      c->launches += (c->epoch > 1) ? 3 : 2;
      c->cur ^= 1;
    } else if (c->world == 1 || gz < 3) {
      if (record(c, 1, 0) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      p.tz0 = 0;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, gz, c->st));
      c->launches += 1;
      if (record(c, 1, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      if (c->opt.pattern == PSM_TWO_ARRAY) c->cur ^= 1;
      if (c->world > 1) {
        if (record(c, 3, 0) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
        st = halo(c, c->A[c->cur], c->st);
        if (st != PSM_OK) return st;
        if (record(c, 3, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      }
    } else {
      // boundary tile layers first, then the halo on the comm stream overlaps the interior
      if (record(c, 1, 0) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      p.tz0 = 0;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, 1, c->st));
      p.tz0 = gz - 1;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, 1, c->st));
      CUDA_TRY(c, cudaEventRecord(c->ev_bnd, c->st));
      CUDA_TRY(c, cudaStreamWaitEvent(c->comm_st, c->ev_bnd, 0));
      st = halo(c, p.dst, c->comm_st);
      if (st != PSM_OK) return st;
      CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_st));
      p.tz0 = 1;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, gz - 2, c->st));
      c->launches += 3;
      if (record(c, 1, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      // the next collide (and any readback) reads the ghost planes: join the halo
      CUDA_TRY(c, cudaStreamWaitEvent(c->st, c->ev_halo, 0));
      c->cur ^= 1;
    }
    if (ahead) CUDA_TRY(c, cudaEventRecord(c->ev_coll, c->st));  // this buffer read: done
    c->step += 1;
    // 4. two-way coupling: this step's force/torque drives the dynamic bodies' next pose
    if (any_dyn && !c->dbg) {
      std::vector<int> ids;
      st = ft_enqueue(c, ids);
      if (st != PSM_OK) return st;
      CUDA_TRY(c, cudaStreamSynchronize(c->st));
      ft_store(c, ids);
      for (int id = 1; id <= kMaxBodies; ++id) {
        Body& b = c->bodies[id];
        if (!b.present || !b.dynamic) continue;
        const double F[3] = {-c->ft[id][0], -c->ft[id][1], -c->ft[id][2]};
        const double T[3] = {-c->ft[id][3], -c->ft[id][4], -c->ft[id][5]};
        integrate_body(c, b, F, T);
      }
    }
  }
  // 4. force/torque of the last step: deterministic two-pass reduction, then allreduce
  std::vector<int> ids;
  if (record(c, 2, 0) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
  st = ft_enqueue(c, ids);
  if (st != PSM_OK) return st;
  const int nb = (int)ids.size();
  if (record(c, 2, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
  unsigned long long* herr =
      reinterpret_cast<unsigned long long*>(c->pinned + (kMaxBodies + 1) * kSlotVals);
  CUDA_TRY(c, cudaMemcpyAsync(herr, c->err, 8, cudaMemcpyDeviceToHost, c->st));
  if (c->p2p) CUDA_TRY(c, cudaMemcpyAsync(herr + 1, c->flags + 2, 8, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  (void)nb;
  ft_store(c, ids);
  if (c->p2p && herr[1] != 0)
    FAIL(c, PSM_E_NCCL, "fused halo: a neighbour did not signal its step within 2 s");
  if (*herr != ~0ull) {
    const long long ncell = (long long)c->grid.nx * c->grid.ny * c->grid.nz;
    const long long stp = (long long)(*herr / (unsigned long long)ncell);
    const long long cell = (long long)(*herr % (unsigned long long)ncell);
    const long long x = cell % c->grid.nx, y = (cell / c->grid.nx) % c->grid.ny,
                    z = cell / (c->grid.nx * c->grid.ny);
    char buf[160];
    std::snprintf(buf, sizeof(buf), "invalid state (rho <= 0 or non-finite) at step %lld, cell "
                  "(%lld,%lld,%lld)", stp, x, y, z);
    CUDA_TRY(c, cudaMemsetAsync(c->err, 0xFF, 8, c->st));
    FAIL(c, PSM_E_STATE, buf);
  }
  return PSM_OK;
}

psm_status psm_force_torque(psm_ctx* c, int32_t id, double F[3], double T[3], double aF[3],
                            double aT[3]) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  if (id < 1 || id > kMaxBodies) FAIL(c, PSM_E_ARG, "body id must be in 1..16");
  if (!c->ft_valid) FAIL(c, PSM_E_STATE, "no step has run since the last state change");
  // the partials hold the momentum the fluid gains (printed Eqs.(10)-(11)); on the body: minus
  for (int a = 0; a < 3; ++a) {
    if (F) F[a] = -c->ft[id][a];
    if (T) T[a] = -c->ft[id][3 + a];
    if (aF) aF[a] = c->ft[id][6 + a];
    if (aT) aT[a] = c->ft[id][9 + a];
  }
  return PSM_OK;
}

psm_status psm_read_fractions(psm_ctx* c, double* B, uint8_t* id, int32_t* cnt) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  psm_status st = ensure_mem(c);
  if (st != PSM_OK) return st;
  const size_t plane = (size_t)c->grid.nx * c->grid.ny;
  const size_t per = plane * (8 + 1 + 4);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(c->nzl,
                                                              (int64_t)(c->stage_bytes / per)));
  for (int64_t za = 0; za < c->nzl; za += chunk) {
    const int64_t zb = std::min<int64_t>(c->nzl, za + chunk);
    const size_t nz = (size_t)(zb - za);
    FracParams p{};
    p.g = c->geom;
    p.word = c->word;
    p.B = c->stage;
    p.cnt = reinterpret_cast<int32_t*>(c->stage + nz * plane);
    p.id = reinterpret_cast<uint8_t*>(p.cnt + nz * plane);
    p.za = (int)za;
    p.zb = (int)zb;
    p.tau = c->tau;
    p.bmode = c->opt.bmode;
    for (int i = 0; i <= kMaxBodies; ++i) p.s[i] = c->bodies[i].s;
    CUDA_TRY(c, launch_read_fractions(p, c->st));
    c->launches += 1;
    if (B)
      CUDA_TRY(c, cudaMemcpyAsync(B + za * plane, p.B, nz * plane * 8, cudaMemcpyDeviceToHost,
                                  c->st));
    if (cnt)
      CUDA_TRY(c, cudaMemcpyAsync(cnt + za * plane, p.cnt, nz * plane * 4,
                                  cudaMemcpyDeviceToHost, c->st));
    if (id)
      CUDA_TRY(c, cudaMemcpyAsync(id + za * plane, p.id, nz * plane, cudaMemcpyDeviceToHost,
                                  c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  }
  return PSM_OK;
}

psm_status psm_debug_set_fields(psm_ctx* c, const double* B, const double* us,
                                const uint8_t* id) {
  if (!c || !B || !us || !id) FAIL(c, PSM_E_ARG, "null argument");
  if (c->opt.pattern != PSM_TWO_ARRAY) FAIL(c, PSM_E_UNSUPPORTED, "debug fields need TWO_ARRAY");
  psm_status st = ensure_mem(c);
  if (st != PSM_OK) return st;
  const size_t N = (size_t)c->ncell_local;
  c->alt_valid = false;
  if (!c->dbg_B) {
    CUDA_TRY(c, cudaMalloc(&c->dbg_B, N * 8));
    CUDA_TRY(c, cudaMalloc(&c->dbg_us, 3 * N * 8));
    CUDA_TRY(c, cudaMalloc(&c->dbg_id, N));
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->dbg_B, B, N * 8, cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dbg_us, us, 3 * N * 8, cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(c, cudaMemcpyAsync(c->dbg_id, id, N, cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(c, cudaMemsetAsync(c->tile_flag, 1, (size_t)c->ntiles, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  c->dbg = true;
  return PSM_OK;
}

psm_status psm_get_step(const psm_ctx* c, int64_t* step) {
  if (!c || !step) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  *step = c->step;
  return PSM_OK;
}

psm_status psm_halo_mode(const psm_ctx* c, int32_t* mode) {
  if (!c || !mode) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  *mode = c->world == 1 ? 0 : (c->p2p ? 2 : 1);
  return PSM_OK;
}

psm_status psm_launch_count(const psm_ctx* c, int64_t* launches) {
  if (!c || !launches) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  *launches = c->launches;
  return PSM_OK;
}

psm_status psm_profile(psm_ctx* c, int32_t enable) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  c->prof = enable != 0;
  return PSM_OK;
}

psm_status psm_profile_read(psm_ctx* c, double ms[PSM_NUM_PHASES],
                            int64_t count[PSM_NUM_PHASES]) {
  if (!c) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null ctx");
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  for (int ph = 0; ph < PSM_NUM_PHASES; ++ph) {
    for (auto& e : c->ev[ph]) {
      float t = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&t, e[0], e[1]));
      c->prof_ms[ph] += t;
      c->prof_cnt[ph] += 1;
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
    c->ev[ph].clear();
    if (ms) ms[ph] = c->prof_ms[ph];
    if (count) count[ph] = c->prof_cnt[ph];
    c->prof_ms[ph] = 0.0;
    c->prof_cnt[ph] = 0;
  }
  return PSM_OK;
}

int32_t psm_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

psm_status psm_nccl_get_unique_id(void* out128) {
  if (!out128) FAIL((psm_ctx*)nullptr, PSM_E_ARG, "null argument");
  ncclUniqueId id;
  NCCL_TRY((psm_ctx*)nullptr, ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return PSM_OK;
}

const char* psm_last_error(const psm_ctx* c) {
  if (c) return c->err_msg.c_str();
  return g_last_error.c_str();
}

}  // extern "C"
