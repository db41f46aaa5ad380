// psm_ctx.h — host-side context of the C ABI (psm_ctx) and the internal interfaces between the
// host translation units: psm_api.cpp (the ABI entry points and the step loop), host_bodies.cpp
// (poses, boxes, the coupling integrator), host_memory.cpp (memory plan, state conversion),
// host_remap.cpp (remap planning, cached bands, remap-ahead) and host_halo.cpp (NCCL and fused
// peer-store halo).  Product library only; nothing here is shared with oracle/.
#pragma once
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

namespace psm {

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
  int words = 1;          // uint64 words of the packed geometry field
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

}  // namespace psm

using psm::Body;
using psm::Box;
using psm::MapState;
using psm::Geom;
using psm::kMaxBodies;
using psm::kSlotVals;

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
  int ahead_blocks_env = 0;          // PSM_AHEAD_BLOCKS (persistent remap blocks when overlapped)
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
  // remap switches read from the environment at psm_create (diagnostics / tests):
  // PSM_BAND_CACHE=0, PSM_REMAP_GENERAL, PSM_SEG_CAP / PSM_BAND_CAP (cap the segment / band lists
  // of the full pipeline so that the in-kernel overflow paths run)
  bool no_cache = false, force_general = false;
  int cache_max_s = 1;     // cached narrow band up to this s, R1 (PSM_CACHE_MAX_S)
  int cache_max_s_r2 = 3;  // the same for R2 bodies (PSM_CACHE_MAX_S_R2)
  int remap_fused12 = 1;   // L1 + L2 in one launch (PSM_REMAP_L12=0: two)
  int hiocc_env = -1;   // PSM_HIOCC: force (1) / forbid (0) the higher-occupancy fp64 collide
  double psm_tile_frac = 0.0;  // PSM tiles / tiles in the last psm_step call
  int64_t seg_cap_env = 0, band_cap_env = 0;
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
  unsigned long long p2p_timeout_ns = 60ull * 1000000000ull;  // handshake bound (PSM_P2P_TIMEOUT_S)
  unsigned char nccl_id[128] = {};
  std::string err_msg;
  int64_t launches = 0;
  bool prof = false;
  std::vector<std::array<cudaEvent_t, 2>> ev[PSM_NUM_PHASES];
  double prof_ms[PSM_NUM_PHASES] = {};
  int64_t prof_cnt[PSM_NUM_PHASES] = {};
};

namespace psm {
extern std::string g_last_error;  // message of the last failing call (psm_last_error(NULL))
}

#define FAIL(ctx, code, msg)                  \
  do {                                        \
    std::string _m = (msg);                   \
    if (ctx) (ctx)->err_msg = _m;             \
    psm::g_last_error = _m;                   \
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


namespace psm {
// host_bodies.cpp
void free_bands(Body& b);
void rodrigues(const double w[3], double n, const double Q0[9], double out[9]);
double extent(const psm_ctx* c, int a);
void pose_at(const psm_ctx* c, const Body& b, int64_t step, double Q[9], double t[3]);
void body_box(const psm_ctx* c, const Body& b, const double Q[9], const double t[3],
              int64_t lo[3], int64_t hi[3]);
int axis_pieces(const psm_ctx* c, int a, int64_t lo, int64_t hi, int64_t out[2][2]);
void add_box(const psm_ctx* c, const int64_t lo[3], const int64_t hi[3], std::vector<Box>& out);
void remap_region(const psm_ctx* c, Body& b, const double Q[9], const double t[3],
                  std::vector<Box>& boxes);
void integrate_body(const psm_ctx* c, Body& b, const double F[3], const double T[3]);
// host_memory.cpp
cudaError_t record(psm_ctx* c, int phase, int which, cudaStream_t s = nullptr);
size_t plan_total_bytes(const psm_ctx* c);
psm_status bind(psm_ctx* c, void* mem, size_t bytes);
psm_status ensure_pinned(psm_ctx* c);
psm_status ensure_comm(psm_ctx* c);
psm_status ensure_mem(psm_ctx* c);
psm_status state_write(psm_ctx* c, const double* host, int mode);
psm_status state_read(psm_ctx* c, double* f, double* rho, double* u, int64_t zbeg = 0,
                      int64_t zend = -1);
// host_halo.cpp
psm_status halo(psm_ctx* c, void* arr, cudaStream_t hst);
psm_status halo_aa(psm_ctx* c, bool after_odd, cudaStream_t hst);
psm_status ensure_p2p(psm_ctx* c);
// host_remap.cpp
psm_status run_map(psm_ctx* c, const std::vector<Box>& boxes);
void swap_buffers(psm_ctx* c);
psm_status ensure_pipeline(psm_ctx* c);
psm_status remap(psm_ctx* c, const std::vector<int>& ids, int64_t step);
psm_status remap_ahead(psm_ctx* c, int64_t next);
}  // namespace psm
