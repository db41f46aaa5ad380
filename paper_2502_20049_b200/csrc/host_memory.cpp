// host_memory.cpp — device memory plan and binding, lazy NCCL/pinned-buffer setup, and the
// chunked conversion between the Eq.(4) state and the pattern-specific PDF storage (k_state.cu).
#include "psm_ctx.h"

namespace psm {

cudaError_t record(psm_ctx* c, int phase, int which, cudaStream_t s) {
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
  if (c->seg_cap_env > 0) p.seg_cap = (int)std::min<int64_t>(p.seg_cap, c->seg_cap_env);
  if (c->band_cap_env > 0) p.band_cap = (int)std::min<int64_t>(p.band_cap, c->band_cap_env);
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


psm_status bind(psm_ctx* c, void* mem, size_t bytes) {
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

psm_status ensure_pinned(psm_ctx* c) {
  if (c->pinned) return PSM_OK;
  if (cudaMallocHost(&c->pinned, (kMaxBodies + 2) * kSlotVals * 8) != cudaSuccess) {
    cudaGetLastError();
    c->pinned = nullptr;
    FAIL(c, PSM_E_OOM, "cudaMallocHost failed");
  }
  return PSM_OK;
}

psm_status ensure_comm(psm_ctx* c) {
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

psm_status ensure_mem(psm_ctx* c) {
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

psm_status state_write(psm_ctx* c, const double* host, int mode) {
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

psm_status state_read(psm_ctx* c, double* f, double* rho, double* u, int64_t zbeg,
                      int64_t zend) {
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


size_t plan_total_bytes(const psm_ctx* c) { return make_plan(c).total; }

}  // namespace psm
