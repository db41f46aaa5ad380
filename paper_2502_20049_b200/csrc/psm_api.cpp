// psm_api.cpp — C ABI of the B200 PSM hot path (include/psm.h): validation, the extern "C" entry
// points and the per-step launch sequence.  Host orchestration only; every arithmetic step of the
// method runs in the sm_100a kernels (k_*.cu).  The rest of the host side is split over
// host_bodies.cpp, host_memory.cpp, host_remap.cpp and host_halo.cpp (psm_ctx.h).
#include "psm_ctx.h"

using namespace psm;

namespace psm {
std::string g_last_error;
}  // namespace psm

namespace {

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

}  // namespace

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
  if (world > 1 && opt->pattern == PSM_AA && grid->bc[0] != PSM_PERIODIC)
    FAIL((psm_ctx*)nullptr, PSM_E_UNSUPPORTED, "PSM_AA across ranks needs a periodic x axis");
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
  if (const char* e = std::getenv("PSM_AHEAD_BLOCKS")) c->ahead_blocks_env = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PSM_P2P_TIMEOUT_S"))
    c->p2p_timeout_ns = (unsigned long long)(std::max(1.0, std::atof(e)) * 1e9);
  if (const char* e = std::getenv("PSM_BAND_CACHE")) c->no_cache = std::strcmp(e, "0") == 0;
  c->force_general = std::getenv("PSM_REMAP_GENERAL") != nullptr;
  if (const char* e = std::getenv("PSM_CACHE_MAX_S")) c->cache_max_s = std::atoi(e);
  if (const char* e = std::getenv("PSM_CACHE_MAX_S_R2")) c->cache_max_s_r2 = std::atoi(e);
  if (const char* e = std::getenv("PSM_REMAP_L12")) c->remap_fused12 = std::atoi(e) != 0;
  if (const char* e = std::getenv("PSM_HIOCC")) c->hiocc_env = std::atoi(e) != 0 ? 1 : 0;
  if (const char* e = std::getenv("PSM_SEG_CAP")) c->seg_cap_env = std::max(1ll, std::atoll(e));
  if (const char* e = std::getenv("PSM_BAND_CAP")) c->band_cap_env = std::max(1ll, std::atoll(e));
  if (const char* e = std::getenv("PSM_AHEAD_THREADS"))  // whole warps (the band pass sums a
    // cell's 8 lanes with full-warp shuffles), at most the remap kernels' launch bound of 256
    c->ahead_threads = std::min(256, std::max(32, std::atoi(e))) / 32 * 32;
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
  if (const char* e = std::getenv("PSM_PLANE_PAD"))  // tuning: elements between direction planes
    g.qstride += (std::max(0ll, std::atoll(e)) + 31) / 32 * 32;
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
  if (c->p2p && c->comm) {
    // this rank's memory is mapped by its neighbours (fused halo): a collective barrier before
    // it is freed, so no rank can still be storing into it (psm_destroy is collective)
    int one = 1;
    int* d = reinterpret_cast<int*>(c->flags + 3);
    cudaMemcpyAsync(d, &one, sizeof(int), cudaMemcpyHostToDevice, c->st);
    ncclAllReduce(d, d, 1, ncclInt32, ncclSum, c->comm, c->st);
  }
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
  *bytes = plan_total_bytes(c);
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
      const int sl = shape->s;
      const size_t nbk = (size_t)(nb.dims[0] * nb.dims[1] * nb.dims[2]);
      // linear bit index (psm_device.cuh BodyGeo::bits): ceil(bricks * 8^s / 64) words
      if (nbk >= (1ull << 31) || ((nbk << (3 * sl)) + 63) / 64 >= (1ull << 31))
        FAIL(c, PSM_E_ARG, "mesh geometry field too large (32-bit brick and word indices)");
      nb.words = (int)(((nbk << (3 * sl)) + 63) / 64);
      CUDA_TRY(c, cudaMalloc(&nb.d_bits, (size_t)nb.words * 8));
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
      // the spare word buffer (and its band) followed the dynamic pose; a body that comes to
      // rest here is not remapped by psm_step, so map it now at the integrated pose
      c->alt_valid = false;
      c->ft_valid = false;
      if (!b.moving) return remap(c, std::vector<int>{id}, c->step);
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
  if (!b.dynamic) {
    c->alt_valid = false;
    c->ft_valid = false;
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
  // fp64 D3Q19: the higher-occupancy collide when PSM tiles were frequent at the end of the
  // previous call (PSM_HIOCC=0/1 forces it).  Break-even measured per operator: fluid-only it
  // costs 0.8-2 %; the AA cumulant's PSM tiles gain enough from 2.5 % of the tiles on (c5wpap,
  // 3.2 %: +0.45 %), the other operators from 8 % (c3 scenario A, 15 %: +4-7 %)
  const bool aa_cum = c->opt.pattern == PSM_AA && c->opt.collision == PSM_CUMULANT;
  p.hiocc = c->hiocc_env >= 0 ? c->hiocc_env
                              : (c->psm_tile_frac > (aa_cum ? 0.025 : 0.08) ? 1 : 0);
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
                                    c->p2p_timeout_ns, c->st));
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
        st = (c->opt.pattern == PSM_AA) ? halo_aa(c, pat == 2, c->st)
                                        : halo(c, c->A[c->cur], c->st);
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
      // (AA: the interior layers neither read nor write the boundary or ghost planes the copies
      // touch, host_halo.cpp)
      st = (c->opt.pattern == PSM_AA) ? halo_aa(c, pat == 2, c->comm_st)
                                      : halo(c, p.dst, c->comm_st);
      if (st != PSM_OK) return st;
      CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_st));
      p.tz0 = 1;
      CUDA_TRY(c, launch_collide(c->Q, fp64, p, pat, force, c->dbg, gz - 2, c->st));
      c->launches += 3;
      if (record(c, 1, 1) != cudaSuccess) FAIL(c, PSM_E_CUDA, "event record failed");
      // the next collide (and any readback) reads the ghost planes: join the halo
      CUDA_TRY(c, cudaStreamWaitEvent(c->st, c->ev_halo, 0));
      if (c->opt.pattern == PSM_TWO_ARRAY) c->cur ^= 1;
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
  if (c->p2p && c->epoch > 0) {
    // fused halo: the neighbours' last collide stores into this rank's ghost planes; wait for
    // their signal so that a readback / state write after this call sees (or overwrites) final
    // values, and no peer store is still in flight when the call returns
    CUDA_TRY(c, launch_p2p_wait(c->has_dn ? c->flags + 0 : nullptr,
                                c->has_up ? c->flags + 1 : nullptr, c->epoch, c->flags + 2,
                                c->p2p_timeout_ns, c->st));
    c->launches += 1;
  }
  CUDA_TRY(c, cudaMemcpyAsync(herr, c->err, 8, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, launch_count_tiles(c->tile_flag, c->ntiles, c->flags + 5, c->st));
  c->launches += 1;
  CUDA_TRY(c, cudaMemcpyAsync(herr + 2, c->flags + 5, 8, cudaMemcpyDeviceToHost, c->st));
  if (c->p2p) CUDA_TRY(c, cudaMemcpyAsync(herr + 1, c->flags + 2, 8, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  (void)nb;
  ft_store(c, ids);
  c->psm_tile_frac = (double)herr[2] / (double)c->ntiles;
  static const bool stats_on = std::getenv("PSM_MAP_STATS") != nullptr;
  if (stats_on)
    std::fprintf(stderr, "[psm step] %lld steps, PSM tiles %.4f of the tiles, hiocc %d\n",
                 (long long)n, c->psm_tile_frac, p.hiocc);
  if (c->p2p && herr[1] != 0)
    FAIL(c, PSM_E_NCCL, "fused halo: a neighbour did not signal its step in time (PSM_P2P_TIMEOUT_S)");
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
