// host_halo.cpp — z-slab halo between ranks: NCCL grouped send/recv of contiguous planes, and the
// setup of the fused peer-store halo (CUDA IPC handles exchanged over NCCL).
#include "psm_ctx.h"

namespace psm {

psm_status halo(psm_ctx* c, void* arr, cudaStream_t hst) {
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

// AA pattern across ranks (ghost planes, NCCL): the even step is local; the odd step reads
// A[ibar][x - c_i] and writes A[i][x + c_i], so it reaches one plane into each neighbour.
//   after an even step: the boundary planes the neighbours' odd step will read go into their
//     ghost planes (top plane, c_z = -1 directions, up; bottom plane, c_z = +1, down);
//   after an odd step: what this rank's odd step wrote into its ghost planes belongs to the
//     neighbours' boundary planes (ghost below, c_z = -1, down; ghost above, c_z = +1, up).
// A ghost slot whose source cell would lie beyond a y wall is not written by this rank's odd
// step (the neighbour bounces that population into its own slot), so the second copy skips that
// row: planes of directions with c_y = +1 start at row 1, with c_y = -1 end at row ny-2 — still
// contiguous.  (x walls would need strided copies; psm_create rejects them with AA across ranks.)
psm_status halo_aa(psm_ctx* c, bool after_odd, cudaStream_t hst) {
  if (c->world == 1) return PSM_OK;
  const int P = c->world, r = c->rank;
  const bool zwall = c->grid.bc[2] == PSM_WALL;
  const int up = (r + 1) % P, down = (r - 1 + P) % P;
  const bool has_up = !(zwall && r == P - 1), has_down = !(zwall && r == 0);
  const size_t plane = (size_t)c->grid.nx * c->grid.ny;
  const ncclDataType_t dt = (c->opt.prec == PSM_F64) ? ncclFloat64 : ncclFloat32;
  char* base = static_cast<char*>(c->A[0]);
  auto ptr = [&](int q, int64_t zs) {
    return base + ((size_t)q * (size_t)c->geom.qstride + (size_t)zs * plane) * c->S;
  };
  const int64_t top = c->nzl, bot = 1, gdn = 0, gup = c->nzl + 1;
  const bool ywall = c->grid.bc[1] == PSM_WALL;
  const size_t nx = (size_t)c->grid.nx;
  NCCL_TRY(c, ncclGroupStart());
  for (int q = 0; q < c->Q; ++q) {
    const int cz = stc_z(q), cy = stc_y(q);
    // rows of the second (after-odd) copy: all, or all but the row beyond the y wall
    const size_t r0 = (after_odd && ywall && cy > 0) ? nx : 0;
    const size_t cnt = (after_odd && ywall && cy != 0) ? plane - nx : plane;
    auto at = [&](int64_t zs) { return ptr(q, zs) + r0 * c->S; };
    if (cz < 0) {
      if (!after_odd) {
        if (has_up) NCCL_TRY(c, ncclSend(ptr(q, top), plane, dt, up, c->comm, hst));
        if (has_down) NCCL_TRY(c, ncclRecv(ptr(q, gdn), plane, dt, down, c->comm, hst));
      } else {
        if (has_down) NCCL_TRY(c, ncclSend(at(gdn), cnt, dt, down, c->comm, hst));
        if (has_up) NCCL_TRY(c, ncclRecv(at(top), cnt, dt, up, c->comm, hst));
      }
    } else if (cz > 0) {
      if (!after_odd) {
        if (has_down) NCCL_TRY(c, ncclSend(ptr(q, bot), plane, dt, down, c->comm, hst));
        if (has_up) NCCL_TRY(c, ncclRecv(ptr(q, gup), plane, dt, up, c->comm, hst));
      } else {
        if (has_up) NCCL_TRY(c, ncclSend(at(gup), cnt, dt, up, c->comm, hst));
        if (has_down) NCCL_TRY(c, ncclRecv(at(bot), cnt, dt, down, c->comm, hst));
      }
    }
  }
  NCCL_TRY(c, ncclGroupEnd());
  return PSM_OK;
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

psm_status ensure_p2p(psm_ctx* c) {
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

}  // namespace psm
