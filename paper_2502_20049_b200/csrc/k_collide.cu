// k_collide.cu — launcher of the fused PSM stream-collide (kernels in k_collide.cuh, one
// translation unit per stencil and precision: k_collide_19f/19d/27f/27d.cu) and the fused-halo
// step handshake kernels.
#include "k_collide.cuh"

namespace psm {

// ---- fused-halo step handshake between neighbouring ranks (peer memory) ----
// signal: after this rank's collide (stream order: its peer stores are complete), publish the
// step count into each neighbour's flag word with system-scope release semantics
__global__ void k_p2p_signal(unsigned long long* up_flag, unsigned long long* dn_flag,
                             unsigned long long v) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (up_flag) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(up_flag), "l"(v) : "memory");
  if (dn_flag) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dn_flag), "l"(v) : "memory");
}

// wait: before the next collide reads the ghost planes (and overwrites the neighbours' other
// array), both neighbours must have signalled step v; bounded spin (default 60 s, host work
// between steps can legitimately skew the ranks) so a lost peer cannot hang the device — then
// the error word records it and the step fails
__global__ void k_p2p_wait(const unsigned long long* from_dn, const unsigned long long* from_up,
                           unsigned long long v, unsigned long long* err,
                           unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long a = v, b = v;
    if (from_dn) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(from_dn) : "memory");
    if (from_up) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(b) : "l"(from_up) : "memory");
    if (a >= v && b >= v) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch(err, 1ull);  // the host turns this into PSM_E_NCCL
      return;
    }
    __nanosleep(200);
  }
}

cudaError_t launch_p2p_signal(unsigned long long* up_flag, unsigned long long* dn_flag,
                              unsigned long long v, cudaStream_t st) {
  k_p2p_signal<<<1, 1, 0, st>>>(up_flag, dn_flag, v);
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const unsigned long long* from_dn, const unsigned long long* from_up,
                            unsigned long long v, unsigned long long* err,
                            unsigned long long timeout_ns, cudaStream_t st) {
  k_p2p_wait<<<1, 1, 0, st>>>(from_dn, from_up, v, err, timeout_ns);
  return cudaGetLastError();
}

// number of flagged (PSM) tiles of a tile-flag buffer: one atomic per block.  (Counting in the
// collide itself, one atomic per PSM tile, measured 8 % slower fp64 kernels from the code it
// changes around the fluid path.)
__global__ void k_count_tiles(const uint8_t* flag, long long n, unsigned long long* out) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += flag[i] != 0;
  c = __reduce_add_sync(0xFFFFFFFFu, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0 && s) atomicAdd(out, s);
}

cudaError_t launch_count_tiles(const uint8_t* flag, long long n, unsigned long long* out,
                               cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, 8, st);
  if (e != cudaSuccess) return e;
  k_count_tiles<<<148, 256, 0, st>>>(flag, n, out);
  return cudaGetLastError();
}

cudaError_t launch_collide(int Q, bool fp64, const CollideParams& p, int pat, bool force,
                           bool dbg, int ntz, cudaStream_t st) {
  if (Q == 19) return fp64 ? launch_collide_19d(p, pat, force, dbg, ntz, st)
                           : launch_collide_19f(p, pat, force, dbg, ntz, st);
  return fp64 ? launch_collide_27d(p, pat, force, dbg, ntz, st)
              : launch_collide_27f(p, pat, force, dbg, ntz, st);
}

}  // namespace psm
