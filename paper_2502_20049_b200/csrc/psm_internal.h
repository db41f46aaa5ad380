// psm_internal.h — host-side launchers of the sm_100a kernels (product library only).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "psm_device.cuh"

namespace psm {

// k_collide.cu
// launches tile layers [p.tz0, p.tz0 + ntz) in z
cudaError_t launch_collide(int Q, bool fp64, const CollideParams& p, int pat, bool force,
                           bool dbg, int ntz, cudaStream_t st);

// flagged tiles of a tile-flag buffer -> *out (k_collide.cu)
cudaError_t launch_count_tiles(const uint8_t* flag, long long n, unsigned long long* out,
                               cudaStream_t st);

// fused-halo handshake (k_collide.cu)
cudaError_t launch_p2p_signal(unsigned long long* up_flag, unsigned long long* dn_flag,
                              unsigned long long v, cudaStream_t st);
cudaError_t launch_p2p_wait(const unsigned long long* from_dn, const unsigned long long* from_up,
                            unsigned long long v, unsigned long long* err,
                            unsigned long long timeout_ns, cudaStream_t st);

// k_voxelize.cu — GPU voxeliser (reading A15), writes the packed bricks and the brick flags
struct VoxParams {
  const long long* V;        // snapped vertices [nv][3], fixed point 2^-(s+12) from the origin
  const int* tris;           // [nt][3]
  long long nt;
  int s;                     // super-sampling level: 2^s samples per LBM cell and axis
  long long NX, NY, NZ;      // geometry cells (= LBM cells << s)
  long long bx, by, bz;      // bricks (= LBM cells of the field)
  int W;                     // uint64 words of the whole packed field
  unsigned long long* words; // [W] output, linear bit index (brick << 3s) + bit in brick
  unsigned* tog;             // scratch: toggle bits, wpr words per (gy, gz) row
  long long wpr;
};
size_t voxelize_scratch_bytes(const VoxParams& p);
cudaError_t launch_voxelize(VoxParams p, void* scratch, uint8_t* mask, cudaStream_t st);

// k_map.cu (general boxes) and k_remap.cu (boxes holding one body)
cudaError_t launch_map(const MapParams& p, cudaStream_t st);
cudaError_t launch_remap_single(const RemapParams& r, int persistent_blocks, cudaStream_t st,
                                int threads = 256);
int remap_l3_kernels(const BodyGeo& b);        // kernels launch_remap_band launches
int remap_single_kernels(const RemapParams& r);  // kernels launch_remap_single launches
cudaError_t launch_remap_band(const RemapParams& r, int persistent_blocks, cudaStream_t st,
                              int threads = 256);

// k_state.cu — conversions between the Eq.(4) state and the storage pattern, z-chunked.
struct StateParams {
  Geom g;
  void* A;               // PDF storage (pattern-specific layout)
  double* stage;         // fp64 staging buffer
  int za, zb;            // local planes [za, zb) handled by this launch
  int stage_z0;          // local z of staging plane 0 (write: za - 1; read: za)
  int stage_nz;          // planes in the staging buffer
  int pattern;           // 0 pull, 1 AA
  int odd;               // AA: current step count is odd
  int mode;              // write: 0 = f from stage [Q][planes], 1 = feq from rho,u stage
                         //        [4][planes], 2 = uniform rho=1,u=0; read: 0 = f, 1 = rho,u
  int ghosts;            // write: also fill the ghost planes adjacent to [za, zb)
  double u_in[3];        // A30 open x faces (g.open_x): inflow velocity
  double rho_out;        //                              outflow density
};
cudaError_t launch_write_state(int Q, bool fp64, const StateParams& p, cudaStream_t st);
cudaError_t launch_read_state(int Q, bool fp64, const StateParams& p, cudaStream_t st);

// fractions readback: words -> B (fp64), id, cnt for local planes [za, zb)
struct FracParams {
  Geom g;
  const uint32_t* word;
  double* B;
  uint8_t* id;
  int32_t* cnt;
  int za, zb;
  double tau;
  int bmode;
  int s[kMaxBodies + 1];
};
cudaError_t launch_read_fractions(const FracParams& p, cudaStream_t st);

// force/torque: two-pass deterministic reduction over the tile partials of one step
cudaError_t launch_ft_reduce(const uint8_t* tile_flag, const double* partial, int ntiles,
                             const double* overflow, const int* ids, int nb, double* scratch,
                             int nchunks, double* out, cudaStream_t st);

}  // namespace psm
