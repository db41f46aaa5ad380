// k_voxelize.cu — the one-time voxelisation of a closed triangle mesh into the super-sampled
// geometry field ("voxelizing the geometry onto the geometry field once as a
// pre-processing step"), on the GPU, producing directly the packed LBM-cell bricks and the
// per-brick early-out flags the remap kernels read.  Bit-identical to the host reference
// implementation of reading A15 (csrc/voxelize.cpp, checked against the oracle's per-row
// voxelizer): the same fixed-point vertices (snapped on the host), the same exact integer
// edge functions with the top-left tie rule, the same crossing rule (strictly x* > x0), and
// parity by XOR, which does not depend on the order in which crossings are found.
//
//   k_vox_tri    one warp per triangle: lanes walk the (y, z) sample rows of its projected
//                bounding box; a covered row gets one toggle bit at the first sample index the
//                crossing does not cover (atomicXor into a bit array, (NX+1) bits per row)
//   k_vox_rows   one thread per row: suffix XOR of the toggles gives inside/outside per sample;
//                each run of 2^s samples of one brick is OR-ed into its bits of the linearly
//                packed field
//   k_vox_any    per brick: any sample inside / any sample outside
//   k_box_pass   separable running-window OR (radius r along one axis, beyond the field = 0)
//   k_vox_mask   the eight early-out bits
#include "psm_device.cuh"
#include "psm_internal.h"

namespace psm {

typedef __int128 i128;

__device__ __forceinline__ bool tl_inside_d(long long ay, long long az, long long by,
                                            long long bz, long long py, long long pz) {
  const i128 e = (i128)(by - ay) * (i128)(pz - az) - (i128)(bz - az) * (i128)(py - ay);
  if (e != 0) return e > 0;
  const long long dy = by - ay, dz = bz - az;
  return (dz == 0 && dy < 0) || dz < 0;  // top or left edge owns its boundary points
}

__device__ __forceinline__ i128 ceil_div_d(i128 a, i128 b) {  // b > 0
  if (a >= 0) return (a + b - 1) / b;
  return -((-a) / b);
}

// rows g with lo <= g*4096 + 2048 <= hi, clipped to [0, n)
__device__ __forceinline__ void row_range_d(long long lo, long long hi, long long n,
                                            long long& r0, long long& r1) {
  r0 = (long long)ceil_div_d((i128)lo - 2048, 4096);
  if (r0 < 0) r0 = 0;
  const long long t = hi - 2048;
  long long f = t >= 0 ? t / 4096 : -((-t + 4095) / 4096);
  r1 = f < n - 1 ? f : n - 1;
}

__global__ void k_vox_tri(const VoxParams p) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.nt) return;
  const long long* A = p.V + 3ll * p.tris[3 * warp];
  const long long* B = p.V + 3ll * p.tris[3 * warp + 1];
  const long long* C = p.V + 3ll * p.tris[3 * warp + 2];
  const i128 area = (i128)(B[1] - A[1]) * (i128)(C[2] - A[2]) -
                    (i128)(B[2] - A[2]) * (i128)(C[1] - A[1]);
  if (area == 0) return;  // degenerate projection: the ray never enters it
  const long long *P1 = (area > 0) ? B : C, *P2 = (area > 0) ? C : B;
  const i128 e1[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
  const i128 e2[3] = {C[0] - A[0], C[1] - A[1], C[2] - A[2]};
  const i128 n0 = e1[1] * e2[2] - e1[2] * e2[1];
  const i128 n1 = e1[2] * e2[0] - e1[0] * e2[2];
  const i128 n2 = e1[0] * e2[1] - e1[1] * e2[0];
  const i128 M = n0 > 0 ? n0 : -n0;
  long long z0, z1, y0, y1;
  row_range_d(min(A[2], min(B[2], C[2])), max(A[2], max(B[2], C[2])), p.NZ, z0, z1);
  row_range_d(min(A[1], min(B[1], C[1])), max(A[1], max(B[1], C[1])), p.NY, y0, y1);
  if (z1 < z0 || y1 < y0) return;
  const long long ny = y1 - y0 + 1, total = ny * (z1 - z0 + 1);
  for (long long k = lane; k < total; k += 32) {
    const long long gz = z0 + k / ny, gy = y0 + k % ny;
    const long long Y0 = gy * 4096 + 2048, Z0 = gz * 4096 + 2048;
    if (!tl_inside_d(A[1], A[2], P1[1], P1[2], Y0, Z0)) continue;
    if (!tl_inside_d(P1[1], P1[2], P2[1], P2[2], Y0, Z0)) continue;
    if (!tl_inside_d(P2[1], P2[2], A[1], A[2], Y0, Z0)) continue;
    // the crossing counts for sample X0 iff M*X0 < Nn; samples gx < (Nn - 2048M)/(4096M)
    const i128 K = n1 * (i128)(A[1] - Y0) + n2 * (i128)(A[2] - Z0);
    const i128 Nraw = n0 * (i128)A[0] + K;
    const i128 Nn = n0 > 0 ? Nraw : -Nraw;
    i128 kmax = ceil_div_d(Nn - 2048 * M, 4096 * M);
    if (kmax <= 0) continue;
    if (kmax > p.NX) kmax = p.NX;
    const long long j = (long long)kmax;
    atomicXor(p.tog + (gz * p.NY + gy) * p.wpr + (j >> 5), 1u << (j & 31));
  }
}

__global__ void k_vox_rows(const VoxParams p) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= p.NY * p.NZ) return;
  const long long gy = row % p.NY, gz = row / p.NY;
  const unsigned* tg = p.tog + row * p.wpr;
  const int s = p.s, n = 1 << s;
  const unsigned run_mask = (n >= 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
  const long long bzi = gz >> s, byi = gy >> s;
  const int off = ((int)(gz & (n - 1)) * n + (int)(gy & (n - 1))) * n;  // bit of (gz, gy) rows
  unsigned carry = 0;  // parity of all toggles above the current word
  for (long long w = p.wpr - 1; w >= 0; --w) {
    const unsigned t = tg[w];
    if (t == 0 && carry == 0) continue;
    unsigned Y = t;  // inclusive suffix XOR within the word (towards lower bits)
    Y ^= Y >> 1;
    Y ^= Y >> 2;
    Y ^= Y >> 4;
    Y ^= Y >> 8;
    Y ^= Y >> 16;
    unsigned in = (Y >> 1) ^ (carry ? 0xFFFFFFFFu : 0u);  // exclusive: toggles at j > gx
    carry ^= (Y & 1u);
    const long long gx0 = w * 32;
    if (gx0 >= p.NX) continue;
    if (p.NX - gx0 < 32) in &= (1u << (p.NX - gx0)) - 1u;
    if (!in) continue;
    for (int c = 0; c < 32; c += n) {
      const unsigned bits = (in >> c) & run_mask;
      if (!bits) continue;
      const long long bxi = (gx0 + c) >> s;
      const long long b = (bzi * p.by + byi) * p.bx + bxi;
      const long long gb = (b << (3 * s)) + off;  // linear bit index (psm_device.cuh)
      atomicOr(p.words + (gb >> 6), (unsigned long long)bits << (gb & 63));
    }
  }
}

__global__ void k_vox_any(const VoxParams p, uint8_t* any_in, uint8_t* any_out) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nb = p.bx * p.by * p.bz;
  if (b >= nb) return;
  const int nbits = 1 << (3 * p.s);
  const long long gb0 = b << (3 * p.s);
  int ones = 0;
  if (nbits >= 64) {
    for (int k = 0; k < nbits / 64; ++k) ones += __popcll(p.words[(gb0 >> 6) + k]);
  } else {
    ones = __popcll((p.words[gb0 >> 6] >> (gb0 & 63)) & ((1ull << nbits) - 1ull));
  }
  any_in[b] = ones > 0;
  any_out[b] = ones < nbits;
}

// v_out[i] = OR of v_in over [i - r, i + r] along one axis (lines of n elements, stride)
__global__ void k_box_pass(const uint8_t* v_in, uint8_t* v_out, long long n, long long stride,
                           long long lines, int axis, long long bx, long long by, int r) {
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lines) return;
  long long b0;
  if (axis == 0) b0 = l * bx;
  else if (axis == 1) b0 = (l / bx) * bx * by + (l % bx);
  else b0 = l;
  int cnt = 0;
  for (long long i = 0; i < min(n, (long long)r); ++i) cnt += v_in[b0 + i * stride];
  for (long long i = 0; i < n; ++i) {
    if (i + r < n) cnt += v_in[b0 + (i + r) * stride];
    if (i - r - 1 >= 0) cnt -= v_in[b0 + (i - r - 1) * stride];
    v_out[b0 + i * stride] = cnt > 0;
  }
}

__global__ void k_vox_mask(long long bx, long long by, long long bz, const uint8_t* in1,
                           const uint8_t* out1, const uint8_t* inK, const uint8_t* outK,
                           const uint8_t* inS, const uint8_t* outS, const uint8_t* in2,
                           const uint8_t* out2, uint8_t* mask) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= bx * by * bz) return;
  const long long ix = b % bx, iy = (b / bx) % by, iz = b / (bx * by);
  auto inside_field = [&](int r) {
    return ix - r >= 0 && iy - r >= 0 && iz - r >= 0 && ix + r < bx && iy + r < by &&
           iz + r < bz;
  };
  uint8_t m = 0;
  if (!in1[b]) m |= 1;
  if (!out1[b] && inside_field(1)) m |= 2;
  if (!inK[b]) m |= 4;
  if (!outK[b] && inside_field(kTileReach)) m |= 8;
  if (!inS[b]) m |= 16;
  if (!outS[b] && inside_field(kSubReach)) m |= 32;
  if (!in2[b]) m |= 64;
  if (!out2[b] && inside_field(2)) m |= 128;
  mask[b] = m;
}

static cudaError_t box_or_dev(uint8_t* v, uint8_t* tmp, long long bx, long long by, long long bz,
                              int r, cudaStream_t st) {
  const int T = 256;
  long long lines = by * bz;
  k_box_pass<<<(unsigned)((lines + T - 1) / T), T, 0, st>>>(v, tmp, bx, 1, lines, 0, bx, by, r);
  lines = bx * bz;
  k_box_pass<<<(unsigned)((lines + T - 1) / T), T, 0, st>>>(tmp, v, by, bx, lines, 1, bx, by, r);
  lines = bx * by;
  k_box_pass<<<(unsigned)((lines + T - 1) / T), T, 0, st>>>(v, tmp, bz, bx * by, lines, 2, bx, by,
                                                           r);
  return cudaMemcpyAsync(v, tmp, (size_t)(bx * by * bz), cudaMemcpyDeviceToDevice, st);
}

size_t voxelize_scratch_bytes(const VoxParams& p) {
  const size_t nb = (size_t)(p.bx * p.by * p.bz);
  return (size_t)(p.NY * p.NZ * p.wpr) * 4 + 10 * nb + 256;
}

cudaError_t launch_voxelize(VoxParams p, void* scratch, uint8_t* mask, cudaStream_t st) {
  const size_t nb = (size_t)(p.bx * p.by * p.bz);
  char* sc = static_cast<char*>(scratch);
  p.tog = reinterpret_cast<unsigned*>(sc);
  uint8_t* f = reinterpret_cast<uint8_t*>(sc + (size_t)(p.NY * p.NZ * p.wpr) * 4);
  uint8_t *in1 = f, *out1 = f + nb, *inK = f + 2 * nb, *outK = f + 3 * nb, *inS = f + 4 * nb,
          *outS = f + 5 * nb, *in2 = f + 6 * nb, *out2 = f + 7 * nb, *tmp = f + 8 * nb;
  cudaError_t e = cudaMemsetAsync(p.tog, 0, (size_t)(p.NY * p.NZ * p.wpr) * 4, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.words, 0, (size_t)p.W * 8, st);
  if (e != cudaSuccess) return e;
  const int T = 256;
  if (p.nt > 0)
    k_vox_tri<<<(unsigned)((p.nt * 32 + T - 1) / T), T, 0, st>>>(p);
  const long long rows = p.NY * p.NZ;
  k_vox_rows<<<(unsigned)((rows + T - 1) / T), T, 0, st>>>(p);
  k_vox_any<<<(unsigned)((nb + T - 1) / T), T, 0, st>>>(p, in1, out1);
  e = cudaMemcpyAsync(inK, in1, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(outK, out1, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(inS, in1, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(outS, out1, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(in2, in1, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out2, out1, nb, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  uint8_t* fields[8] = {in1, out1, inK, outK, inS, outS, in2, out2};
  const int radii[8] = {1, 1, kTileReach, kTileReach, kSubReach, kSubReach, 2, 2};
  for (int k = 0; k < 8; ++k) {
    e = box_or_dev(fields[k], tmp, p.bx, p.by, p.bz, radii[k], st);
    if (e != cudaSuccess) return e;
  }
  k_vox_mask<<<(unsigned)((nb + T - 1) / T), T, 0, st>>>(p.bx, p.by, p.bz, in1, out1, inK, outK,
                                                          inS, outS, in2, out2, mask);
  return cudaGetLastError();
}

}  // namespace psm
