// k_state.cu — state conversion, fraction readback and force/torque reduction kernels.
//
// The ABI always exchanges the Eq.(4) state (pre-collision f_i(x,t)) in fp64;
// storage is pattern-specific (reading A10):
//   pull  : f_i(x) = A_i(x - c_i); at a wall face where x - c_i is outside, f_i(x) = A_ibar(x).
//           Inversely a slot A_j(y) holds f_j(y + c_j), or f_jbar(y) if y + c_j crosses a wall.
//   AA    : even step count: f_i(x) = A[i][x]; odd: f_i(x) = A[ibar][x - c_i] (wall: A[i][x]).
// Conversions are z-chunked through an fp64 staging buffer so arbitrarily large grids stream
// through a bounded device buffer.
#include "psm_device.cuh"
#include "psm_internal.h"

namespace psm {

template <int Q>
__device__ __forceinline__ double feq_d(int q, double rho, double ux, double uy, double uz) {
  const double cu = stc_x(q) * ux + stc_y(q) * uy + stc_z(q) * uz;
  const double usq = ux * ux + uy * uy + uz * uz;
  return stc_w<Q>(q) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
}

// wrap/clip a neighbour coordinate; returns false if it leaves through a wall (or, in ghost
// mode for z, if it is not a stored plane)
__device__ __forceinline__ bool nb_coord(int c, int n, bool wall, int& out) {
  if (c < 0 || c >= n) {
    if (wall) return false;
    c = (c + n) % n;
  }
  out = c;
  return true;
}

// Reading A30 (open x faces), in the pull form f_q(x) = rule(A_qbar(x)) for the populations
// entering through a face:
//   inflow  x = 0,      c_qx = +1: f_q = A_qbar + ubb_q,             ubb_q = 6 w_q (c_q . u_in)
//   outflow x = nx - 1, c_qx = -1: f_q = -A_qbar + abb_q(u_x),
//           abb_q = 2 w_q rho_out (1 + 4.5 (c_qx u_x)^2 - 1.5 u_x^2),
//           u_x = (S_0 + 2 S_+) / rho_out - 1 over the cell's known populations (c_x >= 0).
template <int Q>
__device__ __forceinline__ double open_ubb(int q, const double* u_in) {
  return 6.0 * stc_w<Q>(q) * (stc_x(q) * u_in[0] + stc_y(q) * u_in[1] + stc_z(q) * u_in[2]);
}
template <int Q>
__device__ __forceinline__ double open_abb(int q, double ux, double rho_out) {
  const double cu = stc_x(q) * ux;
  return 2.0 * stc_w<Q>(q) * rho_out * (1.0 + 4.5 * cu * cu - 1.5 * ux * ux);
}

template <int Q, typename T>
__global__ void k_write_state(const StateParams p) {
  const Geom& G = p.g;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  // storage planes handled: [za, zb) plus adjacent ghost planes when requested
  const int lo = (p.ghosts && p.za == 0) ? -1 : p.za;
  const int hi = (p.ghosts && p.zb == G.nzl) ? G.nzl + 1 : p.zb;
  const int z = lo + (int)blockIdx.z;
  if (x >= G.nx || z >= hi) return;
  T* A = static_cast<T*>(p.A);
  const long long plane = (long long)G.nx * G.ny;
  const long long slot = ((long long)(z + G.zghost) * G.ny + y) * G.nx + x;
  auto fetch = [&](int d, int rx, int ry, int rz) -> double {
    // value f_d at local reader cell (rx, ry, rz) from the staging buffer
    int k = rz - p.stage_z0;
    if (k < 0) k += G.nzl;
    if (k >= p.stage_nz) k -= G.nzl;
    const long long c = ((long long)k * G.ny + ry) * G.nx + rx;
    const long long sp = (long long)p.stage_nz * plane;
    if (p.mode == 0) return p.stage[d * sp + c];
    if (p.mode == 1)
      return feq_d<Q>(d, p.stage[c], p.stage[sp + c], p.stage[2 * sp + c], p.stage[3 * sp + c]);
    return stc_w<Q>(d);
  };
  const bool ghost_plane = (z < 0 || z >= G.nzl);
  for (int j = 0; j < Q; ++j) {
    if (p.pattern == 1) {  // AA after a write: even, A[j][x] = f_j(x)
      if (ghost_plane) continue;
      A[j * G.qstride + slot] = (T)fetch(j, x, y, z);
      continue;
    }
    // A30: a slot whose reader y + c_j lies beyond an open x face is the source of the entering
    // population q = jbar at y itself; invert the face rule
    if (G.open_x && (x + stc_x(j) < 0 || x + stc_x(j) >= G.nx)) {
      if (ghost_plane) continue;
      const int q = stc_opp(j);
      double v;
      if (stc_x(j) < 0) {
        v = fetch(q, x, y, z) - open_ubb<Q>(q, p.u_in);
      } else {
        double S0 = 0.0, Sp = 0.0;
        for (int i = 0; i < Q; ++i) {
          if (stc_x(i) == 0) S0 += fetch(i, x, y, z);
          if (stc_x(i) == 1) Sp += fetch(i, x, y, z);
        }
        const double ux = (S0 + 2.0 * Sp) / p.rho_out - 1.0;
        v = open_abb<Q>(q, ux, p.rho_out) - fetch(q, x, y, z);
      }
      A[j * G.qstride + slot] = (T)v;
      continue;
    }
    // the slot is read by y + c_j, or by y itself (bounce) if y + c_j crosses a wall
    int rx = 0, ry = 0, rz = 0;
    bool wall_cross = !nb_coord(x + stc_x(j), G.nx, G.wall[0], rx);
    wall_cross |= !nb_coord(y + stc_y(j), G.ny, G.wall[1], ry);
    bool remote = false;
    if (G.zghost) {
      rz = z + stc_z(j);
      const int zg = G.z0 + rz;
      if (G.wall[2] && (zg < 0 || zg >= G.nz_global))
        wall_cross = true;
      else if (rz < 0 || rz >= G.nzl)
        remote = true;  // the reader lives on another rank
    } else {
      wall_cross |= !nb_coord(z + stc_z(j), G.nzl, G.wall[2], rz);
    }
    double v;
    if (wall_cross) {
      if (ghost_plane) continue;
      v = fetch(stc_opp(j), x, y, z);  // bounce slot: read back as f_jbar(y)
    } else {
      if (remote) continue;
      v = fetch(j, rx, ry, rz);
    }
    A[j * G.qstride + slot] = (T)v;
  }
}

template <int Q, typename T>
__global__ void k_read_state(const StateParams p) {
  const Geom& G = p.g;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int z = p.za + (int)blockIdx.z;
  if (x >= G.nx || z >= p.zb) return;
  const T* A = static_cast<const T*>(p.A);
  const int zs = z + G.zghost;
  const long long self = ((long long)zs * G.ny + y) * G.nx + x;
  const long long sp = (long long)p.stage_nz * G.nx * G.ny;
  const long long c = ((long long)(z - p.stage_z0) * G.ny + y) * G.nx + x;
  double fq[Q];
  for (int q = 0; q < Q; ++q) {
    double v;
    if (p.pattern == 1 && !p.odd) {
      v = (double)A[q * G.qstride + self];
    } else {
      int sx, sy, sz;
      bool in = nb_coord(x - stc_x(q), G.nx, G.wall[0], sx) &&
                nb_coord(y - stc_y(q), G.ny, G.wall[1], sy);
      if (G.zghost) {
        const int zg = G.z0 + z - stc_z(q);
        if (G.wall[2] && (zg < 0 || zg >= G.nz_global)) in = false;
        sz = zs - stc_z(q);
      } else {
        in = in && nb_coord(z - stc_z(q), G.nzl, G.wall[2], sz);
      }
      const long long src = ((long long)sz * G.ny + sy) * G.nx + sx;
      if (p.pattern == 0)
        v = in ? (double)A[q * G.qstride + src] : (double)A[stc_opp(q) * G.qstride + self];
      else
        v = in ? (double)A[stc_opp(q) * G.qstride + src] : (double)A[q * G.qstride + self];
    }
    fq[q] = v;
  }
  if (G.open_x && x == 0) {  // A30 inflow
    for (int q = 0; q < Q; ++q)
      if (stc_x(q) == 1) fq[q] += open_ubb<Q>(q, p.u_in);
  }
  if (G.open_x && x == G.nx - 1) {  // A30 outflow: fq[q] holds A_qbar(x) for c_qx = -1
    double S0 = 0.0, Sp = 0.0;
    for (int q = 0; q < Q; ++q) {
      if (stc_x(q) == 0) S0 += fq[q];
      if (stc_x(q) == 1) Sp += fq[q];
    }
    const double ux = (S0 + 2.0 * Sp) / p.rho_out - 1.0;
    for (int q = 0; q < Q; ++q)
      if (stc_x(q) == -1) fq[q] = open_abb<Q>(q, ux, p.rho_out) - fq[q];
  }
  double rho = 0, j[3] = {0, 0, 0};
  for (int q = 0; q < Q; ++q) {
    const double v = fq[q];
    if (p.mode == 0) {
      p.stage[q * sp + c] = v;
    } else {
      rho += v;
      j[0] += stc_x(q) * v;
      j[1] += stc_y(q) * v;
      j[2] += stc_z(q) * v;
    }
  }
  if (p.mode == 1) {
    p.stage[c] = rho;
    for (int a = 0; a < 3; ++a) p.stage[(a + 1) * sp + c] = j[a] / rho;
  }
}

template <int Q, typename T>
static cudaError_t write_t(const StateParams& p, cudaStream_t st) {
  const int lo = (p.ghosts && p.za == 0) ? -1 : p.za;
  const int hi = (p.ghosts && p.zb == p.g.nzl) ? p.g.nzl + 1 : p.zb;
  if (hi <= lo) return cudaSuccess;
  dim3 grid((p.g.nx + 127) / 128, p.g.ny, hi - lo);
  k_write_state<Q, T><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}
template <int Q, typename T>
static cudaError_t read_t(const StateParams& p, cudaStream_t st) {
  if (p.zb <= p.za) return cudaSuccess;
  dim3 grid((p.g.nx + 127) / 128, p.g.ny, p.zb - p.za);
  k_read_state<Q, T><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_write_state(int Q, bool fp64, const StateParams& p, cudaStream_t st) {
  if (Q == 19) return fp64 ? write_t<19, double>(p, st) : write_t<19, float>(p, st);
  return fp64 ? write_t<27, double>(p, st) : write_t<27, float>(p, st);
}
cudaError_t launch_read_state(int Q, bool fp64, const StateParams& p, cudaStream_t st) {
  if (Q == 19) return fp64 ? read_t<19, double>(p, st) : read_t<19, float>(p, st);
  return fp64 ? read_t<27, double>(p, st) : read_t<27, float>(p, st);
}

// ------------------------------------------------------------------ fraction readback -------
__global__ void k_read_fractions(const FracParams p) {
  const Geom& G = p.g;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int z = p.za + (int)blockIdx.z;
  if (x >= G.nx || z >= p.zb) return;
  const long long c = ((long long)z * G.ny + y) * G.nx + x;
  const long long o = ((long long)(z - p.za) * G.ny + y) * G.nx + x;
  const uint32_t w = p.word[c];
  const int id = (int)(w >> 16), cnt = (int)(w & 0xFFFFu);
  double B = 0.0;
  if (id) {
    const double e = ldexp((double)cnt, -3 * p.s[id]);
    if (p.bmode == 0) {
      B = e;
    } else {
      const double a = __dsub_rn(p.tau, 0.5);
      B = __ddiv_rn(__dmul_rn(e, a), __dadd_rn(__dsub_rn(1.0, e), a));
    }
  }
  if (p.B) p.B[o] = B;
  if (p.id) p.id[o] = (uint8_t)id;
  if (p.cnt) p.cnt[o] = cnt;
}

cudaError_t launch_read_fractions(const FracParams& p, cudaStream_t st) {
  if (p.zb <= p.za) return cudaSuccess;
  dim3 grid((p.g.nx + 127) / 128, p.g.ny, p.zb - p.za);
  k_read_fractions<<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}

// -------------------------------------------------------- force/torque reduction -----------
// Pass 1: block (g, b) sums body b's slots over tile chunk g in a fixed order; pass 2 sums the
// chunks in order and adds the overflow accumulator.  Deterministic for a given tile grid.
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads)
    k_ft_pass1(const uint8_t* flag, const double* partial, int ntiles, const int* ids,
               double* scratch, int nchunks) {
  const int g = blockIdx.x, b = blockIdx.y;
  const int id = ids[b];
  const int per = (ntiles + nchunks - 1) / nchunks;
  const int t0 = g * per, t1 = min(ntiles, t0 + per);
  double acc[kSlotVals];
  for (int k = 0; k < kSlotVals; ++k) acc[k] = 0.0;
  for (int t = t0 + (int)threadIdx.x; t < t1; t += kRedThreads) {
    if (!flag[t]) continue;
    const double* P = partial + (size_t)t * 2 * (1 + kSlotVals);
    for (int s = 0; s < 2; ++s) {
      if ((int)P[s * (1 + kSlotVals)] == id)
        for (int k = 0; k < kSlotVals; ++k) acc[k] += P[s * (1 + kSlotVals) + 1 + k];
    }
  }
  __shared__ double red[kRedThreads];
  for (int k = 0; k < kSlotVals; ++k) {
    red[threadIdx.x] = acc[k];
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) scratch[((size_t)b * nchunks + g) * kSlotVals + k] = red[0];
    __syncthreads();
  }
}

__global__ void k_ft_pass2(const double* scratch, int nchunks, const double* overflow,
                           const int* ids, int nb, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb * kSlotVals) return;
  const int b = i / kSlotVals, k = i % kSlotVals;
  double acc = 0.0;
  for (int g = 0; g < nchunks; ++g) acc += scratch[((size_t)b * nchunks + g) * kSlotVals + k];
  acc += overflow[ids[b] * kSlotVals + k];
  out[i] = acc;
}

cudaError_t launch_ft_reduce(const uint8_t* tile_flag, const double* partial, int ntiles,
                             const double* overflow, const int* ids, int nb, double* scratch,
                             int nchunks, double* out, cudaStream_t st) {
  if (nb <= 0) return cudaSuccess;
  k_ft_pass1<<<dim3(nchunks, nb), kRedThreads, 0, st>>>(tile_flag, partial, ntiles, ids,
                                                         scratch, nchunks);
  k_ft_pass2<<<(nb * kSlotVals + 127) / 128, 128, 0, st>>>(scratch, nchunks, overflow, ids, nb,
                                                            out);
  return cudaGetLastError();
}

}  // namespace psm
