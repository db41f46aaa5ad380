// k_collide.cuh — fused PSM stream-collide (arXiv 2502.20049, Eq.(4)) with the
// SRT fluid operator (Eq.(2)-(3)), the solid operators SC1/SC2/SC3
// (Eqs.(7)-(9)), B(eps) by Eq.(5)/(6) and the per-body
// force/torque partials of Eqs.(10)-(11), for sm_100a.
//
// One thread per cell, one 32x4x2 tile per 256-thread block, SoA f[q][z][y][x] (x fastest):
// every direction plane is read and written with coalesced 32-wide rows.  The kernel is
// HBM-bound (2*Q*S bytes per cell update); the PSM work is confined to tiles whose
// flag the mapping kernel set, so fluid tiles run the plain SRT path and never touch the solid
// words.  Streaming patterns (reading A10):
//   PAT 0  two-array pull : f_i(x) = A_i(x - c_i)  (wall: A_ibar(x)); write B_i(x) = f*_i(x)
//   PAT 1  AA even step   : f_i(x) = A[i][x];                      write A[ibar][x] = f*_i
//   PAT 2  AA odd step    : f_i(x) = A[ibar][x - c_i] (wall: A[i][x]);
//                           write A[i][x + c_i] = f*_i (wall: A[ibar][x])
#pragma once
#include <type_traits>

#include "psm_device.cuh"
#include "psm_internal.h"

// PSM_BOUNDS_CHECK (test builds only: PSM_NVCC_EXTRA=-DPSM_BOUNDS_CHECK): every element offset a
// kernel forms off a direction-plane base must stay inside that plane set; compute-sanitizer is
// not available on the GPU pool, so this is the out-of-bounds check of the parity suite
#if defined(PSM_BOUNDS_CHECK)
#include <cassert>
#define PSM_CHECK_OFF(off, n) assert((long long)(off) >= 0 && (long long)(off) < (long long)(n))
#else
#define PSM_CHECK_OFF(off, n) ((void)0)
#endif

namespace psm {

__device__ __forceinline__ double weight_fraction(double e, double tau, int mode) {
  // Eq.(6) in fp64, fixed operation order (bit-exact with the method definition, A14)
  if (mode == 0) return e;
  const double a = __dsub_rn(tau, 0.5);
  return __ddiv_rn(__dmul_rn(e, a), __dadd_rn(__dsub_rn(1.0, e), a));
}

// Deterministic per-tile reduction of the Eq.(10)-(11) summands without block barriers: each warp
// reduces its (at most) two smallest body ids with butterflies and parks the partials in shared
// memory; the warp that arrives last (shared counter, zeroed before the collision) combines them
// for the tile's two smallest ids in fixed warp order and writes the tile's slots.  A third or
// later body in one tile falls back to fp64 atomics in `overflow` (never happens unless bodies
// overlap one tile).  Slot layout in `out`: [id, v[0..11]] x 2.  Called by every thread of the
// block; no warp waits for another.
struct TileRed {
  unsigned cnt;
  double part[kTileCells / 32][2][1 + kSlotVals];  // per warp: [slot][id, values]
};

__device__ __forceinline__ void tile_partial_reduce(int myid, const double* v, double* out,
                                                    double* overflow, TileRed& sh) {
  constexpr unsigned FULL = 0xFFFFFFFFu, NONE = 0xFFFFFFFFu;
  constexpr int NW = kTileCells / 32;
  const int tid = threadIdx.x + kTileX * (threadIdx.y + kTileY * threadIdx.z);
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned me = myid ? (unsigned)myid : NONE;
  const unsigned k0 = __reduce_min_sync(FULL, me);
  const unsigned k1 = __reduce_min_sync(FULL, (me != k0) ? me : NONE);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const unsigned id = s == 0 ? k0 : k1;
    if (id != NONE) {
      // transpose butterfly: at each stage a lane keeps half of its values and receives the
      // partner's copy of that half, so the 12 (padded 16) sums take 16 shuffles instead of
      // 5 x 12; fixed order, so the result is deterministic.  Afterwards lane L (L even) holds
      // the sum of value ((L>>4)&1)*8 + ((L>>3)&1)*4 + ((L>>2)&1)*2 + ((L>>1)&1).
      double a[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = (k < kSlotVals && me == id) ? v[k < kSlotVals ? k : 0] : 0.0;
#pragma unroll
      for (int o = 16, n = 16; o > 1; o >>= 1, n >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < n / 2; ++k) {
          const double send = up ? a[k] : a[k + n / 2];
          const double keep = up ? a[k + n / 2] : a[k];
          a[k] = keep + __shfl_xor_sync(FULL, send, o);
        }
      }
      a[0] += __shfl_xor_sync(FULL, a[0], 1);
      const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                      ((lane >> 1) & 1);
      if (!(lane & 1) && idx < kSlotVals) sh.part[warp][s][1 + idx] = a[0];
    }
    if (lane == 0) sh.part[warp][s][0] = (id == NONE) ? -1.0 : (double)id;
  }
  if (me != NONE && me != k0 && me != k1)  // third+ body in this warp
    for (int k = 0; k < kSlotVals; ++k) atomicAdd(overflow + myid * kSlotVals + k, v[k]);
  __syncwarp();
  unsigned prev = 0;
  __threadfence_block();
  if (lane == 0) prev = atomicAdd(&sh.cnt, 1u);
  prev = __shfl_sync(FULL, prev, 0);
  if (prev != NW - 1) return;  // not the last warp of the tile
  __threadfence_block();
  // the tile's two smallest ids over every warp slot
  const double idl = lane < 2 * NW ? sh.part[lane >> 1][lane & 1][0] : -1.0;
  const unsigned key = idl >= 0.0 ? (unsigned)idl : NONE;
  const unsigned t0 = __reduce_min_sync(FULL, key);
  const unsigned t1 = __reduce_min_sync(FULL, (key != t0) ? key : NONE);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const unsigned id = s == 0 ? t0 : t1;
    double* o = out + s * (1 + kSlotVals);
    if (id == NONE) {
      if (lane == 0) o[0] = 0.0;
      continue;
    }
    if (lane < kSlotVals) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w)
        for (int t = 0; t < 2; ++t)
          if (sh.part[w][t][0] == (double)id) acc += sh.part[w][t][1 + lane];
      o[1 + lane] = acc;
    }
    if (lane == 0) o[0] = (double)id;
  }
  // a warp slot whose id is not one of the tile's two: its partial goes to the atomics
  if (lane < 2 * NW && key != NONE && key != t0 && key != t1)
    for (int k = 0; k < kSlotVals; ++k)
      atomicAdd(overflow + key * kSlotVals + k, sh.part[lane >> 1][lane & 1][1 + k]);
}

// explicitly rounded arithmetic: the fluid update must give the same bits wherever it runs
// (fluid tiles, B = 0 cells of PSM tiles, every slab decomposition)
__device__ __forceinline__ float rfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double rfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }

// c_i . u with compile-time c (adds/subtracts only)
template <typename T>
__device__ __forceinline__ T cdot(int q, T ux, T uy, T uz) {
  T r = T(0);
  bool first = true;
  if (stc_x(q)) { r = stc_x(q) > 0 ? ux : -ux; first = false; }
  if (stc_y(q)) { r = first ? (stc_y(q) > 0 ? uy : -uy) : (stc_y(q) > 0 ? radd(r, uy) : rsub(r, uy)); first = false; }
  if (stc_z(q)) { r = first ? (stc_z(q) > 0 ? uz : -uz) : (stc_z(q) > 0 ? radd(r, uz) : rsub(r, uz)); }
  return r;
}

// Guo source parts of the pair (i, ibar): symmetric w [-3 u.g + 9 (c.u)(c.g)], antisymmetric
// w 3 c.g (test-only forcing; TRT weights them with (1 - w+/2) and (1 - w-/2)).
template <int Q, typename T>
__device__ __forceinline__ void guo_pair(int i, T ux, T uy, T uz, const T (&g)[3], T& sp, T& sm) {
  const T cx = T(stc_x(i)), cy = T(stc_y(i)), cz = T(stc_z(i));
  const T cu = cx * ux + cy * uy + cz * uz;
  const T cg = cx * g[0] + cy * g[1] + cz * g[2];
  const T ug = ux * g[0] + uy * g[1] + uz * g[2];
  sp = T(stc_w<Q>(i)) * (T(-3) * ug + T(9) * cu * cg);
  sm = T(stc_w<Q>(i)) * (T(3) * cg);
}

// Plain SRT update of one cell, f* = f + omega (f^eq - f) (Eq.(1) with Eq.(2)-(3)), pairs
// (i, ibar) sharing f^eq_i = a + b, f^eq_ibar = a - b.  Explicitly rounded (see fluid_update).
template <int Q, typename T, bool FORCE>
__device__ __forceinline__ void srt_update(T (&f)[Q], T rho, T ux, T uy, T uz, T om,
                                           const T (&gl)[3]) {
  const T usq = rfma(uz, uz, rfma(uy, uy, rmul(ux, ux)));
  const T base = rsub(T(1), rmul(T(1.5), usq));
  const T gp = rsub(T(1), rmul(T(0.5), om));
  {
    T o0 = rmul(om, rsub(rmul(rmul(T(stc_w<Q>(0)), rho), base), f[0]));
    if (FORCE) {
      T sp, sm;
      guo_pair<Q, T>(0, ux, uy, uz, gl, sp, sm);
      o0 = radd(o0, rmul(gp, sp));
    }
    f[0] = radd(f[0], o0);
  }
#pragma unroll
  for (int i = 1; i < Q; ++i) {
    const int j = stc_opp(i);
    if (j < i) continue;
    const T cu = cdot<T>(i, ux, uy, uz);
    const T wr = rmul(T(stc_w<Q>(i)), rho);
    const T a = rmul(wr, rfma(rmul(T(4.5), cu), cu, base));
    const T b = rmul(wr, rmul(T(3), cu));
    T oi = rmul(om, rsub(radd(a, b), f[i]));
    T oj = rmul(om, rsub(rsub(a, b), f[j]));
    if (FORCE) {
      T sp, sm;
      guo_pair<Q, T>(i, ux, uy, uz, gl, sp, sm);
      oi = radd(oi, rmul(gp, radd(sp, sm)));
      oj = radd(oj, rmul(gp, rsub(sp, sm)));
    }
    f[i] = radd(f[i], oi);
    f[j] = radd(f[j], oj);
  }
}

// Fluid update of one cell, f* = f + Omega^F: SRT (Eq.(2)) or TRT, as pairs
// (i, ibar) with f^eq_i = a + b, f^eq_ibar = a - b, a = w rho (1 - 1.5 u.u + 4.5 (c.u)^2),
// b = 3 w rho c.u:  P = w+ (a - f+), M = w- (b - f-), f*_i = f_i + P + M, f*_ibar = f_ibar + P - M
// with f+- = (f_i +- f_ibar)/2.  SRT is w- = w+.  Every operation is explicitly rounded, so the
// update gives the same bits wherever it runs (fluid tiles, B = 0 cells of PSM tiles, any slab
// decomposition).
template <int Q, typename T, bool FORCE>
__device__ __forceinline__ void fluid_update(T (&f)[Q], T rho, T ux, T uy, T uz, T omp, T omm,
                                             const T (&gl)[3]) {
  const T usq = rfma(uz, uz, rfma(uy, uy, rmul(ux, ux)));
  const T base = rsub(T(1), rmul(T(1.5), usq));
  const T gp = rsub(T(1), rmul(T(0.5), omp)), gm = rsub(T(1), rmul(T(0.5), omm));
  {
    T o0 = rmul(omp, rsub(rmul(rmul(T(stc_w<Q>(0)), rho), base), f[0]));
    if (FORCE) {
      T sp, sm;
      guo_pair<Q, T>(0, ux, uy, uz, gl, sp, sm);
      o0 = radd(o0, rmul(gp, sp));
    }
    f[0] = radd(f[0], o0);
  }
#pragma unroll
  for (int i = 1; i < Q; ++i) {
    const int j = stc_opp(i);
    if (j < i) continue;
    const T cu = cdot<T>(i, ux, uy, uz);
    const T wr = rmul(T(stc_w<Q>(i)), rho);
    const T a = rmul(wr, rfma(rmul(T(4.5), cu), cu, base));
    const T b = rmul(wr, rmul(T(3), cu));
    const T fp = rmul(T(0.5), radd(f[i], f[j]));
    const T fm = rmul(T(0.5), rsub(f[i], f[j]));
    T P = rmul(omp, rsub(a, fp));
    T M = rmul(omm, rsub(b, fm));
    if (FORCE) {
      T sp, sm;
      guo_pair<Q, T>(i, ux, uy, uz, gl, sp, sm);
      P = radd(P, rmul(gp, sp));
      M = radd(M, rmul(gm, sm));
    }
    f[i] = radd(f[i], radd(P, M));
    f[j] = radd(f[j], rsub(P, M));
  }
}

// D3Q27 stencil index of the velocity (cx, cy, cz)
__host__ __device__ constexpr int idx27(int cx, int cy, int cz) {
  for (int q = 0; q < 27; ++q)
    if (stc_x(q) == cx && stc_y(q) == cy && stc_z(q) == cz) return q;
  return -1;
}

// 1-D backward central-moment transform along one axis with velocity v: (k0, k1, k2) are the
// central moments of orders 0, 1, 2 of the three populations c = -1, 0, +1.
template <typename T>
__device__ __forceinline__ void back1d(T k0, T k1, T k2, T v, T& fm, T& f0, T& fp) {
  const T m1 = k1 + v * k0;                   // raw first moment  f+ - f-
  const T m2 = k2 + v * (T(2) * k1 + v * k0);  // raw second moment f+ + f-
  f0 = k0 - m2;
  fp = T(0.5) * (m2 + m1);
  fm = T(0.5) * (m2 - m1);
}

// population of velocity (cx, cy, cz), zero for the D3Q27 corners a D3Q19 array does not hold
template <int Q, typename T>
__device__ __forceinline__ T fpop(const T (&f)[Q], int cx, int cy, int cz) {
  const int q = idx27(cx, cy, cz);
  return q < Q ? f[q < Q ? q : 0] : T(0);
}

// 1-D forward transform along one axis: (f-, f0, f+) -> raw moments of orders 0, 1, 2
template <typename T>
__device__ __forceinline__ void fwd1d(T fm, T f0, T fp, T& k0, T& k1, T& k2) {
  k2 = fp + fm;
  k0 = k2 + f0;
  k1 = fp - fm;
}

// Raw moments of orders <= 2 (rho, j, the six second moments) by factorised 1-D sums along z,
// y, then x — the forward transform restricted to what the cumulant operators use (the compiler
// drops the unused branches): ~66 additions for D3Q27 instead of ~170 with one sum per moment;
// the D3Q19 corners fold away.  mm = {rho, jx, jy, jz, mxx, myy, mzz, mxy, mxz, myz}.
template <int Q, typename T>
__device__ __forceinline__ void raw_moments2(const T (&f)[Q], T (&mm)[10]) {
  T zm[3][3][3], ym[3][3][3], xm[3][3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      fwd1d(fpop<Q, T>(f, a - 1, b - 1, -1), fpop<Q, T>(f, a - 1, b - 1, 0),
            fpop<Q, T>(f, a - 1, b - 1, 1), zm[a][b][0], zm[a][b][1], zm[a][b][2]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      fwd1d(zm[a][0][c], zm[a][1][c], zm[a][2][c], ym[a][0][c], ym[a][1][c], ym[a][2][c]);
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      fwd1d(ym[0][b][c], ym[1][b][c], ym[2][b][c], xm[0][b][c], xm[1][b][c], xm[2][b][c]);
  mm[0] = xm[0][0][0];
  mm[1] = xm[1][0][0];
  mm[2] = xm[0][1][0];
  mm[3] = xm[0][0][1];
  mm[4] = xm[2][0][0];
  mm[5] = xm[0][2][0];
  mm[6] = xm[0][0][2];
  mm[7] = xm[1][1][0];
  mm[8] = xm[1][0][1];
  mm[9] = xm[0][1][1];
}

// second raw moments: precomputed (PRE, raw_moments2 in the kernel prologue) or one sum each
template <int Q, typename T, bool PRE>
__device__ __forceinline__ void second_moments(const T (&f)[Q], const T (&pre)[6], T (&m2)[6]) {
  if constexpr (PRE) {
#pragma unroll
    for (int k = 0; k < 6; ++k) m2[k] = pre[k];
  } else {
#pragma unroll
    for (int k = 0; k < 6; ++k) m2[k] = T(0);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int cx = stc_x(q), cy = stc_y(q), cz = stc_z(q);
      if (cx) m2[0] += f[q];
      if (cy) m2[1] += f[q];
      if (cz) m2[2] += f[q];
      if (cx * cy > 0) m2[3] += f[q]; else if (cx * cy < 0) m2[3] -= f[q];
      if (cx * cz > 0) m2[4] += f[q]; else if (cx * cz < 0) m2[4] -= f[q];
      if (cy * cz > 0) m2[5] += f[q]; else if (cy * cz < 0) m2[5] -= f[q];
    }
  }
}

// Cumulant collision (the paper's performance operator), D3Q27, every rate of
// order >= 3 and the bulk rate equal to 1, shear rate omega: normalised second cumulants
// C = kappa / rho relaxed; post-collision central moments are those of a distribution whose
// cumulants of order >= 3 vanish (Wick products); three 1-D backward transforms give f*.
// (second raw moments m_ab from raw_moments2)
template <typename T, bool FORCE = false, bool PRE = true>
__device__ __forceinline__ void cumulant_update(T (&f)[27], T rho, T jx, T jy, T jz,
                                                const T (&m2pre)[6], T ux, T uy, T uz, T om,
                                                const T (&g)[3]) {
  T m2[6];
  second_moments<27, T, PRE>(f, m2pre, m2);
  const T mxx = m2[0], myy = m2[1], mzz = m2[2], mxy = m2[3], mxz = m2[4], myz = m2[5];
  const T ir = T(1) / rho;
  // second central moments about u: m_ab - u_a j_b - u_b j_a + rho u_a u_b, which is
  // m_ab - u_a j_b for u = j / rho; with a force u = (j + g/2)/rho (reading A31) and j_b is
  // replaced by j_b - g_b/2 in the first form
  T Cxx0, Cyy0, Czz0, Kxy, Kxz, Kyz;
  if constexpr (FORCE) {
    const T hx = T(0.5) * g[0], hy = T(0.5) * g[1], hz = T(0.5) * g[2];
    Cxx0 = (mxx - ux * (jx - hx)) * ir;
    Cyy0 = (myy - uy * (jy - hy)) * ir;
    Czz0 = (mzz - uz * (jz - hz)) * ir;
    Kxy = mxy - ux * jy + uy * hx;
    Kxz = mxz - ux * jz + uz * hx;
    Kyz = myz - uy * jz + uz * hy;
  } else {
    Cxx0 = (mxx - ux * jx) * ir;
    Cyy0 = (myy - uy * jy) * ir;
    Czz0 = (mzz - uz * jz) * ir;
    Kxy = mxy - ux * jy;
    Kxz = mxz - ux * jz;
    Kyz = myz - uy * jz;
  }
  const T w1 = T(1) - om;
  const T Cs = T(1);  // bulk rate 1: trace at its equilibrium 3 c_s^2
  const T D1 = w1 * (Cxx0 - Cyy0), D2 = w1 * (Cxx0 - Czz0);
  const T Cxy = w1 * Kxy * ir, Cxz = w1 * Kxz * ir, Cyz = w1 * Kyz * ir;
  const T Cxx = (Cs + D1 + D2) * T(1.0 / 3.0), Cyy = (Cs - T(2) * D1 + D2) * T(1.0 / 3.0),
          Czz = (Cs + D1 - T(2) * D2) * T(1.0 / 3.0);
  // post-collision central moments k[a][b][c] (orders a, b, c in x, y, z)
  T k[3][3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) k[a][b][c] = T(0);
  k[0][0][0] = rho;
  k[2][0][0] = rho * Cxx;
  k[0][2][0] = rho * Cyy;
  k[0][0][2] = rho * Czz;
  k[1][1][0] = rho * Cxy;
  k[1][0][1] = rho * Cxz;
  k[0][1][1] = rho * Cyz;
  k[2][2][0] = rho * (Cxx * Cyy + T(2) * Cxy * Cxy);
  k[2][0][2] = rho * (Cxx * Czz + T(2) * Cxz * Cxz);
  k[0][2][2] = rho * (Cyy * Czz + T(2) * Cyz * Cyz);
  k[2][1][1] = rho * (Cxx * Cyz + T(2) * Cxy * Cxz);
  k[1][2][1] = rho * (Cyy * Cxz + T(2) * Cxy * Cyz);
  k[1][1][2] = rho * (Czz * Cxy + T(2) * Cxz * Cyz);
  k[2][2][2] = rho * (Cxx * Cyy * Czz +
                      T(2) * (Cxx * Cyz * Cyz + Cyy * Cxz * Cxz + Czz * Cxy * Cxy) +
                      T(8) * Cxy * Cxz * Cyz);
  if constexpr (FORCE) {  // first-order central moments: -g/2 before, +g/2 after (A31)
    k[1][0][0] = T(0.5) * g[0];
    k[0][1][0] = T(0.5) * g[1];
    k[0][0][1] = T(0.5) * g[2];
  }
  // backward transforms x, then y, then z (the 1-D transforms commute)
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T fm, f0, fp;
      back1d(k[0][b][c], k[1][b][c], k[2][b][c], ux, fm, f0, fp);
      k[0][b][c] = fm;
      k[1][b][c] = f0;
      k[2][b][c] = fp;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T fm, f0, fp;
      back1d(k[a][0][c], k[a][1][c], k[a][2][c], uy, fm, f0, fp);
      k[a][0][c] = fm;
      k[a][1][c] = f0;
      k[a][2][c] = fp;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      T fm, f0, fp;
      back1d(k[a][b][0], k[a][b][1], k[a][b][2], uz, fm, f0, fp);
      f[idx27(a - 1, b - 1, -1)] = fm;
      f[idx27(a - 1, b - 1, 0)] = f0;
      f[idx27(a - 1, b - 1, 1)] = fp;
    }
}

// D3Q19 cumulant (reading A32; D3Q19 is the stencil of the paper's performance runs,
// PAPER.md:494): the 19 moments x^a y^b z^c (a, b, c <= 2, at least one order zero) that the
// D3Q19 velocity set carries.  Second cumulants as in the D3Q27 operator; the six third-order and
// three fourth-order cumulants of the set are set to 0, so the post-collision central moments
// are k_xxy = 0, k_xxyy = rho (C_xx C_yy + 2 C_xy^2).  Post-collision raw moments by the binomial
// shift about u (third central moments zero, first central moments +g/2 with a force, A31), then
// the populations by the closed-form inverse of the D3Q19 raw-moment map: an edge population of
// the (a, b) plane is (M_aabb + s_b M_aab + s_a M_abb + s_a s_b M_ab)/4, a face population
// ((M_aa - M_aabb - M_aacc) +- (M_a - M_abb - M_acc))/2, the rest population
// rho - sum M_aa + sum M_aabb.
template <typename T>
__device__ __forceinline__ void plane_raw(T u, T v, T ku, T kv, T kuv, T kuuvv, T hu, T hv, T rho,
                                          T& Muv, T& Muuv, T& Muvv, T& Muuvv) {
  const T uu = u * u, vv = v * v, uv = u * v;
  Muv = kuv + u * hv + v * hu + rho * uv;
  Muuv = v * ku + T(2) * u * kuv + T(2) * uv * hu + uu * hv + rho * uu * v;
  Muvv = u * kv + T(2) * v * kuv + T(2) * uv * hv + vv * hu + rho * u * vv;
  Muuvv = kuuvv + vv * ku + T(4) * uv * kuv + uu * kv + T(2) * u * vv * hu + T(2) * uu * v * hv +
          rho * uu * vv;
}

template <typename T, bool FORCE = false, bool PRE = true>
__device__ __forceinline__ void cumulant_update(T (&f)[19], T rho, T jx, T jy, T jz,
                                                const T (&m2pre)[6], T ux, T uy, T uz, T om,
                                                const T (&g)[3]) {
  T m2[6];
  second_moments<19, T, PRE>(f, m2pre, m2);
  const T mxx = m2[0], myy = m2[1], mzz = m2[2], mxy = m2[3], mxz = m2[4], myz = m2[5];
  const T ir = T(1) / rho;
  T Cxx0, Cyy0, Czz0, Kxy, Kxz, Kyz, hx = T(0), hy = T(0), hz = T(0);
  if constexpr (FORCE) {
    hx = T(0.5) * g[0];
    hy = T(0.5) * g[1];
    hz = T(0.5) * g[2];
    Cxx0 = (mxx - ux * (jx - hx)) * ir;
    Cyy0 = (myy - uy * (jy - hy)) * ir;
    Czz0 = (mzz - uz * (jz - hz)) * ir;
    Kxy = mxy - ux * jy + uy * hx;
    Kxz = mxz - ux * jz + uz * hx;
    Kyz = myz - uy * jz + uz * hy;
  } else {
    Cxx0 = (mxx - ux * jx) * ir;
    Cyy0 = (myy - uy * jy) * ir;
    Czz0 = (mzz - uz * jz) * ir;
    Kxy = mxy - ux * jy;
    Kxz = mxz - ux * jz;
    Kyz = myz - uy * jz;
  }
  const T w1 = T(1) - om;
  const T D1 = w1 * (Cxx0 - Cyy0), D2 = w1 * (Cxx0 - Czz0);
  const T Cxy = w1 * Kxy * ir, Cxz = w1 * Kxz * ir, Cyz = w1 * Kyz * ir;
  const T Cxx = (T(1) + D1 + D2) * T(1.0 / 3.0), Cyy = (T(1) - T(2) * D1 + D2) * T(1.0 / 3.0),
          Czz = (T(1) + D1 - T(2) * D2) * T(1.0 / 3.0);
  const T kxx = rho * Cxx, kyy = rho * Cyy, kzz = rho * Czz;
  const T kxy = rho * Cxy, kxz = rho * Cxz, kyz = rho * Cyz;
  const T kxxyy = rho * (Cxx * Cyy + T(2) * Cxy * Cxy);
  const T kxxzz = rho * (Cxx * Czz + T(2) * Cxz * Cxz);
  const T kyyzz = rho * (Cyy * Czz + T(2) * Cyz * Cyz);
  // post-collision raw moments
  const T Mx = rho * ux + hx, My = rho * uy + hy, Mz = rho * uz + hz;
  const T Mxx = kxx + T(2) * ux * hx + rho * ux * ux;
  const T Myy = kyy + T(2) * uy * hy + rho * uy * uy;
  const T Mzz = kzz + T(2) * uz * hz + rho * uz * uz;
  T Mxy, Mxxy, Mxyy, Mxxyy, Mxz, Mxxz, Mxzz, Mxxzz, Myz, Myyz, Myzz, Myyzz;
  plane_raw(ux, uy, kxx, kyy, kxy, kxxyy, hx, hy, rho, Mxy, Mxxy, Mxyy, Mxxyy);
  plane_raw(ux, uz, kxx, kzz, kxz, kxxzz, hx, hz, rho, Mxz, Mxxz, Mxzz, Mxxzz);
  plane_raw(uy, uz, kyy, kzz, kyz, kyyzz, hy, hz, rho, Myz, Myyz, Myzz, Myyzz);
  const T q4 = T(0.25);
#pragma unroll
  for (int sa = -1; sa <= 1; sa += 2)
#pragma unroll
    for (int sb = -1; sb <= 1; sb += 2) {
      const T A = T(sa), Bs = T(sb);
      f[idx27(sa, sb, 0)] = q4 * (Mxxyy + Bs * Mxxy + A * Mxyy + A * Bs * Mxy);
      f[idx27(sa, 0, sb)] = q4 * (Mxxzz + Bs * Mxxz + A * Mxzz + A * Bs * Mxz);
      f[idx27(0, sa, sb)] = q4 * (Myyzz + Bs * Myyz + A * Myzz + A * Bs * Myz);
    }
  const T Ax = Mxx - Mxxyy - Mxxzz, Bx = Mx - Mxyy - Mxzz;
  const T Ay = Myy - Mxxyy - Myyzz, By = My - Mxxy - Myzz;
  const T Az = Mzz - Mxxzz - Myyzz, Bz = Mz - Mxxz - Myyz;
  f[idx27(1, 0, 0)] = T(0.5) * (Ax + Bx);
  f[idx27(-1, 0, 0)] = T(0.5) * (Ax - Bx);
  f[idx27(0, 1, 0)] = T(0.5) * (Ay + By);
  f[idx27(0, -1, 0)] = T(0.5) * (Ay - By);
  f[idx27(0, 0, 1)] = T(0.5) * (Az + Bz);
  f[idx27(0, 0, -1)] = T(0.5) * (Az - Bz);
  f[0] = rho - (Mxx + Myy + Mzz) + (Mxxyy + Mxxzz + Myyzz);
}

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
  // read-only path with normal L2 allocation: the x-shifted rows of neighbouring tiles share
  // sectors in L2 (measured: __ldcs / __ldlu evict-first loads are 4 % slower, c5w and c4)
  return __ldg(p);
}

// AA pattern loads (the array is read and written in the same launch, but every location only
// by the thread that owns it, so the read-only path is legal too; tuning switch)
template <typename T>
__device__ __forceinline__ T aa_load(const T* p) {
#if defined(PSM_AA_LDG)
  return __ldg(p);
#elif defined(PSM_AA_LDCS)
  return __ldcs(p);
#elif defined(PSM_AA_LDCG)
  return __ldcg(p);
#else
  return *p;
#endif
}

// Minimum resident 256-thread blocks per SM (= register budget 65536 / (256 * n)): enough warps
// in flight to cover HBM latency without spilling the populations.
template <int Q, typename T, int PAT, int COLL, int WALLS>
constexpr int collide_min_blocks() {
  // fp64: two blocks (the populations alone are 2*Q registers)
#if defined(PSM_F64_Q19_BLOCKS)
  if (sizeof(T) == 8 && Q == 19) return PSM_F64_Q19_BLOCKS;
#endif
  if (sizeof(T) == 8) return 2;
  // D3Q27 AA odd step, periodic (destinations recomputed after the collision): three fp32
  // blocks at 80 registers (measured 88.2 -> 96.9 % SRT, 82.1 -> 90.6 % cumulant vs two)
  if (Q == 27 && PAT == 2 && !WALLS) return 3;
  // the D3Q27 cumulant keeps a 3x3x3 moment array live (PSM cells stash f in shared memory
  // instead of registers): three fp32 blocks, no spills (four spill 148 B; measured on one box
  // 88.1 % at four vs 93.8 % at three, fluid-only 384^3), AA odd with walls two
  if (COLL == 2 && Q == 27) return PAT == 2 ? 2 : 3;
  // D3Q19 (SRT, TRT, D3Q19 cumulant): four fp32 blocks; the AA odd step with walls keeps the
  // bounce-back selects live as well (three)
  if (Q == 19) return (PAT == 2 && WALLS) ? 3 : 4;
  // D3Q27 SRT/TRT: three (AA odd two)
  return PAT == 2 ? 2 : 3;
}

template <int WALLS>
__device__ __forceinline__ void stencil_offsets(const Geom& G, int xc, int yc, int zc, int (&OX)[3],
                                                int (&OY)[3], int (&OZ)[3], bool (&OUTX)[3],
                                                bool (&OUTY)[3], bool (&OUTZ)[3]) {
  const int nx = G.nx, ny = G.ny, plane = nx * ny;
  OX[0] = 1; OX[1] = 0; OX[2] = -1;
  OY[0] = nx; OY[1] = 0; OY[2] = -nx;
  OZ[0] = plane; OZ[1] = 0; OZ[2] = -plane;
#pragma unroll
  for (int a = 0; a < 3; ++a) OUTX[a] = OUTY[a] = OUTZ[a] = false;
  if (xc == 0) { if (WALLS && G.wall[0]) OUTX[2] = true; else OX[2] = nx - 1; }
  if (xc == nx - 1) { if (WALLS && G.wall[0]) OUTX[0] = true; else OX[0] = 1 - nx; }
  if (yc == 0) { if (WALLS == 1 && G.wall[1]) OUTY[2] = true; else OY[2] = (ny - 1) * nx; }
  if (yc == ny - 1) { if (WALLS == 1 && G.wall[1]) OUTY[0] = true; else OY[0] = (1 - ny) * nx; }
  if (G.zghost) {
    if (WALLS == 1 && G.wall[2]) {
      const int zg = G.z0 + zc;
      OUTZ[2] = (zg == 0);
      OUTZ[0] = (zg == G.nz_global - 1);
    }
  } else {
    if (zc == 0) { if (WALLS == 1 && G.wall[2]) OUTZ[2] = true; else OZ[2] = (G.nzl - 1) * plane; }
    if (zc == G.nzl - 1) { if (WALLS == 1 && G.wall[2]) OUTZ[0] = true; else OZ[0] = (1 - G.nzl) * plane; }
  }
}

// WALLS: 0 fully periodic; 1 runtime wall flags on every axis; 2 only x is non-periodic (open
// x faces or x walls) with y, z periodic — the y/z flag logic compiles out
// OCC = 1: one block per SM more for the fp64 D3Q19 kernels (85 registers, a few spills):
// measured +4 % when PSM tiles are frequent (c3 scenario A), -1.5 % fluid-only, so the host picks
// it from the PSM-tile fraction of the previous psm_step call
template <int Q, typename T, int PAT, int WALLS, bool FORCE, bool DBG, int COLL, int OCC = 0>
__global__ void __launch_bounds__(kTileCells,
                                  (collide_min_blocks<Q, T, PAT, COLL, WALLS>() +
                                   ((OCC && sizeof(T) == 8 && Q == 19) ? 1 : 0)))
    k_collide(const __grid_constant__ CollideParams p) {
  const Geom& G = p.g;
  const int x = blockIdx.x * kTileX + threadIdx.x;
  const int y = blockIdx.y * kTileY + threadIdx.y;
  const int tzl = blockIdx.z + p.tz0;
  const int z = tzl * kTileZ + threadIdx.z;
  const bool act = (x < G.nx) && (y < G.ny) && (z < G.nzl);
  const int tile = (tzl * G.gy + blockIdx.y) * G.gx + blockIdx.x;
  const bool solid_tile = DBG ? true : (p.tile_flag[tile] != 0);
  // PSM tiles, fp64: the cell's solid word is loaded now, with the populations, so its latency
  // is not exposed after the moments (measured: D3Q19 fp64 AA 95.7 -> 100.7 % fluid-only,
  // c5wpap 90.4 -> 96.5 %); the fp32 kernels lose occupancy with it and load it late
  constexpr bool kWordEarly = sizeof(T) == 8;
  // PSM tiles: every cell takes the fluid operator (uniform across the warp) and the solid-covered
  // cells keep their pre-collision f in a shared-memory stash for the Eq.(4) blend, instead of a
  // separate fluid path for the B = 0 lanes of a warp that also holds solid cells
#if defined(PSM_STASH_ALL)
  constexpr bool kStashAll = true;
#else
  constexpr bool kStashAll = COLL == 2;
#endif
  const uint32_t wpre = (kWordEarly && !DBG && solid_tile && act)
                            ? __ldg(p.word + (((long long)z * G.ny + y) * G.nx + x)) : 0u;

  const int nx = G.nx, ny = G.ny;
  const int plane = nx * ny;
  // inactive (ragged-tail) threads alias cell (0,0,0): their loads stay in bounds, no stores
  const int xc = act ? x : 0, yc = act ? y : 0, zc = act ? z : 0;
  const int zs = zc + G.zghost;  // storage plane
  const int self = zs * plane + yc * nx + xc;

  // Offsets (elements) from `self` to the SOURCE of a population with velocity component
  // d = -1, 0, +1 along each axis (the source is at coordinate - d), wrapped on periodic axes;
  // OUT* flags mark a source beyond a wall (half-way bounce-back, reading A23/A10).
  int OX[3], OY[3], OZ[3];
  bool OUTX[3], OUTY[3], OUTZ[3];
  stencil_offsets<WALLS>(G, xc, yc, zc, OX, OY, OZ, OUTX, OUTY, OUTZ);
  int RB[3][3];  // self + OY[cy] + OZ[cz]
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) RB[a][b] = self + OY[a] + OZ[b];

  // ---- gather the pre-collision populations f_i(x) ----
  T f[Q];
  auto gather = [&](auto with_walls) {
    constexpr bool W = decltype(with_walls)::value;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int cx = stc_x(q) + 1, cy = stc_y(q) + 1, cz = stc_z(q) + 1;
      const int src = RB[cy][cz] + OX[cx];
      const bool out = W && (OUTX[cx] || OUTY[cy] || OUTZ[cz]);
      const T* Aq = static_cast<const T*>(p.srcq[q]);
      const T* Ao = static_cast<const T*>(p.srcq[stc_opp(q)]);
      if (PAT == 0) {
        PSM_CHECK_OFF(out ? self : src, G.qstride);
        const T* ptr = out ? (Ao + self) : (Aq + src);
        f[q] = ld_stream(ptr);
      } else if (PAT == 1) {
        PSM_CHECK_OFF(self, G.qstride);
        f[q] = aa_load(Aq + self);
      } else {
        PSM_CHECK_OFF(out ? self : src, G.qstride);
        const T* ptr = out ? (Aq + self) : (Ao + src);
        f[q] = aa_load(ptr);
      }
    }
  };
  if constexpr (WALLS == 2) {
    // only x is non-periodic: the wall/open-face selects matter in the first and last tile
    // column alone (block-uniform branch), every other block runs the periodic gather
    if (blockIdx.x == 0 || blockIdx.x == G.gx - 1) gather(std::true_type{});
    else gather(std::false_type{});
  } else {
    gather(std::integral_constant<bool, (WALLS != 0)>{});
  }

  // PSM tiles: zero the arrival counter of the barrier-free F/T reduction (the one block barrier
  // of the kernel, while the gathered loads are still in flight)
  __shared__ TileRed s_tred;
  if (solid_tile) {
    if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) {
      s_tred.cnt = 0u;
    }
    __syncthreads();
  }

  // ---- open x faces (reading A30): the populations entering at x = 0 / nx-1 were gathered
  // from their bounce-back source A_qbar(x); apply the inflow / outflow rule ----
  if constexpr (WALLS && PAT == 0) {
    if (G.open_x) {
      if (xc == 0) {
        const T ux = T(p.u_in[0]), uy = T(p.u_in[1]), uz = T(p.u_in[2]);
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (stc_x(q) == 1)
            f[q] += T(6) * T(stc_w<Q>(q)) * (T(stc_x(q)) * ux + T(stc_y(q)) * uy +
                                             T(stc_z(q)) * uz);
      }
      if (xc == nx - 1) {
        T S0 = T(0), Sp = T(0);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          if (stc_x(q) == 0) S0 += f[q];
          if (stc_x(q) == 1) Sp += f[q];
        }
        const T ro = T(p.rho_out);
        const T ux = (S0 + T(2) * Sp) / ro - T(1);
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (stc_x(q) == -1)
            f[q] = T(2) * T(stc_w<Q>(q)) * ro * (T(1) + T(4.5) * ux * ux - T(1.5) * ux * ux) - f[q];
      }
    }
  }

  // ---- moments ----
  T rho, jx, jy, jz;
  T m2[6];  // second raw moments (cumulant only)
  // (D3Q19 AA: the second moments are summed inside the operator, as in the plain loop, which
  // measured 1-3 % faster there than the factorised sums in the prologue)
  constexpr bool kFactMoments = COLL == 2 && !(Q == 19 && PAT != 0);
  if constexpr (kFactMoments) {
    T mm[10];
    raw_moments2<Q, T>(f, mm);
    rho = mm[0];
    jx = mm[1];
    jy = mm[2];
    jz = mm[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) m2[k] = mm[4 + k];
  } else {
    rho = f[0];
    jx = jy = jz = T(0);
#pragma unroll
    for (int q = 1; q < Q; ++q) {
      rho += f[q];
      if (stc_x(q) > 0) jx += f[q]; else if (stc_x(q) < 0) jx -= f[q];
      if (stc_y(q) > 0) jy += f[q]; else if (stc_y(q) < 0) jy -= f[q];
      if (stc_z(q) > 0) jz += f[q]; else if (stc_z(q) < 0) jz -= f[q];
    }
  }
  if (act && !(rho > T(0) && rho < T(INFINITY))) {
    const long long cell = ((long long)(G.z0 + z) * G.ny + y) * (long long)G.nx + x;
    const long long ncell = (long long)G.nz_global * G.ny * G.nx;
    atomicMin(p.err, (unsigned long long)(p.step * ncell + cell));
  }
  T ir;
  if constexpr (sizeof(T) == 4) ir = __frcp_rn(rho); else ir = T(1) / rho;
  const T gl[3] = {T(p.gforce[0]), T(p.gforce[1]), T(p.gforce[2])};
  const T ux = FORCE ? rmul(rfma(T(0.5), gl[0], jx), ir) : rmul(jx, ir);
  const T uy = FORCE ? rmul(rfma(T(0.5), gl[1], jy), ir) : rmul(jy, ir);
  const T uz = FORCE ? rmul(rfma(T(0.5), gl[2], jz), ir) : rmul(jz, ir);
  const T usq15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
  const T om = T(p.omega), omm = T(p.omega_m);
  const T gpref = T(1) - T(0.5) * om, gmref = T(1) - T(0.5) * omm;

  // ---- fused halo + scatter (called once, from the fluid-tile or the PSM-tile path) ----
  auto store_all = [&]() {
    // ---- fused halo: the populations leaving the slab through z go straight into the
    // neighbours' ghost planes (peer stores over NVLink), replacing the separate exchange ----
    if (PAT == 0 && act && p.p2p) {  // (multi-rank runs are two-array only)
      const int pl = yc * nx + xc;
      PSM_CHECK_OFF(pl, (long long)nx * ny);
      if (z == G.nzl - 1) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (stc_z(q) > 0 && p.gup[q]) static_cast<T*>(p.gup[q])[pl] = f[q];
      }
      if (z == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (stc_z(q) < 0 && p.gdn[q]) static_cast<T*>(p.gdn[q])[pl] = f[q];
      }
    }

    // ---- scatter ----
    if constexpr (PAT == 2) {
      // AA odd step: the destination offsets are recomputed here instead of keeping the gather's
      // offsets live through the collision — register pressure sets this kernel's occupancy
      // (measured: fp64 SRT 92.3 -> 95.8 %, fp64 cumulant 88.4 -> 94.5 % of HBM; the fp32
      // kernels then fit four blocks per SM)
      int xr = xc, yr = yc, zr = zc;
      asm volatile("" : "+r"(xr), "+r"(yr), "+r"(zr));
      const int selfr = (zr + G.zghost) * plane + yr * nx + xr;
      int OXr[3], OYr[3], OZr[3];
      bool OUTXr[3], OUTYr[3], OUTZr[3];
      stencil_offsets<WALLS>(G, xr, yr, zr, OXr, OYr, OZr, OUTXr, OUTYr, OUTZr);
      if (act) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          // destination x + c_q == source position of the opposite direction
          const int cx = 1 - stc_x(q), cy = 1 - stc_y(q), cz = 1 - stc_z(q);
          const bool out = WALLS && (OUTXr[cx] || OUTYr[cy] || OUTZr[cz]);
          const int off = out ? selfr : selfr + OYr[cy] + OZr[cz] + OXr[cx];
          PSM_CHECK_OFF(off, G.qstride);
          static_cast<T*>(p.dstq[out ? stc_opp(q) : q])[off] = f[q];
        }
      }
    } else if (act) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        T* Dq = static_cast<T*>(p.dstq[q]);
        T* Do = static_cast<T*>(p.dstq[stc_opp(q)]);
        if (PAT == 0) {
          PSM_CHECK_OFF(self, G.qstride);
          Dq[self] = f[q];  // default write-back policy: measured 0.9 % faster than __stcs (c5w)
        } else {
          Do[self] = f[q];
        }
      }
    }
  };

  if (!solid_tile) {  // fluid tile: plain fluid operator, store, done
    if constexpr (COLL == 2)
      cumulant_update<T, FORCE, kFactMoments>(f, rho, jx, jy, jz, m2, ux, uy, uz, om, gl);
    else if (COLL == 1) fluid_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, omm, gl);
    else srt_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, gl);
    store_all();
    return;
  }
  // Eq.(10) summand m = B sum_i Omega^S_i c_i of this cell and its body (0: none); reduced per
  // tile after the scatter, so the block barriers of the reduction never hold back the stores
  double m[3] = {0.0, 0.0, 0.0};
  int myid = 0;
  {
    // ---- PSM cell: B, u_s from the solid word (or the test-only dense fields) ----
    int id = 0;
    double Bd = 0.0;
    double usd[3] = {0.0, 0.0, 0.0};
    double r[3] = {0.0, 0.0, 0.0};
    if (act) {
      if (DBG) {
        const long long c = ((long long)z * ny + y) * nx + x;
        Bd = p.dbg_B[c];
        id = p.dbg_id[c];
        const long long N = (long long)G.nzl * ny * nx;
        usd[0] = p.dbg_us[c];
        usd[1] = p.dbg_us[N + c];
        usd[2] = p.dbg_us[2 * N + c];
      } else {
        const uint32_t w = kWordEarly ? wpre : p.word[((long long)z * ny + y) * nx + x];
        id = (int)(w >> 16);
        if (id) {
          const int cnt = (int)(w & 0xFFFFu);
          const double e = ldexp((double)cnt, -3 * p.bodies[id].s);
          Bd = weight_fraction(e, p.tau, p.bmode);
        }
      }
      if (id) {
        const BodyKin& b = p.bodies[id];
        const double L[3] = {(double)nx, (double)ny, (double)G.nz_global};
        const double xcen[3] = {x + 0.5, y + 0.5, (double)(G.z0 + z) + 0.5};
#pragma unroll
        for (int a = 0; a < 3; ++a) r[a] = min_image(xcen[a] - b.t[a], L[a], !G.wall[a]);
        if (!DBG) {
          usd[0] = b.v[0] + (b.w[1] * r[2] - b.w[2] * r[1]);
          usd[1] = b.v[1] + (b.w[2] * r[0] - b.w[0] * r[2]);
          usd[2] = b.v[2] + (b.w[0] * r[1] - b.w[1] * r[0]);
        }
      }
    }
    // cumulant: every cell of the tile takes the fluid operator once, in place; a solid-covered
    // cell first puts its pre-collision f into a shared-memory stash ([q][thread], conflict-free)
    // so the PSM pair loop never holds both 27-vectors in registers (that peak would halve the
    // occupancy of every tile)
    T* stash = nullptr;
    int tid = 0;
    if constexpr (kStashAll) {
      extern __shared__ __align__(16) unsigned char smem_raw[];
      stash = reinterpret_cast<T*>(smem_raw);
      tid = threadIdx.x + kTileX * (threadIdx.y + kTileY * threadIdx.z);
      if (Bd > 0.0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) stash[q * kTileCells + tid] = f[q];
      }
      if constexpr (COLL == 2)
        cumulant_update<T, FORCE, kFactMoments>(f, rho, jx, jy, jz, m2, ux, uy, uz, om, gl);
      else if (COLL == 1) fluid_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, omm, gl);
      else srt_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, gl);
    }
    if (Bd > 0.0) {
      const T B = T(Bd), B1 = T(1) - T(Bd);
      const T sux = T(usd[0]), suy = T(usd[1]), suz = T(usd[2]);
      const T susq15 = T(1.5) * (sux * sux + suy * suy + suz * suz);
      T msx = T(0), msy = T(0), msz = T(0);
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int j = stc_opp(i);
        if (j < i) continue;  // each (i, ibar) pair once
        T fi = f[i], fj = f[j];
        T fci = fi, fcj = fj;  // fluid post-collision state (stash mode)
        if constexpr (kStashAll) {
          fi = stash[i * kTileCells + tid];
          fj = stash[j * kTileCells + tid];
        }
        // equilibria of the pair: f^eq_i = a + b, f^eq_ibar = a - b with a = w rho (1 - 1.5 u.u
        // + 4.5 (c.u)^2), b = 3 w rho c.u (Eq.(3)), for the fluid u and for u_s
        // (per-direction form for D3Q27 fp32 SRT/TRT: measured 97.6 vs 92.3 % on the AA step;
        // the pair form for every other variant, up to +16 % on the fp32 cumulant AA steps)
        T ei, ej, si, sj;
        if constexpr (COLL != 2 && Q == 27 && sizeof(T) == 4) {
          auto feq = [&](int q, T ux_, T uy_, T uz_, T u15) {
            const T c = T(stc_x(q)) * ux_ + T(stc_y(q)) * uy_ + T(stc_z(q)) * uz_;
            return T(stc_w<Q>(q)) * rho * (T(1) - u15 + c * (T(3) + T(4.5) * c));
          };
          ei = feq(i, ux, uy, uz, usq15);
          ej = feq(j, ux, uy, uz, usq15);
          si = feq(i, sux, suy, suz, susq15);
          sj = feq(j, sux, suy, suz, susq15);
        } else {
          const T wr = T(stc_w<Q>(i)) * rho;
          const T cu = cdot<T>(i, ux, uy, uz), cs = cdot<T>(i, sux, suy, suz);
          const T ae = wr * (T(1) - usq15 + T(4.5) * cu * cu), be = wr * (T(3) * cu);
          const T as = wr * (T(1) - susq15 + T(4.5) * cs * cs), bs = wr * (T(3) * cs);
          ei = ae + be;
          ej = ae - be;
          si = as + bs;
          sj = as - bs;
        }
        // fluid operator on the pair: SRT, or TRT on the symmetric/antisymmetric parts
        T oFi, oFj;
        if constexpr (kStashAll) {  // Omega^F from the fluid update every cell of the tile took
          oFi = fci - fi;
          oFj = fcj - fj;
        } else if (COLL == 1) {
          const T Pp = om * (T(0.5) * (ei + ej) - T(0.5) * (fi + fj));
          const T Mm = omm * (T(0.5) * (ei - ej) - T(0.5) * (fi - fj));
          oFi = Pp + Mm;
          oFj = Pp - Mm;
        } else {
          oFi = om * (ei - fi);
          oFj = om * (ej - fj);
        }
        if (FORCE && !kStashAll) {  // (with the stash the force is in fc; cumulant: A31)
          T sp, sm;
          guo_pair<Q, T>(i, ux, uy, uz, gl, sp, sm);
          oFi += gpref * sp + gmref * sm;
          oFj += gpref * sp - gmref * sm;
        }
        T oSi, oSj;
        if (p.sc == 1) {         // Eq.(7)
          oSi = (fj - ej) - (fi - si);
          oSj = (fi - ei) - (fj - sj);
        } else if (p.sc == 2) {  // Eq.(8) == -(f_i - f^eq_i(rho,u_s))/tau (reading A2)
          oSi = om * (si - fi);
          oSj = om * (sj - fj);
        } else {                 // Eq.(9)
          oSi = (fj - sj) - (fi - si);
          oSj = (fi - si) - (fj - sj);
        }
        f[i] = fi + B1 * oFi + B * oSi;
        if (j != i) {
          f[j] = fj + B1 * oFj + B * oSj;
          const T d = oSi - oSj;  // c_j = -c_i
          msx += T(stc_x(i)) * d;
          msy += T(stc_y(i)) * d;
          msz += T(stc_z(i)) * d;
        }
      }
      m[0] = Bd * (double)msx;
      m[1] = Bd * (double)msy;
      m[2] = Bd * (double)msz;
    } else {
      if constexpr (kStashAll) {
        // done above
      } else if (COLL == 1) fluid_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, omm, gl);
      else srt_update<Q, T, FORCE>(f, rho, ux, uy, uz, om, gl);
    }
    myid = (Bd > 0.0) ? id : 0;
  }

  store_all();
  // ---- per-body F/T partial of this tile (deterministic block reduction, Eqs.(10)-(11)) ----
  {
    double v[kSlotVals];
    double r[3] = {0.0, 0.0, 0.0};
    if (myid) {  // lever arm x_c - R, minimum image (reading A7)
      const BodyKin& b = p.bodies[myid];
      const double L[3] = {(double)nx, (double)ny, (double)G.nz_global};
      const double xcen[3] = {x + 0.5, y + 0.5, (double)(G.z0 + z) + 0.5};
#pragma unroll
      for (int a = 0; a < 3; ++a) r[a] = min_image(xcen[a] - b.t[a], L[a], !G.wall[a]);
    }
    v[0] = m[0]; v[1] = m[1]; v[2] = m[2];
    v[3] = r[1] * m[2] - r[2] * m[1];
    v[4] = r[2] * m[0] - r[0] * m[2];
    v[5] = r[0] * m[1] - r[1] * m[0];
#pragma unroll
    for (int a = 0; a < 6; ++a) v[6 + a] = fabs(v[a]);
    tile_partial_reduce(myid, v, p.partial + (size_t)tile * 2 * (1 + kSlotVals), p.overflow,
                        s_tred);
  }
}

// ------------------------------------------------------------------------------ launcher ---
template <int Q, typename T>
cudaError_t launch_variant(const CollideParams& p, int pat, bool force, bool dbg,
                                  dim3 grid, dim3 block, cudaStream_t st);

template <int Q, typename T>
cudaError_t launch_t(const CollideParams& p, int pat, bool force, bool dbg, int ntz,
                            cudaStream_t st) {
  if (ntz <= 0) return cudaSuccess;
  dim3 grid(p.g.gx, p.g.gy, ntz), block(kTileX, kTileY, kTileZ);
  CollideParams pq = p;
  for (int q = 0; q < Q; ++q) {
    pq.srcq[q] = static_cast<const T*>(p.src) + (size_t)q * p.g.qstride;
    pq.dstq[q] = static_cast<T*>(p.dst) + (size_t)q * p.g.qstride;
  }
  return launch_variant<Q, T>(pq, pat, force, dbg, grid, block, st);
}

// One kernel instantiation: dynamic shared memory for the PSM-cell stash (when the variant uses
// it), with the > 48 KB opt-in set once per instantiation and device (bit per device ordinal).
template <int Q, typename T, int PAT, int WALLS, bool FORCE, bool DBG, int COLL, int OCC = 0>
cudaError_t launch_k(const CollideParams& p, dim3 grid, dim3 block, cudaStream_t st) {
#if defined(PSM_STASH_ALL)
  constexpr bool stash = true;
#else
  constexpr bool stash = COLL == 2;
#endif
  constexpr size_t sm = stash ? (size_t)Q * kTileCells * sizeof(T) : 0;
  if constexpr (sm > 48 * 1024) {
    static unsigned long long attr_devices = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_devices & bit)) {
      e = cudaFuncSetAttribute(k_collide<Q, T, PAT, WALLS, FORCE, DBG, COLL, OCC>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      attr_devices |= bit;
    }
  }
  k_collide<Q, T, PAT, WALLS, FORCE, DBG, COLL, OCC><<<grid, block, sm, st>>>(p);
  return cudaGetLastError();
}

// the variant for the context's operator, pattern, boundaries and test switches
template <int Q, typename T, int COLL>
cudaError_t launch_coll(const CollideParams& p, int pat, bool force, bool dbg, dim3 grid,
                        dim3 block, cudaStream_t st) {
  const bool walls = p.g.wall[0] || p.g.wall[1] || p.g.wall[2];
  const bool xonly = p.g.wall[0] && !p.g.wall[1] && !p.g.wall[2];  // e.g. open x faces
  // body force / debug fields: general two-array variants only
  if (dbg && force) return launch_k<Q, T, 0, 1, true, true, COLL>(p, grid, block, st);
  if (dbg) return launch_k<Q, T, 0, 1, false, true, COLL>(p, grid, block, st);
  if (force) return launch_k<Q, T, 0, 1, true, false, COLL>(p, grid, block, st);
  if constexpr (Q == 19 && sizeof(T) == 8) {  // periodic fast paths at higher occupancy
    if (p.hiocc && !walls) {
      if (pat == 0) return launch_k<Q, T, 0, 0, false, false, COLL, 1>(p, grid, block, st);
      if (pat == 1) return launch_k<Q, T, 1, 0, false, false, COLL, 1>(p, grid, block, st);
      return launch_k<Q, T, 2, 0, false, false, COLL, 1>(p, grid, block, st);
    }
  }
  if (pat == 0) {
    if (!walls) return launch_k<Q, T, 0, 0, false, false, COLL>(p, grid, block, st);
    if (xonly) return launch_k<Q, T, 0, 2, false, false, COLL>(p, grid, block, st);
    return launch_k<Q, T, 0, 1, false, false, COLL>(p, grid, block, st);
  }
  if (pat == 1) return launch_k<Q, T, 1, 0, false, false, COLL>(p, grid, block, st);
  if (walls) return launch_k<Q, T, 2, 1, false, false, COLL>(p, grid, block, st);
  return launch_k<Q, T, 2, 0, false, false, COLL>(p, grid, block, st);
}

template <int Q, typename T>
cudaError_t launch_variant(const CollideParams& p, int pat, bool force, bool dbg, dim3 grid,
                           dim3 block, cudaStream_t st) {
  if (p.trt == 1) return launch_coll<Q, T, 1>(p, pat, force, dbg, grid, block, st);
  if (p.trt == 2) return launch_coll<Q, T, 2>(p, pat, force, dbg, grid, block, st);
  return launch_coll<Q, T, 0>(p, pat, force, dbg, grid, block, st);
}

// one translation unit per (Q, T) instantiates the kernel variants (parallel build)
cudaError_t launch_collide_19f(const CollideParams& p, int pat, bool force, bool dbg, int ntz, cudaStream_t st);
cudaError_t launch_collide_19d(const CollideParams& p, int pat, bool force, bool dbg, int ntz, cudaStream_t st);
cudaError_t launch_collide_27f(const CollideParams& p, int pat, bool force, bool dbg, int ntz, cudaStream_t st);
cudaError_t launch_collide_27d(const CollideParams& p, int pat, bool force, bool dbg, int ntz, cudaStream_t st);

}  // namespace psm
