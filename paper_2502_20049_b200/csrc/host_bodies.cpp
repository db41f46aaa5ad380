// host_bodies.cpp — rigid-body pose arithmetic on the host (closed-form advance, A13),
// remap boxes, and the two-way coupling integrator (reading A28).
#include "psm_ctx.h"

namespace psm {

// ---------------------------------------------------------------------------- helpers ------
void free_bands(Body& b) {  // callers have synchronised the streams
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

void rodrigues(const double w[3], double n, const double Q0[9], double out[9]) {
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

double extent(const psm_ctx* c, int a) {
  return (double)(a == 0 ? c->grid.nx : (a == 1 ? c->grid.ny : c->grid.nz));
}

void pose_at(const psm_ctx* c, const Body& b, int64_t step, double Q[9], double t[3]) {
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
void body_box(const psm_ctx* c, const Body& b, const double Q[9], const double t[3],
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
int axis_pieces(const psm_ctx* c, int a, int64_t lo, int64_t hi, int64_t out[2][2]) {
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

void add_box(const psm_ctx* c, const int64_t lo[3], const int64_t hi[3],
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
void remap_region(const psm_ctx* c, Body& b, const double Q[9], const double t[3],
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

// Semi-implicit Euler step of a dynamic body with the force/torque ON it from the step just
// completed (the oracle implements the same formulas independently).
void integrate_body(const psm_ctx* c, Body& b, const double F[3], const double T[3]) {
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

}  // namespace psm
