/*
 * psm_oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, fp64 CPU oracle of the PSM lattice
 * Boltzmann hot path of arXiv 2502.20049 (Suffa et al.).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2502_20049_b200/) never links, imports or calls anything in this directory, and this
 * file shares no code, header, table or helper with it.
 *
 * It runs the method itself, step by step, in the paper's notation:
 *   Eq.(1)  LB update
 *   Eq.(2)  SRT collision
 *   Eq.(3)  equilibrium             PAPER.md:138-140  (u^2 term with "-", reading A1)
 *   Eq.(4)  PSM update rule
 *   Eq.(5)  B = eps
 *   Eq.(6)  tau-weighted B
 *   Eq.(7)-(9) SC1/SC2/SC3          PAPER.md:178-189  (SC2 in its literal printed form, A2)
 *   Eq.(10)-(11) force / torque     PAPER.md:196-204  (returned with the sign ON the body, A6)
 *   Sec. III geometry field + super-sampled fraction mapping, PAPER.md:299-321 (reading R1, A12;
 *           the literal centre-only reading R2 selectable per mesh)
 * and the NEXT rows built on the same hot path:
 *   TRT fluid operator (listed; reading A27)
 *   cumulant fluid operator, D3Q27 and D3Q19 (readings A29, A32, A31 with a
 *           body force)
 *   velocity inflow / pressure outflow on the x faces (reading A30)
 *   two-way coupling of dynamic bodies (reading A28, optional virtual mass)
 * The readings taken where the paper is silent or garbled are listed in DESIGN.md §3
 * (A1..A34); each use below names its reading.
 *
 * State convention (A10): f holds the Eq.(4) state, i.e. the PRE-collision populations
 * f_i(x,t).  One step = collide every cell, then push f*_i(x) to x + c_i.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (no FMA contraction; explicit fma()
 * only where reading A14 fixes it).  Parallelism: OpenMP over z planes only; every reduction is
 * done per z-plane and then summed in plane order, so results do not depend on thread count.
 *
 * Parity status: every function here is pinned by a test in tests/test_oracle_*.py
 * (DESIGN.md §4 lists the pin for each); none is "parity unpinned" except the absolute drag
 * magnitude (P12(iii)), which the paper does not print.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXB 16

/* ---------------------------------------------------------------- stencils --
 * Order is fixed by our ABI (lbmpy/waLBerla convention; the paper lists stencils only by name,
 * PAPER.md:233).  Weights are the standard D3Q19/D3Q27 ones (sum 1, second moment c_s^2 = 1/3). */
static const int C19[19][3] = {
    {0, 0, 0},  {0, 1, 0},  {0, -1, 0}, {-1, 0, 0}, {1, 0, 0},  {0, 0, 1},   {0, 0, -1},
    {-1, 1, 0}, {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {0, 1, 1},  {0, -1, 1},  {-1, 0, 1},
    {1, 0, 1},  {0, 1, -1}, {0, -1, -1}, {-1, 0, -1}, {1, 0, -1}};
static const int C27x[8][3] = {{1, 1, 1},  {-1, 1, 1},  {1, -1, 1},  {-1, -1, 1},
                               {1, 1, -1}, {-1, 1, -1}, {1, -1, -1}, {-1, -1, -1}};

static void stencil_c(int Q, int i, int c[3]) {
  const int* src = (i < 19) ? C19[i] : C27x[i - 19];
  c[0] = src[0];
  c[1] = src[1];
  c[2] = src[2];
  (void)Q;
}

static double stencil_w(int Q, int i) {
  int c[3];
  stencil_c(Q, i, c);
  int n = abs(c[0]) + abs(c[1]) + abs(c[2]); /* 0 rest, 1 face, 2 edge, 3 corner */
  if (Q == 19) {
    if (n == 0) return 1.0 / 3.0;
    if (n == 1) return 1.0 / 18.0;
    return 1.0 / 36.0;
  }
  if (n == 0) return 8.0 / 27.0;
  if (n == 1) return 2.0 / 27.0;
  if (n == 2) return 1.0 / 54.0;
  return 1.0 / 216.0;
}

/* i-bar: the direction with c_ibar = -c_i, found by search. */
static int stencil_opp(int Q, int i) {
  int c[3], d[3];
  stencil_c(Q, i, c);
  for (int j = 0; j < Q; ++j) {
    stencil_c(Q, j, d);
    if (d[0] == -c[0] && d[1] == -c[1] && d[2] == -c[2]) return j;
  }
  return -1;
}

/* Tables computed once from the definitions above (plain lookups in the per-cell loops). */
static int TC[28][27][3], TOPP[28][27];
static double TW[28][27];
static int tables_ready = 0;
static void tables_init(void) {
  if (tables_ready) return;
  for (int Q = 19; Q <= 27; Q += 8)
    for (int i = 0; i < Q; ++i) {
      stencil_c(Q, i, TC[Q][i]);
      TW[Q][i] = stencil_w(Q, i);
      TOPP[Q][i] = stencil_opp(Q, i);
    }
  tables_ready = 1;
}

void orc_stencil(int Q, int* c, double* w, int* opp) {
  for (int i = 0; i < Q; ++i) {
    stencil_c(Q, i, c + 3 * i);
    w[i] = stencil_w(Q, i);
    opp[i] = stencil_opp(Q, i);
  }
}

/* ---------------------------------------------------------------------- Eq.(3) equilibrium --
 * f_i^eq(u, rho) = w_i rho [1 + c_i.u / c_s^2 + (c_i.u)^2 / (2 c_s^4) - u^2 / (2 c_s^2)],
 * c_s^2 = 1/3.  The printed "+ u^2/(2c_s^2)" is garbled: only "-" gives
 * sum_i f_i^eq = rho (reading A1; pinned by P2). */
static const double CS2 = 1.0 / 3.0;

void orc_equilibrium(int Q, double rho, const double u[3], double* feq) {
  double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int i = 0; i < Q; ++i) {
    int c[3];
    stencil_c(Q, i, c);
    double cu = c[0] * u[0] + c[1] * u[1] + c[2] * u[2];
    feq[i] = stencil_w(Q, i) * rho *
             (1.0 + (cu / CS2 + (cu * cu) / (2.0 * CS2 * CS2) - uu / (2.0 * CS2)));
  }
}

/* ------------------------------------------------------------------ Eq.(5) / Eq.(6): B(eps) --
 * mode 0: B = eps.  mode 1: B = eps(tau-1/2) / ((1-eps) + (tau-1/2))
 * (PAPER.md:159-161), evaluated in fp64 in exactly this operation order (reading A14). */
double orc_weight_fraction(double eps, double tau, int mode) {
  if (mode == 0) return eps;
  return eps * (tau - 0.5) / ((1.0 - eps) + (tau - 0.5));
}

/* ------------------------------------------------------ one-cell collision, Eq.(2),(4),(7)-(9) --
 * Computes f*_i = f_i + (1 - B) Omega^F_i + B Omega^S_i (Eq.(4)) for one cell, and
 * m = B sum_i Omega^S_i c_i (the summand of Eq.(10)).  g is the test-only Guo body force (A-P12):
 * u = (j + g/2)/rho and Omega^F gains (1 - 1/(2 tau)) w_i [(c_i - u)/c_s^2 + (c_i.u) c_i/c_s^4].g.
 * Returns 0, or 1 if rho <= 0 or a value is non-finite (error rule of S:66/S:93). */
/* Fluid operator kind: 0 = SRT, Eq.(2); 2 = cumulant (D3Q27, see below); 1 = TRT (two relaxation
 * times, listed by the paper
 * among lbmpy's operators; standard definition: with f^+-_i = (f_i +- f_ibar)/2,
 * Omega_i = -(1/tau)(f^+_i - f^eq+_i) - (1/tau_-)(f^-_i - f^eq-_i), tau_- = 1/2 + magic/(tau - 1/2);
 * the Guo source splits the same way with (1 - 1/(2 tau)) and (1 - 1/(2 tau_-))). */
static int collide_cell_impl(int Q, const double* f, double tau, int sc, double B,
                             const double us[3], const double g[3], int coll, double magic,
                             double* fstar, double m[3]);

int orc_collide_cell(int Q, const double* f, double tau, int sc, double B, const double us[3],
                     const double g[3], double* fstar, double m[3]) {
  return collide_cell_impl(Q, f, tau, sc, B, us, g, 0, 0.0, fstar, m);
}

int orc_collide_cell_trt(int Q, const double* f, double tau, double magic, int sc, double B,
                         const double us[3], const double g[3], double* fstar, double m[3]) {
  return collide_cell_impl(Q, f, tau, sc, B, us, g, 1, magic, fstar, m);
}

int orc_collide_cell_cum(int Q, const double* f, double tau, int sc, double B, const double us[3],
                         const double g[3], double* fstar, double m[3]) {
  return collide_cell_impl(Q, f, tau, sc, B, us, g, 2, 0.0, fstar, m);
}

static int collide_cell_impl(int Q, const double* f, double tau, int sc, double B,
                             const double us[3], const double g[3], int coll, double magic,
                             double* fstar, double m[3]) {
  tables_init();
  double rho = 0.0, j[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < Q; ++i) {
    int c[3];
    stencil_c(Q, i, c);
    rho += f[i];
    j[0] += f[i] * c[0];
    j[1] += f[i] * c[1];
    j[2] += f[i] * c[2];
  }
  m[0] = m[1] = m[2] = 0.0;
  if (!(rho > 0.0) || !isfinite(rho)) {
    for (int i = 0; i < Q; ++i) fstar[i] = f[i];
    return 1;
  }
  double u[3];
  for (int a = 0; a < 3; ++a) u[a] = (j[a] + 0.5 * g[a]) / rho; /* A4/A5: local pre-collision u */
  double feq[27], fs[27], omF[27], omS[27];
  orc_equilibrium(Q, rho, u, feq);
  double src[27];  /* raw Guo source w_i [(c_i - u)/c_s^2 + (c_i.u) c_i / c_s^4] . g */
  for (int i = 0; i < Q; ++i) {
    int c[3];
    stencil_c(Q, i, c);
    double cu = c[0] * u[0] + c[1] * u[1] + c[2] * u[2];
    double s = 0.0;
    for (int a = 0; a < 3; ++a) s += ((c[a] - u[a]) / CS2 + cu * c[a] / (CS2 * CS2)) * g[a];
    src[i] = stencil_w(Q, i) * s;
  }
  const int forced = (g[0] != 0.0 || g[1] != 0.0 || g[2] != 0.0);
  if (coll == 2) {
    /* Cumulant collision (the operator of the paper's performance runs),
     * D3Q27 (reading A29), or D3Q19 — the paper's performance stencil, PAPER.md:494 — on the 19
     * moments it carries (reading A32), with every relaxation rate of order >= 3 equal to 1 (those cumulants are set to their
     * equilibrium 0), the bulk rate 1 and the shear rate 1/tau.  Plain form: second central
     * moments by brute force; normalised cumulants C = kappa/rho relaxed; post-collision central
     * moments of a distribution whose cumulants of order >= 3 vanish (Wick products of the C's);
     * populations recovered by solving the 27x27 central-moment system. */
    double k2[3][3] = {{0}};
    for (int i = 0; i < Q; ++i) {
      int c[3];
      stencil_c(Q, i, c);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) k2[a][b] += f[i] * (c[a] - u[a]) * (c[b] - u[b]);
    }
    double C[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) C[a][b] = k2[a][b] / rho;
    const double w1 = 1.0 / tau, wb = 1.0;
    double Cs = C[0][0] + C[1][1] + C[2][2];
    double D1 = C[0][0] - C[1][1], D2 = C[0][0] - C[2][2];
    Cs = Cs + wb * (1.0 - Cs); /* trace equilibrium 3 c_s^2 = 1 */
    D1 = (1.0 - w1) * D1;
    D2 = (1.0 - w1) * D2;
    double Cxy = (1.0 - w1) * C[0][1], Cxz = (1.0 - w1) * C[0][2], Cyz = (1.0 - w1) * C[1][2];
    double Cxx = (Cs + D1 + D2) / 3.0, Cyy = (Cs - 2.0 * D1 + D2) / 3.0,
           Czz = (Cs + D1 - 2.0 * D2) / 3.0;
    /* post-collision central moments kstar[a][b][c] (orders a, b, c in x, y, z) */
    double ks[3][3][3];
    memset(ks, 0, sizeof(ks));
    ks[0][0][0] = rho;
    ks[2][0][0] = rho * Cxx;
    ks[0][2][0] = rho * Cyy;
    ks[0][0][2] = rho * Czz;
    ks[1][1][0] = rho * Cxy;
    ks[1][0][1] = rho * Cxz;
    ks[0][1][1] = rho * Cyz;
    ks[2][2][0] = rho * (Cxx * Cyy + 2.0 * Cxy * Cxy);
    ks[2][0][2] = rho * (Cxx * Czz + 2.0 * Cxz * Cxz);
    ks[0][2][2] = rho * (Cyy * Czz + 2.0 * Cyz * Cyz);
    ks[2][1][1] = rho * (Cxx * Cyz + 2.0 * Cxy * Cxz);
    ks[1][2][1] = rho * (Cyy * Cxz + 2.0 * Cxy * Cyz);
    ks[1][1][2] = rho * (Czz * Cxy + 2.0 * Cxz * Cyz);
    ks[2][2][2] = rho * (Cxx * Cyy * Czz + 2.0 * (Cxx * Cyz * Cyz + Cyy * Cxz * Cxz +
                                                  Czz * Cxy * Cxy) + 8.0 * Cxy * Cxz * Cyz);
    /* forcing (reading A31): about u = (j + g/2)/rho the first-order central moments are -g/2
     * before the collision and +g/2 after it (sign flip), so the post-collision momentum is
     * j + g; zero without a force */
    ks[1][0][0] = 0.5 * g[0];
    ks[0][1][0] = 0.5 * g[1];
    ks[0][0][1] = 0.5 * g[2];
    /* solve sum_i (c_ix - ux)^a (c_iy - uy)^b (c_iz - uz)^c fc_i = ks[a][b][c] over the
     * moments the velocity set carries: D3Q27 all 27 orders a, b, c <= 2; D3Q19 (reading A32)
     * the 19 with at least one zero order (it has no (+-1,+-1,+-1) velocities, so xyz, x^2yz,
     * ... are not independent moments of it) */
    double M[27][28];
    int nr = 0;
    for (int r = 0; r < 27; ++r) {
      int a = r % 3, b = (r / 3) % 3, cc = r / 9;
      if (Q == 19 && a > 0 && b > 0 && cc > 0) continue;
      for (int i = 0; i < Q; ++i) {
        int c[3];
        stencil_c(Q, i, c);
        M[nr][i] = pow(c[0] - u[0], a) * pow(c[1] - u[1], b) * pow(c[2] - u[2], cc);
      }
      M[nr][Q] = ks[a][b][cc];
      ++nr;
    }
    for (int col = 0; col < Q; ++col) { /* Gaussian elimination, partial pivoting */
      int piv = col;
      for (int r = col + 1; r < Q; ++r)
        if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
      if (piv != col)
        for (int k = 0; k <= Q; ++k) {
          double t = M[col][k];
          M[col][k] = M[piv][k];
          M[piv][k] = t;
        }
      for (int r = 0; r < Q; ++r) {
        if (r == col) continue;
        double fac = M[r][col] / M[col][col];
        for (int k = col; k <= Q; ++k) M[r][k] -= fac * M[col][k];
      }
    }
    for (int i = 0; i < Q; ++i) omF[i] = M[i][Q] / M[i][i] - f[i];
  } else if (coll == 0) {
    /* Eq.(2): Omega^F_i = -(1/tau)(f_i - f_i^eq) */
    for (int i = 0; i < Q; ++i) {
      omF[i] = -(f[i] - feq[i]) / tau;
      if (forced) omF[i] += (1.0 - 1.0 / (2.0 * tau)) * src[i];
    }
  } else {
    /* TRT on the symmetric / antisymmetric parts of each (i, ibar) pair */
    const double taum = 0.5 + magic / (tau - 0.5);
    for (int i = 0; i < Q; ++i) {
      int ib = TOPP[Q][i];
      double fp = 0.5 * (f[i] + f[ib]), fm = 0.5 * (f[i] - f[ib]);
      double ep = 0.5 * (feq[i] + feq[ib]), em = 0.5 * (feq[i] - feq[ib]);
      omF[i] = -(fp - ep) / tau - (fm - em) / taum;
      if (forced) {
        double sp = 0.5 * (src[i] + src[ib]), sm = 0.5 * (src[i] - src[ib]);
        omF[i] += (1.0 - 1.0 / (2.0 * tau)) * sp + (1.0 - 1.0 / (2.0 * taum)) * sm;
      }
    }
  }
  if (B > 0.0) {
    orc_equilibrium(Q, rho, us, fs); /* f^eq(rho, u_s), rho = local rho (A3) */
    for (int i = 0; i < Q; ++i) {
      int ib = TOPP[Q][i];
      if (sc == 1) /* Eq.(7) SC1 */
        omS[i] = (f[ib] - feq[ib]) - (f[i] - fs[i]);
      else if (sc == 2) /* Eq.(8) SC2, literal printed form with the missing ")" closed (A2) */
        omS[i] = (fs[i] - f[i]) + (1.0 - 1.0 / tau) * (f[i] - fs[i]);
      else /* Eq.(9) SC3 */
        omS[i] = (f[ib] - fs[ib]) - (f[i] - fs[i]);
    }
    double sum[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < Q; ++i) {
      int c[3];
      stencil_c(Q, i, c);
      fstar[i] = f[i] + (1.0 - B) * omF[i] + B * omS[i];
      sum[0] += omS[i] * c[0];
      sum[1] += omS[i] * c[1];
      sum[2] += omS[i] * c[2];
    }
    m[0] = B * sum[0];
    m[1] = B * sum[1];
    m[2] = B * sum[2];
  } else {
    for (int i = 0; i < Q; ++i) fstar[i] = f[i] + omF[i]; /* Eq.(1) with Eq.(2) */
  }
  for (int i = 0; i < Q; ++i)
    if (!isfinite(fstar[i])) return 1;
  return 0;
}

/* --------------------------------------------------------------------------- pose (A13) -----
 * Closed-form prescribed motion (one-way coupling): t_n = t_0 + n v, wrapped
 * into [0, L) on periodic axes; Q_n = Rot(w/|w|, n|w|) Q_0 by Rodrigues' formula, host libm. */
void orc_pose_advance(const double Q0[9], const double t0[3], const double v[3],
                      const double w[3], int64_t n, const double L[3], const int periodic[3],
                      double Qn[9], double tn[3]) {
  for (int a = 0; a < 3; ++a) {
    double t = t0[a] + (double)n * v[a];
    if (periodic[a]) t = t - L[a] * floor(t / L[a]);
    tn[a] = t;
  }
  double wn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  if (wn > 0.0) {
    double k[3] = {w[0] / wn, w[1] / wn, w[2] / wn};
    double th = (double)n * wn, s = sin(th), c = cos(th);
    double K[9] = {0, -k[2], k[1], k[2], 0, -k[0], -k[1], k[0], 0};
    double K2[9];
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int l = 0; l < 3; ++l) acc += K[3 * r + l] * K[3 * l + cc];
        K2[3 * r + cc] = acc;
      }
    for (int e = 0; e < 9; ++e) R[e] += s * K[e] + (1.0 - c) * K2[e];
  }
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) {
      double acc = 0.0;
      for (int l = 0; l < 3; ++l) acc += R[3 * r + l] * Q0[3 * l + cc];
      Qn[3 * r + cc] = acc;
    }
}

/* ------------------------------------------------------------ voxelizer (A15) --
 * Geometry field G of a closed mesh, spacing h = 2^-s in the body frame,
 * extent = mesh bbox padded by 2 LBM cells with an integer origin o_G (A17).  G[g] = 1 iff the
 * sub-cell centre o_G + (g + 1/2) h is inside the mesh by ray parity along +x, decided exactly:
 * vertices are snapped to the fixed-point grid 2^-(s+12) relative to o_G (sub-cell centres are
 * then integers g*4096 + 2048), the (y,z) containment uses 2D edge functions with a top-left
 * tie rule on the counter-clockwise-oriented projection, and a crossing counts iff it lies
 * strictly at x > x_0 (sign of an exact int128 expression).  Degenerate projections count 0.
 * Plain form: for every row (gy,gz), every triangle is tested; for each containing triangle the
 * crossing is compared exactly with every sample of the row. */
typedef __int128 i128;

static int edge_inside(int64_t ay, int64_t az, int64_t by, int64_t bz, int64_t py, int64_t pz) {
  /* E > 0 : P strictly left of a->b (inside for a CCW triangle).  Tie (E == 0): inside iff the
   * edge is a "top" edge (horizontal, pointing to -y) or a "left" edge (pointing to -z). */
  i128 e = (i128)(by - ay) * (i128)(pz - az) - (i128)(bz - az) * (i128)(py - ay);
  if (e > 0) return 1;
  if (e < 0) return 0;
  int64_t dy = by - ay, dz = bz - az;
  if (dz == 0 && dy < 0) return 1; /* top edge */
  if (dz < 0) return 1;            /* left edge */
  return 0;
}

int64_t orc_geometry_extent(const double* verts, int64_t nv, int s, double origin[3],
                            int64_t dims[3]) {
  for (int a = 0; a < 3; ++a) {
    double lo = verts[a], hi = verts[a];
    for (int64_t k = 1; k < nv; ++k) {
      double x = verts[3 * k + a];
      if (x < lo) lo = x;
      if (x > hi) hi = x;
    }
    origin[a] = floor(lo) - 2.0;
    dims[a] = ((int64_t)(ceil(hi) + 2.0 - origin[a])) << s;
  }
  return dims[0] * dims[1] * dims[2];
}

/* bits: [dims2][dims1][dims0] bytes (0/1), sized by orc_geometry_extent. */
void orc_voxelize(const double* verts, int64_t nv, const int32_t* tris, int64_t nt, int s,
                  uint8_t* bits) {
  double origin[3];
  int64_t dims[3];
  orc_geometry_extent(verts, nv, s, origin, dims);
  int64_t* V = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)nv);
  double scale = ldexp(1.0, s + 12);
  for (int64_t k = 0; k < nv; ++k)
    for (int a = 0; a < 3; ++a) V[3 * k + a] = llround((verts[3 * k + a] - origin[a]) * scale);
  int64_t NX = dims[0];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t row = 0; row < dims[1] * dims[2]; ++row) {
    int64_t gy = row % dims[1], gz = row / dims[1];
    int64_t Y0 = gy * 4096 + 2048, Z0 = gz * 4096 + 2048;
    uint8_t* cnt = (uint8_t*)calloc((size_t)NX, 1);
    for (int64_t t = 0; t < nt; ++t) {
      const int64_t* A = V + 3 * (int64_t)tris[3 * t + 0];
      const int64_t* Bv = V + 3 * (int64_t)tris[3 * t + 1];
      const int64_t* Cv = V + 3 * (int64_t)tris[3 * t + 2];
      /* projected signed area (2x) in the (y,z) plane */
      i128 area = (i128)(Bv[1] - A[1]) * (i128)(Cv[2] - A[2]) -
                  (i128)(Bv[2] - A[2]) * (i128)(Cv[1] - A[1]);
      if (area == 0) continue;
      const int64_t *P0 = A, *P1 = Bv, *P2 = Cv;
      if (area < 0) { /* orient counter-clockwise */
        P1 = Cv;
        P2 = Bv;
      }
      if (!edge_inside(P0[1], P0[2], P1[1], P1[2], Y0, Z0)) continue;
      if (!edge_inside(P1[1], P1[2], P2[1], P2[2], Y0, Z0)) continue;
      if (!edge_inside(P2[1], P2[2], P0[1], P0[2], Y0, Z0)) continue;
      /* plane normal n = (B-A) x (C-A) (original orientation; only the sign test below uses it) */
      i128 e1[3] = {Bv[0] - A[0], Bv[1] - A[1], Bv[2] - A[2]};
      i128 e2[3] = {Cv[0] - A[0], Cv[1] - A[1], Cv[2] - A[2]};
      i128 n0 = e1[1] * e2[2] - e1[2] * e2[1];
      i128 n1 = e1[2] * e2[0] - e1[0] * e2[2];
      i128 n2 = e1[0] * e2[1] - e1[1] * e2[0];
      /* crossing x* satisfies n.(X - A) = 0; x* - X0 = D / n0 with D = n.(A - P) */
      for (int64_t gx = 0; gx < NX; ++gx) {
        int64_t X0 = gx * 4096 + 2048;
        i128 D = n0 * (i128)(A[0] - X0) + n1 * (i128)(A[1] - Y0) + n2 * (i128)(A[2] - Z0);
        int right = (n0 > 0) ? (D > 0) : (D < 0);
        if (right) cnt[gx] ^= 1;
      }
    }
    uint8_t* dst = bits + row * NX;
    for (int64_t gx = 0; gx < NX; ++gx) dst[gx] = cnt[gx];
    free(cnt);
  }
  free(V);
}

/* ---------------------------------------------------------------------------- simulation ---- */
typedef struct {
  int present, kind, s; /* kind 0 sphere, 1 mesh */
  double radius, rbound;
  double Q[9], t[3], v[3], w[3];
  int dynamic;          /* two-way coupled: orc_integrate advances Q, t, v, w */
  int mapping;          /* meshes: 0 = R1 every sub-sample, 1 = R2 centre only (A12) */
  double mass, I[9], fext[3], text[3];
  double Ma, Ia[9];     /* virtual mass / inertia (A28), 0 = plain semi-implicit Euler */
  double dv[3], dw[3];  /* last velocity increments, world frame */
  double gorigin[3];
  int64_t gdims[3];
  uint8_t* gbits;
} orc_body;

typedef struct {
  int nx, ny, nz, Q;
  double tau;
  int bc[3]; /* 0 periodic, 1 wall, 2 (x only, nx >= 2) velocity inflow at x = 0 / pressure
                outflow at x = nx - 1 (reading A30) */
  double u_in[3], rho_out; /* A30 inflow velocity and outflow density */
  int sc, bmode;
  double g[3];
  double *f, *fnew;
  double* B;
  double* us;
  uint8_t* id;
  int32_t* cnt;
  orc_body bodies[ORC_MAXB + 1];
  double SF[ORC_MAXB + 1][3], ST[ORC_MAXB + 1][3], AF[ORC_MAXB + 1][3], AT[ORC_MAXB + 1][3];
  int64_t step;
  int64_t err_cell; /* -1 none */
  int map_all_cells; /* 1: evaluate every cell for every body (no bbox restriction) */
  int coll;          /* 0 SRT, 1 TRT */
  double magic;      /* TRT magic parameter */
} orc_sim;

static int64_t cidx(const orc_sim* S, int x, int y, int z) {
  return ((int64_t)z * S->ny + y) * S->nx + x;
}

orc_sim* orc_create(int nx, int ny, int nz, int Q, double tau, const int bc[3], int sc,
                    int bmode) {
  tables_init();
  orc_sim* S = (orc_sim*)calloc(1, sizeof(orc_sim));
  S->nx = nx;
  S->ny = ny;
  S->nz = nz;
  S->Q = Q;
  S->tau = tau;
  for (int a = 0; a < 3; ++a) S->bc[a] = bc[a];
  S->sc = sc;
  S->bmode = bmode;
  int64_t N = (int64_t)nx * ny * nz;
  S->f = (double*)calloc((size_t)(Q * N), sizeof(double));
  S->fnew = (double*)calloc((size_t)(Q * N), sizeof(double));
  S->B = (double*)calloc((size_t)N, sizeof(double));
  S->us = (double*)calloc((size_t)(3 * N), sizeof(double));
  S->id = (uint8_t*)calloc((size_t)N, 1);
  S->cnt = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  S->err_cell = -1;
  S->rho_out = 1.0;
  return S;
}

/* Reading A30 (P:584, P:593 name "boundary handling for inflow and outflow" without defining
 * it): velocity inflow and pressure outflow on the x faces. */
void orc_set_open_boundary(orc_sim* S, const double u_in[3], double rho_out) {
  for (int a = 0; a < 3; ++a) S->u_in[a] = u_in[a];
  S->rho_out = rho_out;
}

void orc_destroy(orc_sim* S) {
  if (!S) return;
  for (int b = 0; b <= ORC_MAXB; ++b) free(S->bodies[b].gbits);
  free(S->f);
  free(S->fnew);
  free(S->B);
  free(S->us);
  free(S->id);
  free(S->cnt);
  free(S);
}

void orc_set_force(orc_sim* S, const double g[3]) {
  for (int a = 0; a < 3; ++a) S->g[a] = g[a];
}
void orc_set_map_all_cells(orc_sim* S, int on) { S->map_all_cells = on; }
void orc_set_collision(orc_sim* S, int coll, double magic) {
  S->coll = coll;
  S->magic = magic;
}

void orc_init_equilibrium(orc_sim* S, const double* rho, const double* u) {
  int64_t N = (int64_t)S->nx * S->ny * S->nz;
  for (int64_t x = 0; x < N; ++x) {
    double r = rho ? rho[x] : 1.0;
    double uu[3] = {u ? u[x] : 0.0, u ? u[N + x] : 0.0, u ? u[2 * N + x] : 0.0};
    double feq[27];
    orc_equilibrium(S->Q, r, uu, feq);
    for (int i = 0; i < S->Q; ++i) S->f[(int64_t)i * N + x] = feq[i];
  }
  S->step = 0;
}

void orc_set_pdfs(orc_sim* S, const double* f) {
  memcpy(S->f, f, sizeof(double) * (size_t)S->Q * S->nx * S->ny * S->nz);
}
void orc_get_pdfs(const orc_sim* S, double* f) {
  memcpy(f, S->f, sizeof(double) * (size_t)S->Q * S->nx * S->ny * S->nz);
}

/* rho and u = j / rho of the Eq.(4) state */
void orc_get_velocity(const orc_sim* S, double* rho, double* u) {
  int64_t N = (int64_t)S->nx * S->ny * S->nz;
  for (int64_t x = 0; x < N; ++x) {
    double r = 0, j[3] = {0, 0, 0};
    for (int i = 0; i < S->Q; ++i) {
      int c[3];
      stencil_c(S->Q, i, c);
      double fi = S->f[(int64_t)i * N + x];
      r += fi;
      j[0] += fi * c[0];
      j[1] += fi * c[1];
      j[2] += fi * c[2];
    }
    if (rho) rho[x] = r;
    if (u)
      for (int a = 0; a < 3; ++a) u[(int64_t)a * N + x] = j[a] / r;
  }
}

/* Body setup.  Sphere: radius r, bounding radius r.  Mesh: voxelised once here,
 * bounding radius = max |vertex| (body frame). */
int orc_set_sphere(orc_sim* S, int id, double r, int s) {
  if (id < 1 || id > ORC_MAXB) return -1;
  orc_body* b = &S->bodies[id];
  free(b->gbits);
  memset(b, 0, sizeof(*b));
  b->present = 1;
  b->kind = 0;
  b->s = s;
  b->radius = r;
  b->rbound = r;
  b->Q[0] = b->Q[4] = b->Q[8] = 1.0;
  return 0;
}

int orc_set_mesh(orc_sim* S, int id, const double* verts, int64_t nv, const int32_t* tris,
                 int64_t nt, int s) {
  if (id < 1 || id > ORC_MAXB) return -1;
  orc_body* b = &S->bodies[id];
  free(b->gbits);
  memset(b, 0, sizeof(*b));
  b->present = 1;
  b->kind = 1;
  b->s = s;
  int64_t n = orc_geometry_extent(verts, nv, s, b->gorigin, b->gdims);
  b->gbits = (uint8_t*)calloc((size_t)n, 1);
  orc_voxelize(verts, nv, tris, nt, s, b->gbits);
  double rb = 0.0;
  for (int64_t k = 0; k < nv; ++k) {
    double x = verts[3 * k], y = verts[3 * k + 1], z = verts[3 * k + 2];
    double r = sqrt(x * x + y * y + z * z);
    if (r > rb) rb = r;
  }
  b->rbound = rb;
  b->Q[0] = b->Q[4] = b->Q[8] = 1.0;
  return 0;
}

void orc_remove_body(orc_sim* S, int id) {
  if (id < 1 || id > ORC_MAXB) return;
  free(S->bodies[id].gbits);
  memset(&S->bodies[id], 0, sizeof(orc_body));
}

int orc_get_geometry(const orc_sim* S, int id, double origin[3], int64_t dims[3],
                     uint8_t* bits) {
  const orc_body* b = &S->bodies[id];
  if (!b->present || b->kind != 1) return -1;
  for (int a = 0; a < 3; ++a) {
    origin[a] = b->gorigin[a];
    dims[a] = b->gdims[a];
  }
  if (bits) memcpy(bits, b->gbits, (size_t)(b->gdims[0] * b->gdims[1] * b->gdims[2]));
  return 0;
}

void orc_set_pose(orc_sim* S, int id, const double Q[9], const double t[3], const double v[3],
                  const double w[3]) {
  orc_body* b = &S->bodies[id];
  memcpy(b->Q, Q, sizeof(b->Q));
  memcpy(b->t, t, sizeof(b->t));
  memcpy(b->v, v, sizeof(b->v));
  memcpy(b->w, w, sizeof(b->w));
  if (b->dynamic)  /* a new initial state of a dynamic body: no previous increments */
    for (int a = 0; a < 3; ++a) b->dv[a] = b->dw[a] = 0.0;
}

/* Minimum image on a periodic axis of length L (A7). */
static double mi(double d, double L, int periodic) {
  if (!periodic) return d;
  if (d >= 0.5 * L)
    d -= L;
  else if (d < -0.5 * L)
    d += L;
  return d;
}

/* Inside test of one sub-sample for body b, at world point p (reading R1, A12): the sample is
 * mapped into the body frame, q = Q^T mi(p - t), with the fma order of A14. */
static int sample_inside(const orc_sim* S, const orc_body* b, const double p[3]) {
  double L[3] = {S->nx, S->ny, S->nz};
  double d[3];
  for (int a = 0; a < 3; ++a) d[a] = mi(p[a] - b->t[a], L[a], S->bc[a] == 0);
  double q[3];
  for (int a = 0; a < 3; ++a)
    q[a] = fma(b->Q[6 + a], d[2], fma(b->Q[3 + a], d[1], b->Q[0 + a] * d[0]));
  if (b->kind == 0) return fma(q[2], q[2], fma(q[1], q[1], q[0] * q[0])) <= b->radius * b->radius;
  double hs = ldexp(1.0, b->s);
  int64_t g[3];
  for (int a = 0; a < 3; ++a) {
    double x = floor((q[a] - b->gorigin[a]) * hs);
    if (!(x >= 0.0) || x >= (double)b->gdims[a]) return 0; /* outside the field: outside (A17) */
    g[a] = (int64_t)x;
  }
  return b->gbits[(g[2] * b->gdims[1] + g[1]) * b->gdims[0] + g[0]];
}

/* Reading R2 of the mapping (A12; the paper's literal wording: "multiplying the
 * cell center in LBM space with a rotation matrix"): only the cell centre p_c is mapped into the
 * body frame, q_c = Q^T mi(p_c - t) (A14 order), and the count is the number of set geometry cells
 * g with g_a in [g0_a, g0_a + 2^s), g0_a = floor((q_c,a - o_a) 2^s - 2^(s-1) + 1/2): the block of
 * 2^s x 2^s x 2^s geometry cells "corresponding" to the cell.  Cells beyond the
 * field count 0. */
static int r2_count(const orc_sim* S, const orc_body* b, int x, int y, int z) {
  double L[3] = {S->nx, S->ny, S->nz};
  double pc[3] = {x + 0.5, y + 0.5, z + 0.5}, d[3], q[3];
  for (int a = 0; a < 3; ++a) d[a] = mi(pc[a] - b->t[a], L[a], S->bc[a] == 0);
  for (int a = 0; a < 3; ++a)
    q[a] = fma(b->Q[6 + a], d[2], fma(b->Q[3 + a], d[1], b->Q[0 + a] * d[0]));
  int n = 1 << b->s;
  double hs = ldexp(1.0, b->s), half = ldexp(1.0, b->s - 1);
  int64_t g0[3];
  for (int a = 0; a < 3; ++a) g0[a] = (int64_t)floor((q[a] - b->gorigin[a]) * hs - half + 0.5);
  int cnt = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int64_t g[3] = {g0[0] + i, g0[1] + j, g0[2] + k};
        int in = 1;
        for (int a = 0; a < 3; ++a)
          if (g[a] < 0 || g[a] >= b->gdims[a]) in = 0;
        if (in) cnt += b->gbits[(g[2] * b->gdims[1] + g[1]) * b->gdims[0] + g[0]];
      }
  return cnt;
}

void orc_set_mapping(orc_sim* S, int id, int mode) { S->bodies[id].mapping = mode; }

/* Fraction mapping: for each cell, eps_b = (#inside sub-samples)/2^(3s) over
 * the 2^(3s) sub-cell centres (A16); the body with the largest eps wins, ties to the lower id
 * (A18); B by Eq.(5)/(6); u_s = v + w x mi(x_c - t) (rigid motion). */
void orc_map(orc_sim* S) {
  double L[3] = {S->nx, S->ny, S->nz};
#pragma omp parallel for schedule(static)
  for (int z = 0; z < S->nz; ++z)
    for (int y = 0; y < S->ny; ++y)
      for (int x = 0; x < S->nx; ++x) {
        int64_t c = cidx(S, x, y, z);
        int best = 0, bestcnt = 0;
        double xc[3] = {x + 0.5, y + 0.5, z + 0.5};
        for (int id = 1; id <= ORC_MAXB; ++id) {
          const orc_body* b = &S->bodies[id];
          if (!b->present) continue;
          if (!S->map_all_cells) { /* conservative bbox: |mi(x_c - t)|_a <= rbound + 1 per axis */
            int in = 1;
            for (int a = 0; a < 3; ++a)
              if (fabs(mi(xc[a] - b->t[a], L[a], S->bc[a] == 0)) > b->rbound + 1.0) in = 0;
            if (!in) continue;
          }
          int n = 1 << b->s, cnt = 0;
          double h = ldexp(1.0, -b->s);
          if (b->kind == 1 && b->mapping == 1) {
            cnt = r2_count(S, b, x, y, z);
          } else {
            for (int gz = 0; gz < n; ++gz)
              for (int gy = 0; gy < n; ++gy)
                for (int gx = 0; gx < n; ++gx) {
                  double p[3] = {x + (gx + 0.5) * h, y + (gy + 0.5) * h, z + (gz + 0.5) * h};
                  cnt += sample_inside(S, b, p);
                }
          }
          /* compare eps exactly: cnt / 8^s as a dyadic double */
          double e = ldexp((double)cnt, -3 * b->s);
          double eb = best ? ldexp((double)bestcnt, -3 * S->bodies[best].s) : 0.0;
          if (cnt > 0 && e > eb) {
            best = id;
            bestcnt = cnt;
          }
        }
        S->cnt[c] = bestcnt;
        S->id[c] = (uint8_t)best;
        int64_t N = (int64_t)S->nx * S->ny * S->nz;
        if (best) {
          const orc_body* b = &S->bodies[best];
          double e = ldexp((double)bestcnt, -3 * b->s);
          S->B[c] = orc_weight_fraction(e, S->tau, S->bmode);
          double r[3];
          for (int a = 0; a < 3; ++a) r[a] = mi(xc[a] - b->t[a], L[a], S->bc[a] == 0);
          S->us[c] = b->v[0] + (b->w[1] * r[2] - b->w[2] * r[1]);
          S->us[N + c] = b->v[1] + (b->w[2] * r[0] - b->w[0] * r[2]);
          S->us[2 * N + c] = b->v[2] + (b->w[0] * r[1] - b->w[1] * r[0]);
        } else {
          S->B[c] = 0.0;
          S->us[c] = S->us[N + c] = S->us[2 * N + c] = 0.0;
        }
      }
}

/* TEST-ONLY explicit fields (P4): B[N], us[3][N], id[N]. */
void orc_set_fields(orc_sim* S, const double* B, const double* us, const uint8_t* id) {
  int64_t N = (int64_t)S->nx * S->ny * S->nz;
  memcpy(S->B, B, sizeof(double) * (size_t)N);
  memcpy(S->us, us, sizeof(double) * 3 * (size_t)N);
  memcpy(S->id, id, (size_t)N);
  memset(S->cnt, 0, sizeof(int32_t) * (size_t)N);
}

void orc_get_fractions(const orc_sim* S, double* B, uint8_t* id, int32_t* cnt, double* us) {
  int64_t N = (int64_t)S->nx * S->ny * S->nz;
  if (B) memcpy(B, S->B, sizeof(double) * (size_t)N);
  if (id) memcpy(id, S->id, (size_t)N);
  if (cnt) memcpy(cnt, S->cnt, sizeof(int32_t) * (size_t)N);
  if (us) memcpy(us, S->us, sizeof(double) * 3 * (size_t)N);
}

/* One time step n -> n+1 (DESIGN.md §3 "oracle step"): collide every cell with the current B,
 * u_s, id fields (Eq.(4)), accumulate Eqs.(10)-(11), then push f*_i(x) to x + c_i (Eq.(1)); on a
 * wall axis a population leaving the domain returns as f_ibar(x) (half-way bounce-back, A23).
 * Returns 0, or 1 on an invalid state (first offending cell in cell order is recorded). */
int orc_step(orc_sim* S) {
  const int Q = S->Q, nx = S->nx, ny = S->ny, nz = S->nz;
  const int64_t N = (int64_t)nx * ny * nz;
  double L[3] = {nx, ny, nz};
  double(*pSF)[ORC_MAXB + 1][3] = calloc((size_t)nz, sizeof(*pSF));
  double(*pST)[ORC_MAXB + 1][3] = calloc((size_t)nz, sizeof(*pST));
  double(*pAF)[ORC_MAXB + 1][3] = calloc((size_t)nz, sizeof(*pAF));
  double(*pAT)[ORC_MAXB + 1][3] = calloc((size_t)nz, sizeof(*pAT));
  int64_t* perr = (int64_t*)malloc(sizeof(int64_t) * (size_t)nz);
#pragma omp parallel for schedule(static)
  for (int z = 0; z < nz; ++z) {
    perr[z] = -1;
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        int64_t c = cidx(S, x, y, z);
        double f[27], fs[27], m[3];
        for (int i = 0; i < Q; ++i) f[i] = S->f[(int64_t)i * N + c];
        double us[3] = {S->us[c], S->us[N + c], S->us[2 * N + c]};
        double B = S->B[c];
        int bad = collide_cell_impl(Q, f, S->tau, S->sc, B, us, S->g, S->coll, S->magic, fs, m);
        if (bad && perr[z] < 0) perr[z] = c;
        int id = S->id[c];
        if (B > 0.0) {
          double R[3] = {0, 0, 0};
          if (id > 0) R[0] = S->bodies[id].t[0], R[1] = S->bodies[id].t[1],
                      R[2] = S->bodies[id].t[2];
          double xc[3] = {x + 0.5, y + 0.5, z + 0.5}, r[3];
          for (int a = 0; a < 3; ++a) r[a] = mi(xc[a] - R[a], L[a], S->bc[a] == 0);
          double tq[3] = {r[1] * m[2] - r[2] * m[1], r[2] * m[0] - r[0] * m[2],
                          r[0] * m[1] - r[1] * m[0]};
          for (int a = 0; a < 3; ++a) {
            pSF[z][id][a] += m[a];
            pST[z][id][a] += tq[a];
            pAF[z][id][a] += fabs(m[a]);
            pAT[z][id][a] += fabs(tq[a]);
          }
        }
        /* stream (push) */
        for (int i = 0; i < Q; ++i) {
          int cc[3];
          stencil_c(Q, i, cc);
          int xn[3] = {x + cc[0], y + cc[1], z + cc[2]};
          int n3[3] = {nx, ny, nz};
          const int ib = TOPP[Q][i];
          if (S->bc[0] == 2 && (xn[0] < 0 || xn[0] >= nx)) {
            /* A30: the x faces take precedence over walls on the other axes (domain edges) */
            int cb[3];
            stencil_c(Q, ib, cb);
            const double wb = stencil_w(Q, ib);
            if (xn[0] < 0) {
              /* velocity inflow, moving-wall bounce-back with rho_w = 1:
               * f_ibar(x) = f*_i(x) + 2 w_ibar rho_w (c_ibar . u_in) / c_s^2 */
              double cu = cb[0] * S->u_in[0] + cb[1] * S->u_in[1] + cb[2] * S->u_in[2];
              S->fnew[(int64_t)ib * N + c] = fs[i] + 2.0 * wb * 1.0 * cu / CS2;
            } else {
              /* pressure outflow, anti-bounce-back: f_ibar(x) = -f*_i(x) + (equilibrium part,
               * added by the outflow pass after streaming, which needs the new state) */
              S->fnew[(int64_t)ib * N + c] = -fs[i];
            }
            continue;
          }
          int wall = 0;
          for (int a = 0; a < 3; ++a) {
            if (xn[a] < 0 || xn[a] >= n3[a]) {
              if (S->bc[a] == 1)
                wall = 1;
              else
                xn[a] = (xn[a] + n3[a]) % n3[a];
            }
          }
          if (wall)
            S->fnew[(int64_t)ib * N + c] = fs[i];
          else
            S->fnew[(int64_t)i * N + cidx(S, xn[0], xn[1], xn[2])] = fs[i];
        }
      }
  }
  if (S->bc[0] == 2) {
    /* A30 pressure outflow at x = nx-1, completed on the new state: the populations entering
     * from outside (c_x = -1) are unknown; the known ones give, with rho = rho_out (Zou & He),
     * u_x = (S_0 + 2 S_+) / rho_out - 1 (S_0: c_x = 0, S_+: c_x = +1), u_y = u_z = 0, and
     * f_q = -f*_qbar + 2 w_q rho_out [1 + (c_q.u)^2/(2c_s^4) - u^2/(2c_s^2)]. */
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y) {
        const int64_t c = cidx(S, nx - 1, y, z);
        double S0 = 0.0, Sp = 0.0;
        for (int i = 0; i < Q; ++i) {
          int cc[3];
          stencil_c(Q, i, cc);
          if (cc[0] == 0) S0 += S->fnew[(int64_t)i * N + c];
          if (cc[0] == 1) Sp += S->fnew[(int64_t)i * N + c];
        }
        const double u[3] = {(S0 + 2.0 * Sp) / S->rho_out - 1.0, 0.0, 0.0};
        const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
        for (int i = 0; i < Q; ++i) {
          int cc[3];
          stencil_c(Q, i, cc);
          if (cc[0] != -1) continue;
          const double cu = cc[0] * u[0] + cc[1] * u[1] + cc[2] * u[2];
          S->fnew[(int64_t)i * N + c] +=
              2.0 * stencil_w(Q, i) * S->rho_out *
              (1.0 + (cu * cu) / (2.0 * CS2 * CS2) - uu / (2.0 * CS2));
        }
      }
  }
  for (int id = 0; id <= ORC_MAXB; ++id)
    for (int a = 0; a < 3; ++a) S->SF[id][a] = S->ST[id][a] = S->AF[id][a] = S->AT[id][a] = 0.0;
  int err = 0;
  for (int z = 0; z < nz; ++z) {
    for (int id = 0; id <= ORC_MAXB; ++id)
      for (int a = 0; a < 3; ++a) {
        S->SF[id][a] += pSF[z][id][a];
        S->ST[id][a] += pST[z][id][a];
        S->AF[id][a] += pAF[z][id][a];
        S->AT[id][a] += pAT[z][id][a];
      }
    if (!err && perr[z] >= 0) {
      err = 1;
      S->err_cell = perr[z];
    }
  }
  free(pSF);
  free(pST);
  free(pAF);
  free(pAT);
  free(perr);
  double* t = S->f;
  S->f = S->fnew;
  S->fnew = t;
  S->step += 1;
  return err;
}

int64_t orc_error_cell(const orc_sim* S) { return S->err_cell; }

/* ---------------------------------------------------------------- two-way coupling -------
 * (NEXT row; the paper couples force and torque back to a settling sphere, PAPER.md:441-447,
 * without stating the integrator; DESIGN.md §12 fixes semi-implicit Euler.)  For every dynamic
 * body, with F, T the force and torque ON the body from the last orc_step:
 *   v <- v + (F + F_ext)/m;  t <- t + v (wrapped into [0, L) on periodic axes);
 *   I_w = Q I Q^T;  w <- w + I_w^{-1} (T + T_ext)  (adjugate / determinant);
 *   Q <- Rot(w/|w|, |w|) Q;  columns of Q re-orthonormalised (Gram-Schmidt). */
void orc_set_dynamics(orc_sim* S, int id, double mass, const double I[9], const double fext[3],
                      const double text[3], double Ma, const double Ia[9]) {
  orc_body* b = &S->bodies[id];
  if (!b->dynamic)
    for (int a = 0; a < 3; ++a) b->dv[a] = b->dw[a] = 0.0;
  b->dynamic = 1;
  b->mass = mass;
  memcpy(b->I, I, sizeof(b->I));
  memcpy(b->fext, fext, sizeof(b->fext));
  memcpy(b->text, text, sizeof(b->text));
  b->Ma = Ma;
  memcpy(b->Ia, Ia, sizeof(b->Ia));
}

void orc_integrate(orc_sim* S) {
  double L[3] = {S->nx, S->ny, S->nz};
  for (int id = 1; id <= ORC_MAXB; ++id) {
    orc_body* b = &S->bodies[id];
    if (!b->present || !b->dynamic) continue;
    double F[3], T[3];
    for (int a = 0; a < 3; ++a) {
      F[a] = -S->SF[id][a];
      T[a] = -S->ST[id][a];
    }
    /* virtual-mass form (A28): (m + M_a) dv_new = F + F_e + M_a dv_old; M_a = 0: plain Euler */
    for (int a = 0; a < 3; ++a) {
      b->dv[a] = (F[a] + b->fext[a] + b->Ma * b->dv[a]) / (b->mass + b->Ma);
      b->v[a] = b->v[a] + b->dv[a];
    }
    for (int a = 0; a < 3; ++a) {
      double x = b->t[a] + b->v[a];
      if (S->bc[a] == 0) x = x - L[a] * floor(x / L[a]);
      b->t[a] = x;
    }
    /* I_w = Q I Q^T, A_w = Q I_a Q^T (world frame) */
    double QI[9], Iw[9], QA[9], Aw[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0, acc2 = 0.0;
        for (int k = 0; k < 3; ++k) {
          acc += b->Q[3 * r + k] * b->I[3 * k + c];
          acc2 += b->Q[3 * r + k] * b->Ia[3 * k + c];
        }
        QI[3 * r + c] = acc;
        QA[3 * r + c] = acc2;
      }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0, acc2 = 0.0;
        for (int k = 0; k < 3; ++k) {
          acc += QI[3 * r + k] * b->Q[3 * c + k];
          acc2 += QA[3 * r + k] * b->Q[3 * c + k];
        }
        Iw[3 * r + c] = acc;
        Aw[3 * r + c] = acc2;
      }
    double Adw[3];
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += Aw[3 * r + k] * b->dw[k];
      Adw[r] = acc;
    }
    for (int k = 0; k < 9; ++k) Iw[k] = Iw[k] + Aw[k];
    /* inverse by the adjugate: inv = adj / det */
    double a = Iw[0], bb = Iw[1], c = Iw[2], d = Iw[3], e = Iw[4], f = Iw[5], g = Iw[6],
           h = Iw[7], i = Iw[8];
    double adj[9] = {e * i - f * h, c * h - bb * i, bb * f - c * e,
                     f * g - d * i, a * i - c * g, c * d - a * f,
                     d * h - e * g, bb * g - a * h, a * e - bb * d};
    double det = a * (e * i - f * h) - bb * (d * i - f * g) + c * (d * h - e * g);
    double tt[3] = {T[0] + b->text[0] + Adw[0], T[1] + b->text[1] + Adw[1],
                    T[2] + b->text[2] + Adw[2]};
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += adj[3 * r + k] * tt[k];
      b->dw[r] = acc / det;
    }
    for (int r = 0; r < 3; ++r) b->w[r] = b->w[r] + b->dw[r];
    double Qn[9], zero[3] = {0, 0, 0}, one[3] = {1, 1, 1}, tdummy[3];
    int noper[3] = {0, 0, 0};
    orc_pose_advance(b->Q, zero, zero, b->w, 1, one, noper, Qn, tdummy);
    double c0[3] = {Qn[0], Qn[3], Qn[6]}, c1[3] = {Qn[1], Qn[4], Qn[7]}, c2[3];
    double n0 = sqrt(c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2]);
    for (int k = 0; k < 3; ++k) c0[k] = c0[k] / n0;
    double d01 = c0[0] * c1[0] + c0[1] * c1[1] + c0[2] * c1[2];
    for (int k = 0; k < 3; ++k) c1[k] = c1[k] - d01 * c0[k];
    double n1 = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int k = 0; k < 3; ++k) c1[k] = c1[k] / n1;
    c2[0] = c0[1] * c1[2] - c0[2] * c1[1];
    c2[1] = c0[2] * c1[0] - c0[0] * c1[2];
    c2[2] = c0[0] * c1[1] - c0[1] * c1[0];
    for (int k = 0; k < 3; ++k) {
      b->Q[3 * k + 0] = c0[k];
      b->Q[3 * k + 1] = c1[k];
      b->Q[3 * k + 2] = c2[k];
    }
  }
}

void orc_get_body_state(const orc_sim* S, int id, double Q[9], double t[3], double v[3],
                        double w[3]) {
  const orc_body* b = &S->bodies[id];
  memcpy(Q, b->Q, sizeof(b->Q));
  memcpy(t, b->t, 3 * sizeof(double));
  memcpy(v, b->v, 3 * sizeof(double));
  memcpy(w, b->w, 3 * sizeof(double));
}

/* Force and torque ON body id (A6): F = -sum B sum_i Omega^S_i c_i (the printed Eq.(10) sum is
 * the momentum the fluid gains), T = -sum B (x_c - R) x sum_i Omega^S_i c_i (Eq.(11), A7). */
void orc_force_torque(const orc_sim* S, int id, double F[3], double T[3], double AF[3],
                      double AT[3]) {
  for (int a = 0; a < 3; ++a) {
    F[a] = -S->SF[id][a];
    T[a] = -S->ST[id][a];
    if (AF) AF[a] = S->AF[id][a];
    if (AT) AT[a] = S->AT[id][a];
  }
}
