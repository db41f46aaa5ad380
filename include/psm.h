/*
 * psm.h — C ABI of the B200-native Partially Saturated Cells (PSM) lattice Boltzmann hot path.
 *
 * Method: Suffa, Kemmler, Köstler, Rüde, "Large-Scale Simulations of Fully Resolved Complex
 * Moving Geometries with Partially Saturated Cells" (arXiv 2502.20049).  Citations below are
 * "PAPER.md:<line>" of the paper text plus the equation they fall in.  Equation numbers follow
 * the LaTeX environments (Eq.(1) at PAPER.md:127 ... Eq.(11) at PAPER.md:201).
 *
 * Conventions shared by every call:
 *   - Lattice units, dx = dt = 1, c_s^2 = 1/3.  Cell (i,j,k) covers [i,i+1)x[j,j+1)x[k,k+1); its
 *     centre is x_c = (i+1/2, j+1/2, k+1/2) in GLOBAL coordinates.
 *   - Host field arrays are the calling rank's LOCAL z-slab, layout [..][nz_local][ny][nx],
 *     x fastest; PDF arrays are [Q][nz_local][ny][nx] in the stencil order of DESIGN.md §2.1.
 *     With world == 1 the slab is the whole grid.
 *   - The "state" read and written through this ABI is always the Eq.(4) state: the
 *     PRE-collision populations f_i(x,t) of PAPER.md:144-147 (collide-then-push form), in fp64,
 *     whatever storage pattern (two-array pull or AA) and precision the context uses inside.
 *   - Every call returns psm_status; no C++ exception crosses this boundary.  On error the
 *     context is left unchanged unless stated; psm_last_error() gives a one-line reason.
 *   - Host pointers are borrowed for the duration of the call only (meshes and fields are
 *     copied).  All device work is enqueued on the context's CUDA stream; calls that return
 *     host data synchronise that stream.  A context must be used from one host thread.
 */
#ifndef PSM_H_
#define PSM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct psm_ctx psm_ctx; /* opaque, owned by the library */

typedef enum {
  PSM_OK = 0,
  PSM_E_ARG = -1,        /* invalid argument (tau <= 1/2, bad extents, bad body id, ...)     */
  PSM_E_OOM = -2,        /* device/host allocation failed or bound buffer too small         */
  PSM_E_MESH = -3,       /* triangle index out of range or mesh not watertight              */
  PSM_E_POSE = -4,       /* pose matrix not a proper rotation (|Q^T Q - I|_inf > 1e-9, det<=0)*/
  PSM_E_STATE = -5,      /* a cell reached rho <= 0 or a non-finite value                   */
  PSM_E_CUDA = -6,       /* CUDA runtime error                                              */
  PSM_E_NCCL = -7,       /* NCCL error                                                      */
  PSM_E_UNSUPPORTED = -8 /* valid request this build does not implement                     */
} psm_status;

typedef enum { PSM_D3Q19 = 19, PSM_D3Q27 = 27 } psm_stencil;
/* Solid collision operators, Eqs.(7)-(9). */
typedef enum { PSM_SC1 = 1, PSM_SC2 = 2, PSM_SC3 = 3 } psm_solid_op;
/* B(eps): Eq.(5) direct B = eps; Eq.(6) tau-weighted. */
typedef enum { PSM_B_DIRECT = 0, PSM_B_WEIGHTED = 1 } psm_bmode;
typedef enum { PSM_F64 = 0, PSM_F32 = 1 } psm_precision;
/* Streaming realisation: two-field pull or in-place AA pattern. */
typedef enum { PSM_TWO_ARRAY = 0, PSM_AA = 1 } psm_pattern;
/* Domain boundary per axis: periodic, half-way bounce-back resting wall, or (x axis
 * only, nx >= 3, PSM_TWO_ARRAY only) the open boundaries of the paper's application runs
 * ("boundary handling for inflow and outflow"; reading A30): velocity inflow
 * at x = 0, pressure outflow at x = nx - 1, values set by psm_set_open_boundary.  On domain edges
 * the x faces take precedence over walls. */
typedef enum { PSM_PERIODIC = 0, PSM_WALL = 1, PSM_INOUT = 2 } psm_bc;
typedef enum { PSM_SPHERE = 0, PSM_MESH = 1 } psm_shape_kind;
/* Fluid collision operator: SRT (Eq.(2)), TRT (two relaxation times, one of the
 * operators the paper lists; symmetric rate 1/tau, antisymmetric 1/tau_- with
 * tau_- = 1/2 + Lambda/(tau - 1/2)), or the cumulant operator of the paper's performance runs
 * (D3Q27, reading A29, or D3Q19 — the paper's performance stencil — on the 19
 * moments that stencil carries, reading A32; shear rate 1/tau, bulk and higher-order rates 1; a
 * body force flips the first-order central moments about the force-shifted velocity, A31). */
typedef enum { PSM_SRT = 0, PSM_TRT = 1, PSM_CUMULANT = 2 } psm_collision;

typedef struct {
  int64_t nx, ny, nz; /* GLOBAL extents in cells, each >= 1                                  */
  int32_t bc[3];      /* psm_bc per axis x, y, z                                             */
} psm_grid;

typedef struct {
  int32_t prec;          /* psm_precision of the stored PDFs and of the collision arithmetic */
  int32_t pattern;       /* psm_pattern                                                      */
  int32_t sc;            /* psm_solid_op                                                     */
  int32_t bmode;         /* psm_bmode                                                        */
  double body_force[3];  /* constant Guo body force on the fluid part, TEST-ONLY (default 0); */
                         /* only supported with PSM_TWO_ARRAY                               */
  int32_t rank, world;   /* z-slab decomposition: this rank of `world` (world >= 1)         */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId (fresh per context) shared by all ranks; NULL iff world==1 */
  void* cuda_stream;     /* cudaStream_t to enqueue on (e.g. torch's current stream); NULL = */
                         /* the legacy default stream                                       */
  int32_t collision;     /* psm_collision: fluid operator Omega^F                            */
  double trt_magic;      /* TRT magic parameter Lambda = (tau - 1/2)(tau_- - 1/2) (> 0);     */
                         /* 3/16 puts half-way bounce-back walls exactly mid-link            */
} psm_options;

/* Create a context.  Host-only: validates and plans the layout; no device memory yet.  With
 * world > 1 the NCCL communicator is created at the first device call (bind/alloc), which is
 * collective: every rank must reach it.  Rank r owns global z in [r*nz/world, (r+1)*nz/world).
 * Errors: PSM_E_ARG if tau <= 1/2 or non-finite (Eq.(2): tau is the relaxation time and the
 * viscosity (tau-1/2)/3 must be positive), any extent < 1, nz < world, or an unknown enum;
 * PSM_E_UNSUPPORTED for body_force with PSM_AA, or world > 1 with PSM_AA and a non-periodic x axis.
 * Ownership: *out is owned by the caller and released with psm_destroy. */
psm_status psm_create(const psm_grid* grid, psm_stencil stencil, double tau,
                      const psm_options* opt, psm_ctx** out);
/* Release the context and everything it allocated.  Collective when world > 1 and the fused
 * peer-store halo is active (psm_halo_mode 2): the neighbours map this rank's memory, so every
 * rank calls psm_destroy (an NCCL barrier precedes the release). */
psm_status psm_destroy(psm_ctx* ctx);

/* Device bytes the big per-rank fields need (PDF storage, solid words, tile flags, partials,
 * staging).  The caller may provide them with psm_bind_memory (e.g. a torch uint8 tensor; it
 * must stay alive until psm_destroy); otherwise the first device call allocates them itself.
 * Per-body geometry fields are always library-allocated (psm_set_body). */
psm_status psm_required_bytes(const psm_ctx* ctx, size_t* bytes);
/* Bind caller-owned device memory; dev_ptr must be 256-byte aligned.  PSM_E_OOM if too small;
 * PSM_E_STATE if memory is already bound/allocated. */
psm_status psm_bind_memory(psm_ctx* ctx, void* dev_ptr, size_t bytes);

/* This rank's slab: global z range [z0, z0 + nz_local). */
psm_status psm_local_extent(const psm_ctx* ctx, int64_t* z0, int64_t* nz_local);

/* Initialise every local cell to f_i = f_i^eq(rho(x), u(x)) of Eq.(3) (with the
 * -u^2/(2 c_s^2) sign, reading A1).  rho: [nz_l][ny][nx] or NULL (= 1);
 * u: [3][nz_l][ny][nx] or NULL (= 0).  Resets the step counter to 0. */
psm_status psm_init_equilibrium(psm_ctx* ctx, const double* rho, const double* u);
/* Write the Eq.(4) state f: [Q][nz_l][ny][nx] fp64 (rounded to the context precision).
 * Resets the step counter to 0. */
psm_status psm_write_pdfs(psm_ctx* ctx, const double* f);
/* Read the Eq.(4) state f: [Q][nz_l][ny][nx] fp64 (converted from the storage pattern). */
psm_status psm_read_pdfs(psm_ctx* ctx, double* f);
/* Read the Eq.(4) state of local planes [z_begin, z_begin + nz): f [Q][nz][ny][nx] fp64 (probes and
 * sampled checks of large grids).  PSM_E_ARG if the range leaves the local slab. */
psm_status psm_read_pdfs_planes(psm_ctx* ctx, int64_t z_begin, int64_t nz, double* f);
/* Read density rho = sum_i f_i [nz_l][ny][nx] and velocity u = sum_i f_i c_i / rho
 * [3][nz_l][ny][nx] of the Eq.(4) state (either pointer may be NULL). */
psm_status psm_read_velocity(psm_ctx* ctx, double* rho, double* u);

/* Rigid body description.  Geometry is given in the BODY frame, lattice units; the body origin is
 * its centre of mass R.  s is the super-sampling exponent (2^s sub-samples per axis,
 * PAPER.md:306-308), 0 <= s <= 3.
 *   PSM_SPHERE: radius > 0.
 *   PSM_MESH  : closed triangle mesh verts[nverts][3] (fp64), tris[ntris][3] (int32, 0-based).
 *               Voxelised ONCE into the super-sampled binary geometry field
 *               by an exact fixed-point ray-parity test (reading A15). */
/* Mesh fraction mapping (reading A12): R1 maps every sub-sample of the world-fixed cell
 * into the body frame (consistent overlap estimator; default); R2 is the paper's literal wording
 * — transform only the cell centre q_c and average the 2^s x 2^s x 2^s geometry
 * cells g with g_a in [g0_a, g0_a + 2^s), g0_a = floor((q_c,a - o_a) 2^s - 2^(s-1) + 1/2). */
typedef enum { PSM_MAP_R1 = 0, PSM_MAP_R2 = 1 } psm_mapping;
typedef struct {
  int32_t kind; /* psm_shape_kind */
  int32_t s;
  double radius;
  const double* verts;
  int64_t nverts;
  const int32_t* tris;
  int64_t ntris;
  int32_t mapping; /* psm_mapping (meshes; spheres always sample, R1) */
} psm_shape;
typedef struct {
  double Q[9]; /* row-major rotation body -> world: x_world = Q x_body + t                   */
  double t[3]; /* world position of the body origin (= centre of mass R)                      */
} psm_pose;
typedef struct {
  double v[3];     /* linear velocity, lattice units per step                                  */
  double omega[3]; /* angular velocity (rad per step) about t, world frame                     */
} psm_velocity;

/* Create or update body `body_id` (1..PSM_MAX_BODIES).  shape == NULL keeps the existing shape
 * (only pose/velocity change, no re-voxelisation).  A body with v == omega == 0 is static: it is
 * mapped here and never remapped.  A moving body advances in closed form from this pose at each
 * psm_step: t_n = t + n v (wrapped on periodic axes), Q_n = Rot(omega/|omega|, n |omega|) Q
 * (Rodrigues, host fp64).  The fraction field of ALL bodies is remapped at the new pose before
 * return.
 * Errors: PSM_E_ARG (id out of range, s out of range, radius <= 0, no shape for a new body, bounding
 * radius + 1 >= half a periodic extent); PSM_E_MESH (index out of range or an edge not shared by
 * exactly two triangles); PSM_E_POSE; PSM_E_OOM (geometry field over the 1 GiB cap). */
#define PSM_MAX_BODIES 16
psm_status psm_set_body(psm_ctx* ctx, int32_t body_id, const psm_shape* shape,
                        const psm_pose* pose, const psm_velocity* vel);
psm_status psm_remove_body(psm_ctx* ctx, int32_t body_id);

/* Two-way coupling (NEXT row of the hot path; the paper's settling-sphere validation couples the
 * PSM force back to the body; its integrator is unstated).
 * With dyn != NULL the body becomes dynamic: after every step the library reduces F, T of
 * Eqs.(10)-(11) on the device (allreduced over ranks), and integrates on the host in fp64:
 *   dv = (F + ext_force + M_a dv_prev) / (mass + M_a);  v += dv;  t += v (wrapped);
 *   I_w = Q I Q^T, A_w = Q I_a Q^T;  dw = (I_w + A_w)^-1 (T + ext_torque + A_w dw_prev);  omega += dw;
 *   Q = Rot(omega/|omega|, |omega|) Q, then Gram-Schmidt on the columns of Q.
 * (M_a, I_a) is an optional virtual mass (default 0: plain semi-implicit Euler): the fluid's
 * reaction to the body's acceleration reaches the body one step late, which makes explicit
 * coupling unstable for density ratios near 1; adding M_a dv on both sides, lagged on the right,
 * cancels that lag (consistent: at constant acceleration the two terms are equal).  A natural
 * choice is the displaced fluid, M_a = rho_f V, I_a = (rho_f V / mass) I (A28).
 * The pose and velocities given to psm_set_body are the initial state.  dyn == NULL returns the
 * body to prescribed motion (closed form from its current state).  Errors: PSM_E_ARG (unknown
 * body, mass <= 0, inertia not symmetric positive definite). */
typedef struct {
  double mass;           /* > 0, lattice units                                                */
  double inertia[9];     /* body-frame inertia tensor about the body origin, row-major        */
  double ext_force[3];   /* constant external force, world frame (e.g. (m - rho_f V) g)       */
  double ext_torque[3];  /* constant external torque, world frame                             */
  double added_mass;     /* M_a >= 0 (virtual-mass stabilisation, see above; 0 = off)         */
  double added_inertia[9];  /* I_a, body frame, symmetric positive semi-definite (0 = off)    */
} psm_dynamics;
psm_status psm_set_dynamics(psm_ctx* ctx, int32_t body_id, const psm_dynamics* dyn);
/* Current pose and velocities of a body (the state the next step will map and use for u_s). */
psm_status psm_get_body_state(const psm_ctx* ctx, int32_t body_id, psm_pose* pose,
                              psm_velocity* vel);

/* Host-only: the super-sampled geometry field psm_set_body builds for a mesh (PAPER.md:299-308,
 * exact ray parity, A15/A17).  dims[3] (geometry cells per axis, = LBM cells * 2^s) and
 * origin[3] (body frame, integer valued) are always written; bits (one byte 0/1 per geometry
 * cell, [dims2][dims1][dims0]) is written if non-NULL and must hold dims0*dims1*dims2 bytes.
 * Errors: PSM_E_ARG (s out of 0..3, NULL arrays), PSM_E_MESH (as psm_set_body). */
psm_status psm_voxelize(const double* verts, int64_t nverts, const int32_t* tris, int64_t ntris,
                        int32_t s, double origin[3], int64_t dims[3], uint8_t* bits);

/* Open-boundary values for bc[0] == PSM_INOUT (reading A30; PAPER.md:584, 593 name the
 * boundaries without defining them):
 *   inflow  (x = 0):      f_q = f*_qbar + 6 w_q rho_w (c_q . u_in), rho_w = 1, for c_qx = +1
 *                         (half-way bounce-back from a wall moving with u_in);
 *   outflow (x = nx - 1): f_q = -f*_qbar + 2 w_q rho_out [1 + 9/2 (c_q . u)^2 - 3/2 u^2] for
 *                         c_qx = -1 (anti-bounce-back), u = (u_x, 0, 0) with
 *                         u_x = (S_0 + 2 S_+) / rho_out - 1 from the known populations of the
 *                         cell (S_0: c_x = 0, S_+: c_x = +1; Zou & He's normal velocity).
 * Defaults u_in = 0, rho_out = 1.  The device keeps the post-collision face sources f*_qbar, and
 * the entering populations are formed with the values current when the state is next stepped or
 * read — set them before psm_init_equilibrium / psm_write_pdfs so the written state is exact.
 * Errors: PSM_E_ARG (NULL, non-finite u_in, rho_out not finite and > 0), PSM_E_UNSUPPORTED
 * (bc[0] != PSM_INOUT). */
psm_status psm_set_open_boundary(psm_ctx* ctx, const double u_in[3], double rho_out);

/* Recompute the solid fraction field of every body at its current pose:
 * eps = (#inside sub-samples) / 2^(3s) (reading R1, A12), B by Eq.(5)/(6). */
psm_status psm_map_fractions(psm_ctx* ctx);

/* Advance n time steps.  Each step: pose advance of moving bodies (host), fraction remap of moving
 * bodies (GPU), fused PSM stream-collide Eq.(4) with the context's fluid operator (SRT Eq.(2)-(3),
 * TRT or cumulant) and SC1/2/3 Eqs.(7)-(9) (GPU), per-body force/torque partials Eqs.(10)-(11)
 * (GPU), halo exchange (world > 1), and for dynamic bodies the coupling integrator (host, one
 * synchronisation per step).  With n > 1 and bodies in prescribed motion the remap of step k+1
 * runs on a second stream while step k collides (results identical to n calls with n = 1).  One
 * D2H copy at the end (error word, force/torque).  PSM_E_STATE if any cell had rho <= 0 or a
 * non-finite value (the first offending step/cell is in psm_last_error()); the state is then
 * undefined.  PSM_E_NCCL if a neighbour rank stopped stepping (fused halo, psm_halo_mode). */
psm_status psm_step(psm_ctx* ctx, int64_t n);

/* Force and torque ON body `body_id` during the most recent step, lattice units (all ranks
 * summed):  F = -sum_x B sum_i Omega^S_i c_i,  T = -sum_x B (x_c - R) x sum_i Omega^S_i c_i.
 * The printed Eqs.(10)-(11) are the momentum the FLUID gains; the sign is
 * flipped so the result is the hydrodynamic load on the solid (reading A6).
 * abs_F/abs_T (may be NULL) return sum |m| and sum |(x_c-R) x m| componentwise (tolerance scale). */
psm_status psm_force_torque(psm_ctx* ctx, int32_t body_id, double F[3], double T[3],
                            double abs_F[3], double abs_T[3]);

/* Read the fraction field of the current step: B [nz_l][ny][nx] fp64 (as used by the collision,
 * before rounding to the context precision), covering body id [nz_l][ny][nx] (0 = none) and the
 * integer sub-sample count [nz_l][ny][nx].  Any pointer may be NULL. */
psm_status psm_read_fractions(psm_ctx* ctx, double* B, uint8_t* body_id, int32_t* count);

/* TEST-ONLY: replace the solid fields by explicit per-cell B [N], u_s [3][N] and id [N] (id 0 =
 * fluid).  Stays in effect until psm_set_body/psm_map_fractions.  PSM_TWO_ARRAY only. */
psm_status psm_debug_set_fields(psm_ctx* ctx, const double* B, const double* us,
                                const uint8_t* id);

/* Diagnostics: current step counter; number of kernels this context launched so far;
 * per-phase device time accumulated while profiling is enabled (CUDA events on the context
 * stream).  Phases: 0 = fraction remap, 1 = stream-collide, 2 = force/torque reduction,
 * 3 = halo exchange. */
#define PSM_NUM_PHASES 4
psm_status psm_get_step(const psm_ctx* ctx, int64_t* step);
psm_status psm_launch_count(const psm_ctx* ctx, int64_t* launches);
psm_status psm_profile(psm_ctx* ctx, int32_t enable);
psm_status psm_profile_read(psm_ctx* ctx, double ms[PSM_NUM_PHASES],
                            int64_t count[PSM_NUM_PHASES]);

/* How the z halo moves between ranks (world > 1, decided collectively at the first psm_step):
 * 0 = single rank, 1 = NCCL grouped send/recv after the collide, 2 = fused: the collide kernel
 * stores the outgoing populations straight into the neighbours' ghost planes (peer memory over
 * NVLink, CUDA IPC), with a per-step flag handshake.  2 needs peer access between every pair of
 * neighbours and PSM_TWO_ARRAY; the environment variable PSM_HALO=nccl forces 1.  With 2 a step
 * waits on the device for both neighbours' previous step, bounded by PSM_P2P_TIMEOUT_S seconds
 * (default 60); a neighbour that never arrives makes psm_step return PSM_E_NCCL. */
psm_status psm_halo_mode(const psm_ctx* ctx, int32_t* mode);

/* Size of an ncclUniqueId (128) and a fresh one for rank 0 to broadcast (world > 1). */
int32_t psm_nccl_id_bytes(void);
psm_status psm_nccl_get_unique_id(void* out128);

/* Thread-local-free: reason for the last failing call on ctx (or a global message if ctx NULL). */
const char* psm_last_error(const psm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PSM_H_ */
