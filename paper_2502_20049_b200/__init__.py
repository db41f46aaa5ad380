"""B200-native PSM lattice Boltzmann hot path (arXiv 2502.20049) — thin Python binding.

Marshals arguments to the C ABI of ``libpsm.so`` (declared in ``include/psm.h``); every step of
the method runs in the library's sm_100a kernels.  PyTorch is used only for device memory
(``psm_bind_memory`` of a ``torch.uint8`` CUDA tensor), the CUDA stream, and
``torch.distributed`` (to broadcast the NCCL unique id).  There is no CPU fallback: if the
library is missing or no CUDA device is present, the calls raise.

Function names follow the ABI (``psm_create``, ``psm_set_body``, ``psm_map_fractions``,
``psm_step``, ``psm_force_torque``, ``psm_read_pdfs``, ``psm_read_velocity``, ...);
``Simulation`` bundles them for convenience.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpsm.so")

PSM_OK, PSM_E_ARG, PSM_E_OOM, PSM_E_MESH, PSM_E_POSE, PSM_E_STATE, PSM_E_CUDA, PSM_E_NCCL, \
    PSM_E_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7, -8
PSM_D3Q19, PSM_D3Q27 = 19, 27
PSM_SC1, PSM_SC2, PSM_SC3 = 1, 2, 3
PSM_B_DIRECT, PSM_B_WEIGHTED = 0, 1
PSM_F64, PSM_F32 = 0, 1
PSM_TWO_ARRAY, PSM_AA = 0, 1
PSM_PERIODIC, PSM_WALL, PSM_INOUT = 0, 1, 2
PSM_SPHERE, PSM_MESH = 0, 1
PSM_SRT, PSM_TRT, PSM_CUMULANT = 0, 1, 2
PSM_MAP_R1, PSM_MAP_R2 = 0, 1
PSM_MAX_BODIES = 16
PSM_NUM_PHASES = 4
PHASES = ("map", "collide", "ft_reduce", "halo")

EXPORTED = (
    "psm_create", "psm_destroy", "psm_required_bytes", "psm_bind_memory", "psm_local_extent",
    "psm_init_equilibrium", "psm_write_pdfs", "psm_read_pdfs", "psm_read_pdfs_planes",
    "psm_read_velocity",
    "psm_set_body", "psm_remove_body", "psm_voxelize", "psm_set_dynamics",
    "psm_set_open_boundary",
    "psm_get_body_state", "psm_map_fractions", "psm_step", "psm_force_torque",
    "psm_read_fractions", "psm_debug_set_fields", "psm_get_step", "psm_launch_count",
    "psm_profile", "psm_profile_read", "psm_nccl_id_bytes", "psm_nccl_get_unique_id",
    "psm_halo_mode",
    "psm_last_error",
)


class psm_grid(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("bc", C.c_int32 * 3)]


class psm_options(C.Structure):
    _fields_ = [("prec", C.c_int32), ("pattern", C.c_int32), ("sc", C.c_int32),
                ("bmode", C.c_int32), ("body_force", C.c_double * 3), ("rank", C.c_int32),
                ("world", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("cuda_stream", C.c_void_p), ("collision", C.c_int32),
                ("trt_magic", C.c_double)]


class psm_shape(C.Structure):
    _fields_ = [("kind", C.c_int32), ("s", C.c_int32), ("radius", C.c_double),
                ("verts", C.c_void_p), ("nverts", C.c_int64), ("tris", C.c_void_p),
                ("ntris", C.c_int64), ("mapping", C.c_int32)]


class psm_pose(C.Structure):
    _fields_ = [("Q", C.c_double * 9), ("t", C.c_double * 3)]


class psm_velocity(C.Structure):
    _fields_ = [("v", C.c_double * 3), ("omega", C.c_double * 3)]


class psm_dynamics(C.Structure):
    _fields_ = [("mass", C.c_double), ("inertia", C.c_double * 9),
                ("ext_force", C.c_double * 3), ("ext_torque", C.c_double * 3),
                ("added_mass", C.c_double), ("added_inertia", C.c_double * 9)]


class PSMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"psm error {code}: {msg}")
        self.code = code


_lib = None


def load(build_if_missing: bool = True):
    """Load libpsm.so (building it with nvcc first if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build
    alt = os.environ.get("PSM_LIB")  # kernel-tuning experiments: an in-tree variant build
    if alt:
        L = C.CDLL(os.path.abspath(alt))
    else:
        if build_if_missing and _build.needs_build():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
    P, I32, I64, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t
    sig = {
        "psm_create": [P, I32, D, P, P], "psm_destroy": [P], "psm_required_bytes": [P, P],
        "psm_bind_memory": [P, P, SZ], "psm_local_extent": [P, P, P],
        "psm_init_equilibrium": [P, P, P], "psm_write_pdfs": [P, P], "psm_read_pdfs": [P, P],
        "psm_read_velocity": [P, P, P], "psm_set_body": [P, I32, P, P, P],
        "psm_read_pdfs_planes": [P, I64, I64, P],
        "psm_remove_body": [P, I32], "psm_map_fractions": [P],
        "psm_voxelize": [P, I64, P, I64, I32, P, P, P], "psm_step": [P, I64],
        "psm_set_dynamics": [P, I32, P], "psm_get_body_state": [P, I32, P, P],
        "psm_set_open_boundary": [P, P, C.c_double],
        "psm_force_torque": [P, I32, P, P, P, P], "psm_read_fractions": [P, P, P, P],
        "psm_debug_set_fields": [P, P, P, P], "psm_get_step": [P, P],
        "psm_launch_count": [P, P], "psm_profile": [P, I32], "psm_profile_read": [P, P, P],
        "psm_nccl_get_unique_id": [P], "psm_halo_mode": [P, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.psm_nccl_id_bytes.argtypes = []
    L.psm_nccl_id_bytes.restype = C.c_int32
    L.psm_last_error.argtypes = [P]
    L.psm_last_error.restype = C.c_char_p
    _lib = L
    return L


def _check(code, ctx=None):
    if code != PSM_OK:
        msg = load().psm_last_error(ctx)
        raise PSMError(code, msg.decode() if msg else "")


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _c64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        assert a.size == int(np.prod(shape)), (a.shape, shape)
    return a


# ---------------------------------------------------------------- ABI-named thin wrappers ---
def psm_create(grid: psm_grid, stencil: int, tau: float, opt: psm_options):
    ctx = C.c_void_p()
    _check(load().psm_create(C.byref(grid), stencil, float(tau), C.byref(opt), C.byref(ctx)))
    return ctx


def psm_destroy(ctx):
    _check(load().psm_destroy(ctx))


def psm_required_bytes(ctx) -> int:
    n = C.c_size_t()
    _check(load().psm_required_bytes(ctx, C.byref(n)), ctx)
    return n.value


def psm_bind_memory(ctx, dev_ptr: int, nbytes: int):
    _check(load().psm_bind_memory(ctx, C.c_void_p(dev_ptr), nbytes), ctx)


def psm_local_extent(ctx):
    z0, nzl = C.c_int64(), C.c_int64()
    _check(load().psm_local_extent(ctx, C.byref(z0), C.byref(nzl)), ctx)
    return z0.value, nzl.value


def psm_init_equilibrium(ctx, rho=None, u=None):
    _check(load().psm_init_equilibrium(ctx, _ptr(rho), _ptr(u)), ctx)


def psm_write_pdfs(ctx, f):
    _check(load().psm_write_pdfs(ctx, _ptr(f)), ctx)


def psm_read_pdfs(ctx, out):
    _check(load().psm_read_pdfs(ctx, _ptr(out)), ctx)


def psm_read_pdfs_planes(ctx, z_begin: int, nz: int, out):
    _check(load().psm_read_pdfs_planes(ctx, int(z_begin), int(nz), _ptr(out)), ctx)


def psm_read_velocity(ctx, rho, u):
    _check(load().psm_read_velocity(ctx, _ptr(rho), _ptr(u)), ctx)


def psm_set_body(ctx, body_id: int, shape, pose: psm_pose, vel: psm_velocity):
    _check(load().psm_set_body(ctx, body_id, None if shape is None else C.byref(shape),
                               C.byref(pose), C.byref(vel)), ctx)


def psm_remove_body(ctx, body_id: int):
    _check(load().psm_remove_body(ctx, body_id), ctx)


def psm_voxelize(verts, tris, s: int):
    """Host-side geometry field of a closed mesh: (origin[3], bits[gz, gy, gx] uint8)."""
    verts = _c64(verts)
    tris = np.ascontiguousarray(tris, np.int32)
    origin = np.zeros(3)
    dims = np.zeros(3, np.int64)
    L = load()
    _check(L.psm_voxelize(_ptr(verts), len(verts), _ptr(tris), len(tris), s, _ptr(origin),
                          _ptr(dims), None))
    bits = np.zeros(int(np.prod(dims)), np.uint8)
    _check(L.psm_voxelize(_ptr(verts), len(verts), _ptr(tris), len(tris), s, _ptr(origin),
                          _ptr(dims), _ptr(bits)))
    return origin, bits.reshape(int(dims[2]), int(dims[1]), int(dims[0]))


def psm_set_dynamics(ctx, body_id: int, dyn):
    _check(load().psm_set_dynamics(ctx, body_id, None if dyn is None else C.byref(dyn)), ctx)


def psm_set_open_boundary(ctx, u_in, rho_out: float = 1.0):
    u = (C.c_double * 3)(*[float(v) for v in u_in])
    _check(load().psm_set_open_boundary(ctx, u, float(rho_out)), ctx)


def psm_get_body_state(ctx, body_id: int):
    pose, vel = psm_pose(), psm_velocity()
    _check(load().psm_get_body_state(ctx, body_id, C.byref(pose), C.byref(vel)), ctx)
    return (np.array(pose.Q[:]).reshape(3, 3), np.array(pose.t[:]), np.array(vel.v[:]),
            np.array(vel.omega[:]))


def psm_map_fractions(ctx):
    _check(load().psm_map_fractions(ctx), ctx)


def psm_step(ctx, n: int = 1):
    _check(load().psm_step(ctx, int(n)), ctx)


def psm_force_torque(ctx, body_id: int):
    F, T, aF, aT = (np.zeros(3) for _ in range(4))
    _check(load().psm_force_torque(ctx, body_id, _ptr(F), _ptr(T), _ptr(aF), _ptr(aT)), ctx)
    return F, T, aF, aT


def psm_read_fractions(ctx, B, bid, cnt):
    _check(load().psm_read_fractions(ctx, _ptr(B), _ptr(bid), _ptr(cnt)), ctx)


def psm_debug_set_fields(ctx, B, us, bid):
    _check(load().psm_debug_set_fields(ctx, _ptr(B), _ptr(us), _ptr(bid)), ctx)


def psm_launch_count(ctx) -> int:
    n = C.c_int64()
    _check(load().psm_launch_count(ctx, C.byref(n)), ctx)
    return n.value


def psm_halo_mode(ctx) -> int:
    """0 single rank, 1 NCCL send/recv halo, 2 fused peer-store halo (decided at the first
    psm_step of a multi-rank context)."""
    m = C.c_int32()
    _check(load().psm_halo_mode(ctx, C.byref(m)), ctx)
    return m.value


def psm_get_step(ctx) -> int:
    n = C.c_int64()
    _check(load().psm_get_step(ctx, C.byref(n)), ctx)
    return n.value


def psm_profile(ctx, enable: bool):
    _check(load().psm_profile(ctx, int(bool(enable))), ctx)


def psm_profile_read(ctx):
    ms = (C.c_double * PSM_NUM_PHASES)()
    cnt = (C.c_int64 * PSM_NUM_PHASES)()
    _check(load().psm_profile_read(ctx, ms, cnt), ctx)
    return {PHASES[i]: (ms[i], cnt[i]) for i in range(PSM_NUM_PHASES)}


def psm_nccl_get_unique_id() -> bytes:
    n = load().psm_nccl_id_bytes()
    buf = (C.c_uint8 * n)()
    _check(load().psm_nccl_get_unique_id(buf))
    return bytes(buf)


# ------------------------------------------------------------------------ convenience -------
class Simulation:
    """One rank's PSM simulation context (z-slab of the global grid)."""

    def __init__(self, nx, ny, nz, Q=19, tau=0.8, bc=(0, 0, 0), prec="f64", pattern="two_array",
                 sc=1, bmode=1, body_force=(0.0, 0.0, 0.0), rank=0, world=1, nccl_id=None,
                 stream=None, device=None, collision="srt", trt_magic=3.0 / 16.0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2502_20049_b200 needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else device)
        self.Q = Q
        self.nx, self.ny, self.nz = nx, ny, nz
        g = psm_grid(nx, ny, nz, (C.c_int32 * 3)(*bc))
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._idbuf = None
        if world > 1:
            self._idbuf = (C.c_uint8 * len(nccl_id)).from_buffer_copy(nccl_id)
        o = psm_options(PSM_F64 if prec == "f64" else PSM_F32,
                        PSM_TWO_ARRAY if pattern == "two_array" else PSM_AA, sc, bmode,
                        (C.c_double * 3)(*body_force), rank, world,
                        C.cast(self._idbuf, C.c_void_p) if self._idbuf is not None else None,
                        C.c_void_p(self._stream.cuda_stream),
                        {"srt": PSM_SRT, "trt": PSM_TRT, "cumulant": PSM_CUMULANT}[collision],
                        float(trt_magic))
        self.ctx = psm_create(g, Q, tau, o)
        nbytes = psm_required_bytes(self.ctx)
        self.mem = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.mem.data_ptr()
        aligned = (base + 255) & ~255
        psm_bind_memory(self.ctx, aligned, nbytes)
        self.z0, self.nzl = psm_local_extent(self.ctx)
        self.shape = (self.nzl, ny, nx)
        self.N = self.nzl * ny * nx

    def close(self):
        if getattr(self, "ctx", None):
            psm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_equilibrium(self, rho=None, u=None):
        rho = _c64(rho, self.shape)
        u = _c64(u, (3,) + self.shape)
        psm_init_equilibrium(self.ctx, rho, u)

    def write_pdfs(self, f):
        psm_write_pdfs(self.ctx, _c64(f, (self.Q,) + self.shape))

    def pdfs(self):
        out = np.empty((self.Q,) + self.shape)
        psm_read_pdfs(self.ctx, out)
        return out

    def pdfs_planes(self, z_begin, nz):
        out = np.empty((self.Q, nz, self.ny, self.nx))
        psm_read_pdfs_planes(self.ctx, z_begin, nz, out)
        return out

    def velocity(self):
        rho = np.empty(self.shape)
        u = np.empty((3,) + self.shape)
        psm_read_velocity(self.ctx, rho, u)
        return rho, u

    def set_sphere(self, bid, r, s, Q=np.eye(3), t=(0, 0, 0), v=(0, 0, 0), w=(0, 0, 0)):
        sh = psm_shape(PSM_SPHERE, s, float(r), None, 0, None, 0, PSM_MAP_R1)
        psm_set_body(self.ctx, bid, sh, _pose(Q, t), _vel(v, w))

    def set_mesh(self, bid, verts, tris, s, Q=np.eye(3), t=(0, 0, 0), v=(0, 0, 0),
                 w=(0, 0, 0), mapping="R1"):
        verts = _c64(verts)
        tris = np.ascontiguousarray(tris, np.int32)
        sh = psm_shape(PSM_MESH, s, 0.0, verts.ctypes.data, len(verts), tris.ctypes.data,
                       len(tris), PSM_MAP_R2 if mapping == "R2" else PSM_MAP_R1)
        psm_set_body(self.ctx, bid, sh, _pose(Q, t), _vel(v, w))

    def set_pose(self, bid, Q=np.eye(3), t=(0, 0, 0), v=(0, 0, 0), w=(0, 0, 0)):
        psm_set_body(self.ctx, bid, None, _pose(Q, t), _vel(v, w))

    def set_dynamics(self, bid, mass=None, inertia=None, ext_force=(0, 0, 0),
                     ext_torque=(0, 0, 0), added_mass=0.0, added_inertia=None):
        """Two-way coupled body (mass=None: back to prescribed motion); optional virtual mass
        (added_mass, added_inertia) for density ratios near 1 (psm.h, A28)."""
        if mass is None:
            psm_set_dynamics(self.ctx, bid, None)
            return
        ai = np.zeros(9) if added_inertia is None else np.ravel(added_inertia)
        d = psm_dynamics(float(mass), (C.c_double * 9)(*np.ravel(inertia)),
                         (C.c_double * 3)(*ext_force), (C.c_double * 3)(*ext_torque),
                         float(added_mass), (C.c_double * 9)(*ai))
        psm_set_dynamics(self.ctx, bid, d)

    def body_state(self, bid):
        return psm_get_body_state(self.ctx, bid)

    def set_open_boundary(self, u_in=(0.0, 0.0, 0.0), rho_out=1.0):
        """bc[0] == PSM_INOUT: inflow velocity at x = 0, outflow density at x = nx-1 (A30)."""
        psm_set_open_boundary(self.ctx, u_in, rho_out)

    def remove_body(self, bid):
        psm_remove_body(self.ctx, bid)

    def map_fractions(self):
        psm_map_fractions(self.ctx)

    def step(self, n=1):
        psm_step(self.ctx, n)

    def force_torque(self, bid):
        return psm_force_torque(self.ctx, bid)

    def fractions(self):
        B = np.empty(self.shape)
        bid = np.empty(self.shape, np.uint8)
        cnt = np.empty(self.shape, np.int32)
        psm_read_fractions(self.ctx, B, bid, cnt)
        return B, bid, cnt

    def debug_set_fields(self, B, us, bid):
        psm_debug_set_fields(self.ctx, _c64(B, self.shape), _c64(us, (3,) + self.shape),
                             np.ascontiguousarray(bid, np.uint8))

    @property
    def launches(self):
        return psm_launch_count(self.ctx)

    @property
    def step_count(self):
        return psm_get_step(self.ctx)

    def profile(self, on=True):
        psm_profile(self.ctx, on)

    def profile_read(self):
        return psm_profile_read(self.ctx)


def _pose(Q, t):
    Q = np.asarray(Q, np.float64).reshape(9)
    return psm_pose((C.c_double * 9)(*Q), (C.c_double * 3)(*[float(x) for x in t]))


def _vel(v, w):
    return psm_velocity((C.c_double * 3)(*[float(x) for x in v]),
                        (C.c_double * 3)(*[float(x) for x in w]))
