"""TEST INFRASTRUCTURE ONLY — ctypes binding of the plain fp64 CPU oracle (psm_oracle.c).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2502_20049_b200`` never imports it and shares no code with it.

Every method cites the passage of arXiv 2502.20049 (``PAPER.md:<line>``) that the C code it wraps
follows; see ``psm_oracle.c`` for the arithmetic.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "psm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P, D, I, I64 = C.c_void_p, C.c_double, C.c_int, C.c_int64
        sig = {
            "orc_stencil": (None, [I, P, P, P]),
            "orc_equilibrium": (None, [I, D, P, P]),
            "orc_weight_fraction": (D, [D, D, I]),
            "orc_collide_cell": (I, [I, P, D, I, D, P, P, P, P]),
            "orc_collide_cell_trt": (I, [I, P, D, D, I, D, P, P, P, P]),
            "orc_set_collision": (None, [P, I, D]),
            "orc_collide_cell_cum": (I, [I, P, D, I, D, P, P, P, P]),
            "orc_pose_advance": (None, [P, P, P, P, I64, P, P, P, P]),
            "orc_geometry_extent": (I64, [P, I64, I, P, P]),
            "orc_voxelize": (None, [P, I64, P, I64, I, P]),
            "orc_create": (P, [I, I, I, I, D, P, I, I]),
            "orc_destroy": (None, [P]),
            "orc_set_force": (None, [P, P]),
            "orc_set_open_boundary": (None, [P, P, D]),
            "orc_set_map_all_cells": (None, [P, I]),
            "orc_init_equilibrium": (None, [P, P, P]),
            "orc_set_pdfs": (None, [P, P]),
            "orc_get_pdfs": (None, [P, P]),
            "orc_get_velocity": (None, [P, P, P]),
            "orc_set_sphere": (I, [P, I, D, I]),
            "orc_set_mesh": (I, [P, I, P, I64, P, I64, I]),
            "orc_remove_body": (None, [P, I]),
            "orc_get_geometry": (I, [P, I, P, P, P]),
            "orc_set_pose": (None, [P, I, P, P, P, P]),
            "orc_map": (None, [P]),
            "orc_set_fields": (None, [P, P, P, P]),
            "orc_get_fractions": (None, [P, P, P, P, P]),
            "orc_step": (I, [P]),
            "orc_error_cell": (I64, [P]),
            "orc_force_torque": (None, [P, I, P, P, P, P]),
            "orc_set_dynamics": (None, [P, I, D, P, P, P, D, P]),
            "orc_set_mapping": (None, [P, I, I]),
            "orc_integrate": (None, [P]),
            "orc_get_body_state": (None, [P, I, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- pure functions (for pins) ---
def stencil(Q: int):
    """(c [Q,3] int32, w [Q] f64, opp [Q] int32) in the ABI order."""
    c = np.zeros((Q, 3), np.int32)
    w = np.zeros(Q, np.float64)
    opp = np.zeros(Q, np.int32)
    lib().orc_stencil(Q, _p(c), _p(w), _p(opp))
    return c, w, opp


def equilibrium(Q: int, rho: float, u) -> np.ndarray:
    """Eq.(3), PAPER.md:138-140 (u^2 sign per reading A1)."""
    u = _f64(u)
    out = np.zeros(Q, np.float64)
    lib().orc_equilibrium(Q, float(rho), _p(u), _p(out))
    return out


def weight_fraction(eps: float, tau: float, mode: int) -> float:
    """Eq.(5) (mode 0) / Eq.(6) (mode 1)."""
    return lib().orc_weight_fraction(float(eps), float(tau), int(mode))


def collide_cell(Q, f, tau, sc, B, us, g=(0.0, 0.0, 0.0)):
    """One-cell Eq.(4) collision; returns (f*, m = B sum_i Omega^S_i c_i, err)."""
    f = _f64(f)
    us = _f64(us)
    g = _f64(g)
    out = np.zeros(Q, np.float64)
    m = np.zeros(3, np.float64)
    err = lib().orc_collide_cell(Q, _p(f), float(tau), int(sc), float(B), _p(us), _p(g),
                                 _p(out), _p(m))
    return out, m, err


def collide_cell_trt(Q, f, tau, magic, sc, B, us, g=(0.0, 0.0, 0.0)):
    """One-cell Eq.(4) collision with the TRT fluid operator."""
    f = _f64(f)
    us = _f64(us)
    g = _f64(g)
    out = np.zeros(Q, np.float64)
    m = np.zeros(3, np.float64)
    err = lib().orc_collide_cell_trt(Q, _p(f), float(tau), float(magic), int(sc), float(B),
                                     _p(us), _p(g), _p(out), _p(m))
    return out, m, err


def collide_cell_cum(Q, f, tau, sc, B, us, g=(0.0, 0.0, 0.0)):
    """One-cell Eq.(4) collision with the cumulant fluid operator (D3Q27 reading A29, D3Q19
    reading A32), optional body force g (reading A31)."""
    f = _f64(f)
    us = _f64(us)
    g = _f64(g)
    out = np.zeros(Q, np.float64)
    m = np.zeros(3, np.float64)
    err = lib().orc_collide_cell_cum(Q, _p(f), float(tau), int(sc), float(B), _p(us), _p(g),
                                     _p(out), _p(m))
    return out, m, err


def pose_advance(Q0, t0, v, w, n, L, periodic):
    """Closed-form prescribed pose after n steps (A13)."""
    Qn = np.zeros(9)
    tn = np.zeros(3)
    keep = [_f64(np.ravel(Q0)), _f64(t0), _f64(v), _f64(w), _f64(L),
            np.ascontiguousarray(periodic, np.int32)]
    lib().orc_pose_advance(_p(keep[0]), _p(keep[1]), _p(keep[2]), _p(keep[3]), int(n),
                           _p(keep[4]), _p(keep[5]), _p(Qn), _p(tn))
    return Qn.reshape(3, 3), tn


def voxelize(verts, tris, s: int):
    """Geometry field of a closed mesh (A15): (origin[3], bits[gz,gy,gx] u8)."""
    verts = _f64(verts)
    tris = np.ascontiguousarray(tris, np.int32)
    origin = np.zeros(3)
    dims = np.zeros(3, np.int64)
    n = lib().orc_geometry_extent(_p(verts), len(verts), s, _p(origin), _p(dims))
    bits = np.zeros(n, np.uint8)
    lib().orc_voxelize(_p(verts), len(verts), _p(tris), len(tris), s, _p(bits))
    return origin, bits.reshape(dims[2], dims[1], dims[0])


# ------------------------------------------------------------------------------ simulation ---
class Oracle:
    """Plain PSM-LBM simulation on the whole grid (fp64, push form, Eq.(4) state)."""

    def __init__(self, nx, ny, nz, Q=19, tau=0.8, bc=(0, 0, 0), sc=1, bmode=1):
        self.nx, self.ny, self.nz, self.Q = nx, ny, nz, Q
        self.N = nx * ny * nz
        bc = np.ascontiguousarray(bc, np.int32)
        self._h = lib().orc_create(nx, ny, nz, Q, float(tau), _p(bc), sc, bmode)
        assert self._h

    def close(self):
        if self._h:
            lib().orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_force(self, g):
        g = _f64(g)
        lib().orc_set_force(self._h, _p(g))

    def set_open_boundary(self, u_in=(0.0, 0.0, 0.0), rho_out: float = 1.0):
        """bc[0] == 2: velocity inflow u_in at x = 0, pressure outflow rho_out at x = nx-1
        (reading A30)."""
        u = _f64(u_in)
        lib().orc_set_open_boundary(self._h, _p(u), float(rho_out))

    def set_collision(self, kind: str = "srt", magic: float = 3.0 / 16.0):
        lib().orc_set_collision(self._h, {"srt": 0, "trt": 1, "cumulant": 2}[kind], float(magic))

    def set_map_all_cells(self, on: bool):
        lib().orc_set_map_all_cells(self._h, int(bool(on)))

    def init_equilibrium(self, rho=None, u=None):
        rho, u = _f64(rho), _f64(u)
        lib().orc_init_equilibrium(self._h, _p(rho), _p(u))

    def set_pdfs(self, f):
        f = _f64(f)
        assert f.size == self.Q * self.N
        lib().orc_set_pdfs(self._h, _p(f))

    def pdfs(self):
        out = np.zeros((self.Q, self.nz, self.ny, self.nx))
        lib().orc_get_pdfs(self._h, _p(out))
        return out

    def velocity(self):
        rho = np.zeros((self.nz, self.ny, self.nx))
        u = np.zeros((3, self.nz, self.ny, self.nx))
        lib().orc_get_velocity(self._h, _p(rho), _p(u))
        return rho, u

    def set_sphere(self, bid, r, s):
        assert lib().orc_set_sphere(self._h, bid, float(r), s) == 0

    def set_mesh(self, bid, verts, tris, s):
        verts = _f64(verts)
        tris = np.ascontiguousarray(tris, np.int32)
        assert lib().orc_set_mesh(self._h, bid, _p(verts), len(verts), _p(tris), len(tris), s) == 0

    def set_mapping(self, bid, mode: str):
        """Mesh fraction mapping: "R1" every sub-sample (default) or "R2" centre only (A12)."""
        lib().orc_set_mapping(self._h, bid, 1 if mode == "R2" else 0)

    def remove_body(self, bid):
        lib().orc_remove_body(self._h, bid)

    def set_pose(self, bid, Q=np.eye(3), t=(0, 0, 0), v=(0, 0, 0), w=(0, 0, 0)):
        keep = [_f64(np.ravel(Q)), _f64(t), _f64(v), _f64(w)]
        lib().orc_set_pose(self._h, bid, *[_p(k) for k in keep])

    def map(self):
        lib().orc_map(self._h)

    def set_fields(self, B, us, bid):
        keep = [_f64(B), _f64(us), np.ascontiguousarray(bid, np.uint8)]
        lib().orc_set_fields(self._h, *[_p(k) for k in keep])

    def fractions(self):
        sh = (self.nz, self.ny, self.nx)
        B = np.zeros(sh)
        bid = np.zeros(sh, np.uint8)
        cnt = np.zeros(sh, np.int32)
        us = np.zeros((3,) + sh)
        lib().orc_get_fractions(self._h, _p(B), _p(bid), _p(cnt), _p(us))
        return B, bid, cnt, us

    def step(self, n: int = 1):
        for _ in range(n):
            err = lib().orc_step(self._h)
            if err:
                raise FloatingPointError(
                    f"oracle: invalid state at cell {lib().orc_error_cell(self._h)}")

    def set_dynamics(self, bid, mass, inertia, ext_force=(0, 0, 0), ext_torque=(0, 0, 0),
                     added_mass=0.0, added_inertia=None):
        ai = np.zeros(9) if added_inertia is None else np.ravel(added_inertia)
        keep = [_f64(np.ravel(inertia)), _f64(ext_force), _f64(ext_torque), _f64(ai)]
        lib().orc_set_dynamics(self._h, bid, float(mass), _p(keep[0]), _p(keep[1]), _p(keep[2]),
                               float(added_mass), _p(keep[3]))

    def integrate(self):
        """Advance the dynamic bodies with the force/torque of the last step (two-way coupling)."""
        lib().orc_integrate(self._h)

    def body_state(self, bid):
        Q, t, v, w = np.zeros(9), np.zeros(3), np.zeros(3), np.zeros(3)
        lib().orc_get_body_state(self._h, bid, _p(Q), _p(t), _p(v), _p(w))
        return Q.reshape(3, 3), t, v, w

    def force_torque(self, bid):
        F, T, AF, AT = (np.zeros(3) for _ in range(4))
        lib().orc_force_torque(self._h, bid, _p(F), _p(T), _p(AF), _p(AT))
        return F, T, AF, AT
