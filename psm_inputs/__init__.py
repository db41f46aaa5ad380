"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no equilibrium, no collision, no mapping): only
random numbers (counter-based splitmix64), the per-config macroscopic initial fields (rho, u)
that each side turns into PDFs with its OWN equilibrium, body placements, and deterministic
triangle meshes.  Both ``oracle`` and ``paper_2502_20049_b200`` consume these arrays; neither
imports the other.  Recipes are documented in DESIGN.md §5.
"""
from __future__ import annotations

import numpy as np

from .meshgen import box_mesh, cylinder_mesh, propeller_mesh, uv_sphere_mesh  # noqa: F401

SEED_BASE = 2502_20049
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """Counter-based splitmix64: element k = mix(seed + (k+1) * golden), uint64."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    """xi in [-1, 1) as fp64: 53 random bits scaled exactly."""
    z = splitmix64(seed, n)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def perturbed_flow(shape, seed: int, rho_amp=0.01, u0=(0.05, 0.0, 0.0), u_amp=0.01):
    """rho = 1 + rho_amp*xi, u = u0 + u_amp*xi (independent xi per value, cell order).

    shape = (nz, ny, nx).  Returns rho [nz,ny,nx] and u [3,nz,ny,nx] (fp64).
    """
    n = int(np.prod(shape))
    xi = uniform_pm1(seed, 4 * n)
    rho = 1.0 + rho_amp * xi[:n].reshape(shape)
    u = np.empty((3,) + tuple(shape))
    for a in range(3):
        u[a] = u0[a] + u_amp * xi[(a + 1) * n:(a + 2) * n].reshape(shape)
    return rho, u


def random_unit(seed: int, n: int) -> np.ndarray:
    """n values uniform in [0, 1)."""
    return (uniform_pm1(seed, n) + 1.0) * 0.5


def random_pdfs(Q: int, shape, seed: int, w=None, amp=0.1):
    """Positive random PDFs f_i = w_i (1 + amp*xi) for invariance tests (w given by caller)."""
    n = int(np.prod(shape))
    xi = uniform_pm1(seed, Q * n).reshape((Q,) + tuple(shape))
    w = np.asarray(w, np.float64).reshape((Q,) + (1,) * len(shape))
    return w * (1.0 + amp * xi)


def rotation_about(axis, angle: float) -> np.ndarray:
    """Input poses: rotation matrix for test inputs (numpy, explicit formula)."""
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


def rot90(axis: int, k: int) -> np.ndarray:
    """Exact rotation by k*90 degrees about a lattice axis (entries in {0, +-1})."""
    k %= 4
    c = [1, 0, -1, 0][k]
    s = [0, 1, 0, -1][k]
    if axis == 0:
        return np.array([[1, 0, 0], [0, c, -s], [0, s, c]], np.float64)
    if axis == 1:
        return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], np.float64)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], np.float64)


def cror_rotor(front: bool, faces: str = "full"):
    """Synthetic CROR rotor of BASELINE config c5 (SURVEY §8(d) recipe): front rotor 12 blades,
    tip 200; rear rotor 10 blades, tip 180; propeller_mesh geometry scaled from the c3 recipe
    (hub r=12, length 48, chord 28->12, pitch 55->20 deg, 4-cell section at tip 110).
    faces="full": ~0.6 M faces per rotor (P:284's ~1.2 M for the pair); "small" for tests."""
    n_bl, tip = (12, 200.0) if front else (10, 180.0)
    n_st, n_pts, hub = (200, 128, 256) if faces == "full" else (16, 24, 32)
    return propeller_mesh(n_blades=n_bl, scale=tip / 110.0, n_st=n_st, n_pts=n_pts,
                          hub_seg=hub)


# ----------------------------------------------------------------------- BASELINE configs ---
CONFIGS = {
    # c1: D3Q19 PSM fp64, 32^3 periodic, stationary sphere r=6 at a lattice vertex, tau=0.8
    "c1": dict(grid=(32, 32, 32), bc=(0, 0, 0), Q=19, tau=0.8, sphere_r=6.0,
               t=(16.0, 16.0, 16.0), v=(0.0, 0.0, 0.0), s=2, steps=100, seed=SEED_BASE + 1),
    # c2: D3Q19 PSM 128x64x64 channel (x periodic, y/z walls), translating sphere, Re = 15
    "c2": dict(grid=(128, 64, 64), bc=(0, 1, 1), Q=19, tau=0.575, sphere_r=6.0,
               t=(32.0, 32.0, 32.0), v=(1.0 / 32.0, 0.0, 0.0), s=2, sc=2, steps=100,
               seed=SEED_BASE + 2),
    # c4: D3Q19 PSM fp32 512^3 roofline sweep, sphere r=64, translating v=1/32, s=1
    "c4": dict(grid=(512, 512, 512), bc=(0, 0, 0), Q=19, tau=0.6, sphere_r=64.0,
               t=(256.0, 256.0, 256.0), v=(1.0 / 32.0, 0.0, 0.0), s=1, sc=1,
               seed=SEED_BASE + 4),
}
