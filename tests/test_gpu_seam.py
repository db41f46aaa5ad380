"""GPU parity of the fraction remap at periodic seams and ragged tiles.

The method maps every sub-sample with its own minimum image, d = mi(p - t) (PAPER.md:313-317,
reading A14).  A region (tile, segment, cell) whose cells lie on both sides of the cut at
t +- L/2 therefore cannot be decided from its centre; in a ragged last tile the unclamped tile
centre even lies beyond the grid edge and wraps to the far side of the body.  These tests put
large bodies next to their seams on grids that are not multiples of the 32x4x2 tile and require
the counts to be bit-exact against the oracle at every step, through every remap path: the
full narrow-band pipeline, the cached band (margin 1), remap-ahead, the general multi-body
kernel, and the list-overflow fallbacks (forced small list capacities).
"""
import contextlib
import os

import numpy as np
import pytest

import oracle
import psm_inputs as pi

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def _env(**kv):
    """Remap switches are read at psm_create (psm_ctx.h): set them around the construction."""
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _sim(env=None, **kw):
    import paper_2502_20049_b200 as psm
    with _env(**(env or {})):
        return psm.Simulation(**kw)


# ------------------------------------------------------------------ Table I at N = 40 -------
def _table1_pose(k, steps=100):
    # the cube rotates about all three axes over the 100 steps
    return pi.rotation_about([1.0, 2.0, 3.0], k * (np.pi / 2) / steps) @ pi.rotation_about(
        [1, 0, 0], 0.1)


@pytest.mark.parametrize("mapping", ["R1", "R2"])
@pytest.mark.parametrize("s", [0, 1, 2])
def test_table1_cube_n40_counts_bit_exact(s, mapping):
    """Table I protocol at N = 40 on the 78^3 grid of
    tools/table1_cube.py (78 = 2 x 32 + 14: a ragged tile column next to the seam of a cube
    whose corners reach 34.6 of the 39 cells to the cut): all 100 poses, counts bit-exact."""
    N = 40
    n = int(np.ceil(N * np.sqrt(3))) + 8
    v, t = pi.box_mesh([-N / 2] * 3, [N / 2] * 3)
    c = np.array([n / 2 + 0.13, n / 2 + 0.29, n / 2 + 0.41])
    o = oracle.Oracle(n, n, n, 19, 0.8, (0, 0, 0), 1, 1)
    o.set_mesh(1, v, t, s)
    o.set_mapping(1, mapping)
    g = _sim(nx=n, ny=n, nz=n, Q=19, tau=0.8, prec="f32")
    for k in range(100):
        Q = _table1_pose(k)
        if k == 0:
            g.set_mesh(1, v, t, s, Q, c, mapping=mapping)
        else:
            g.set_pose(1, Q, c)
        o.set_pose(1, Q, c)
        o.map()
        co = o.fractions()[2]
        cg = g.fractions()[2]
        assert np.array_equal(co, cg), (k, int((co != cg).sum()))
    g.close()


# ---------------------------------------------------- large rotating body at its seam -------
GRID = (70, 45, 38)  # ragged in x (70 = 2 x 32 + 6), y (45 = 11 x 4 + 1) and z (38 = 19 x 2)


def _seam_propeller():
    v, tr = pi.propeller_mesh(n_blades=3, scale=1.0, n_st=10, n_pts=16, hub_seg=16)
    rb = np.max(np.linalg.norm(v, axis=1))
    # bounding radius 17.5 of the 18 the library accepts on the 38-cell z axis (r + 1 < L/2)
    return v * (17.5 / rb), tr


def _pose_fn(Q0, t0, v, w):
    return lambda k: oracle.pose_advance(Q0, t0, v, w, k, list(GRID), [1, 1, 1])


SEAM_CASES = {
    # (body, s, psm_step call size, remap env switches)
    "mesh_s1_band": ("mesh", 1, 1, {}),
    "mesh_s1_ahead": ("mesh", 1, 4, {}),
    "mesh_s1_nocache": ("mesh", 1, 1, {"PSM_BAND_CACHE": "0"}),
    "mesh_s1_general": ("mesh", 1, 1, {"PSM_REMAP_GENERAL": "1"}),
    "mesh_s1_overflow": ("mesh", 1, 1, {"PSM_SEG_CAP": "7", "PSM_BAND_CAP": "13"}),
    "mesh_s1_overflow_nocache": ("mesh", 1, 1, {"PSM_SEG_CAP": "5", "PSM_BAND_CAP": "11",
                                                 "PSM_BAND_CACHE": "0"}),
    "mesh_s2_ahead": ("mesh", 2, 3, {}),
    "mesh_s2_overflow": ("mesh", 2, 1, {"PSM_SEG_CAP": "9", "PSM_BAND_CAP": "17"}),
    "sphere_s1_band": ("sphere", 1, 1, {}),
    "sphere_s2_general": ("sphere", 2, 1, {"PSM_REMAP_GENERAL": "1"}),
    # the two-launch L1/L2 form (PSM_REMAP_L12=0) and the R2 mapping's cached band at s = 2, 3
    "mesh_s2_l1l2": ("mesh", 2, 1, {"PSM_REMAP_L12": "0"}),
    "mesh_s2_r2_band": ("mesh", 2, 1, {}, "R2"),
    "mesh_s3_r2_ahead": ("mesh", 3, 2, {}, "R2"),
}


@pytest.mark.parametrize("case", sorted(SEAM_CASES))
def test_large_body_at_periodic_seam(case):
    """A body of bounding radius 17.5 (the limit on the 38-cell axis is < 18) centred next to
    the domain corner, rotating about an oblique axis and translating across every periodic
    boundary, remapped by the library's own closed-form advance (psm_step, rows a1/a2): the
    library's pose equals oracle.pose_advance bit for bit and the counts are bit-exact against
    the oracle at every checked step."""
    kind, s, chunk, env = SEAM_CASES[case][:4]
    mapping = SEAM_CASES[case][4] if len(SEAM_CASES[case]) > 4 else "R1"
    nx, ny, nz = GRID
    Q0 = pi.rotation_about([0.3, -1.0, 0.5], 0.7)
    t0 = [66.3, 2.1, 36.7]
    # the solid sphere displaces far more fluid than the thin blades: slower (surface speed
    # <= 0.1, lattice Mach limit) so that the fluid it drives stays stable for the 24 steps
    sv = 1.0 if kind == "mesh" else 0.3
    v = [0.11 * sv, -0.07 * sv, 0.05 * sv]
    w = np.array([0.012, 0.02, -0.009]) * sv
    pose = _pose_fn(Q0, t0, v, w)
    o = oracle.Oracle(nx, ny, nz, 19, 0.9, (0, 0, 0), 1, 1)
    o.set_map_all_cells(True)  # brute force over every cell: no bounding box on the oracle side
    g = _sim(env, nx=nx, ny=ny, nz=nz, Q=19, tau=0.9, prec="f32")
    g.init_equilibrium()
    if kind == "mesh":
        mv, mt = _seam_propeller()
        o.set_mesh(1, mv, mt, s)
        o.set_mapping(1, mapping)
        g.set_mesh(1, mv, mt, s, Q0, t0, v, w, mapping=mapping)
    else:
        o.set_sphere(1, 17.5, s)
        g.set_sphere(1, 17.5, s, Q0, t0, v, w)
    steps = 24
    done = 0
    while done < steps:
        g.step(chunk)
        done += chunk
        k = done - 1  # the words in use were mapped at the pose of the call's last step
        Qk, tk = pose(k)
        Qg, tg, _, _ = g.body_state(1)
        Qn, tn = pose(done)
        assert np.array_equal(Qg, Qn) and np.array_equal(tg, tn), (done, Qg - Qn, tg - tn)
        o.set_pose(1, Qk, tk)
        o.map()
        co = o.fractions()[2]
        cg = g.fractions()[2]
        assert co.sum() > 0
        assert np.array_equal(co, cg), (case, k, int((co != cg).sum()))
    g.close()


ROD_GRID = (78, 36, 34)  # x periodic and ragged (78 = 2 x 32 + 14); y, z walls
ROD_CASES = {
    "band": {},
    "nocache": {"PSM_BAND_CACHE": "0"},
    "general": {"PSM_REMAP_GENERAL": "1"},
    "overflow": {"PSM_SEG_CAP": "6", "PSM_BAND_CAP": "10"},
}


@pytest.mark.parametrize("case", sorted(ROD_CASES))
def test_asymmetric_rod_reaches_its_seam_in_a_ragged_tile(case):
    """A rod reaching 36.5 cells along +x but only 10 along -x from its origin, on a periodic
    78-cell x axis: the ragged last tile [64, 78) holds the rod's +x end, while the tile's
    unclamped centre (x = 80) wraps to 37 cells on the -x side, 27 cells beyond the rod's short
    end — a whole-tile "all outside" there would skip solid cells.  The rod spins about x and
    drifts along x (closed-form advance in the library); counts bit-exact every step."""
    nx, ny, nz = ROD_GRID
    v, t = pi.box_mesh([-10.0, -2.5, -2.5], [36.5, 2.5, 2.5])
    Q0 = pi.rotation_about([1.0, 0.0, 0.0], 0.3)
    t0 = [39.13, 18.29, 17.41]
    vel = [0.04, 0.0, 0.0]
    w = np.array([0.03, 0.0, 0.0])
    o = oracle.Oracle(nx, ny, nz, 19, 0.9, (0, 1, 1), 1, 1)
    o.set_map_all_cells(True)
    o.set_mesh(1, v, t, 1)
    g = _sim(ROD_CASES[case], nx=nx, ny=ny, nz=nz, Q=19, tau=0.9, bc=(0, 1, 1), prec="f32")
    g.init_equilibrium()
    g.set_mesh(1, v, t, 1, Q0, t0, vel, w)
    for k in range(16):
        g.step(1)
        Qk, tk = oracle.pose_advance(Q0, t0, vel, w, k, list(ROD_GRID), [1, 0, 0])
        o.set_pose(1, Qk, tk)
        o.map()
        co = o.fractions()[2]
        cg = g.fractions()[2]
        assert co[:, :, 64:].sum() > 0  # solid in the ragged tile column
        assert np.array_equal(co, cg), (case, k, int((co != cg).sum()))
    g.close()


def test_seam_parity_fp64_pdfs_and_force():
    """Full step parity (PDFs <= 1e-12, F/T every step) for the seam body on the ragged grid:
    the collide's u_s and lever arm use the same minimum image as the remap."""
    nx, ny, nz = GRID
    Q0 = pi.rotation_about([0.3, -1.0, 0.5], 0.7)
    t0 = [66.3, 2.1, 36.7]
    v = [0.11, -0.07, 0.05]
    w = np.array([0.012, 0.02, -0.009])
    pose = _pose_fn(Q0, t0, v, w)
    mv, mt = _seam_propeller()
    rho, u = pi.perturbed_flow((nz, ny, nx), 41, u0=(0.02, 0.0, 0.01))
    o = oracle.Oracle(nx, ny, nz, 19, 0.7, (0, 0, 0), 1, 1)
    g = _sim(nx=nx, ny=ny, nz=nz, Q=19, tau=0.7, prec="f64")
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    o.set_mesh(1, mv, mt, 1)
    g.set_mesh(1, mv, mt, 1, Q0, t0, v, w)
    for k in range(20):
        Qk, tk = pose(k)
        o.set_pose(1, Qk, tk, v, w)
        o.map()
        o.step(1)
        g.step(1)
        Fg, Tg, _, _ = g.force_torque(1)
        Fo, To, aF, aT = o.force_torque(1)
        assert np.all(np.abs(Fg - Fo) <= 1e-10 * np.maximum(np.abs(Fo), aF) + 1e-300), k
        assert np.all(np.abs(Tg - To) <= 1e-10 * np.maximum(np.abs(To), aT) + 1e-300), k
    d = np.max(np.abs(o.pdfs() - g.pdfs()))
    assert d <= 1e-12, d
    g.close()
