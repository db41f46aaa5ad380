"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star, DESIGN.md §4 P15): fp64 max|df| <= 1e-12 after 100 steps;
force/torque |dF_a| <= 1e-10 * max(|F_a|, A_F,a) (A_F = sum |m| componentwise); fp32 vs the fp64
oracle <= 2e-5; fractions (count, id, B) bit-exact in both precisions.
"""
import numpy as np
import pytest

import oracle
import psm_inputs as pi

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12
F32_TOL = 2e-5
FT_REL = 1e-10


def _sim(**kw):
    import paper_2502_20049_b200 as psm
    return psm.Simulation(**kw)


def _ft_close(g, o, rel=FT_REL):
    Fg, Tg, aFg, aTg = g
    Fo, To, aFo, aTo = o
    okF = np.all(np.abs(Fg - Fo) <= rel * np.maximum(np.abs(Fo), aFo) + 1e-300)
    okT = np.all(np.abs(Tg - To) <= rel * np.maximum(np.abs(To), aTo) + 1e-300)
    return okF and okT, (Fg, Fo, Tg, To, aFo, aTo)


def _run_pair(nx, ny, nz, Q, tau, bc, sc, bmode, prec, pattern, bodies, steps, seed,
              u0=(0.05, 0.0, 0.0), ft_every=True, force=(0.0, 0.0, 0.0), collision="srt",
              magic=3.0 / 16.0, ft_rel=FT_REL, open_bc=None):
    """bodies: list of dicts (id, kind, r | mesh, s, pose(k) -> (Q, t), v, w).  Explicit poses
    are passed every step to both sides (reading A13)."""
    shape = (nz, ny, nx)
    rho, u = pi.perturbed_flow(shape, seed, u0=u0)
    o = oracle.Oracle(nx, ny, nz, Q, tau, bc, sc, bmode)
    o.set_force(force)
    o.set_collision(collision, magic)
    g = _sim(nx=nx, ny=ny, nz=nz, Q=Q, tau=tau, bc=bc, prec=prec, pattern=pattern, sc=sc,
             bmode=bmode, body_force=force, collision=collision, trt_magic=magic)
    if open_bc is not None:  # before the state is written (psm.h psm_set_open_boundary)
        o.set_open_boundary(*open_bc)
        g.set_open_boundary(*open_bc)
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    for b in bodies:
        Qp, tp = b["pose"](0)
        if b["kind"] == "sphere":
            o.set_sphere(b["id"], b["r"], b["s"])
            g.set_sphere(b["id"], b["r"], b["s"], Qp, tp, b.get("v", (0, 0, 0)),
                         b.get("w", (0, 0, 0)))
        else:
            o.set_mesh(b["id"], b["verts"], b["tris"], b["s"])
            o.set_mapping(b["id"], b.get("mapping", "R1"))
            g.set_mesh(b["id"], b["verts"], b["tris"], b["s"], Qp, tp, b.get("v", (0, 0, 0)),
                       b.get("w", (0, 0, 0)), mapping=b.get("mapping", "R1"))
        o.set_pose(b["id"], Qp, tp, b.get("v", (0, 0, 0)), b.get("w", (0, 0, 0)))
    worst_ft = 0.0
    for k in range(steps):
        for b in bodies:
            Qp, tp = b["pose"](k)
            o.set_pose(b["id"], Qp, tp, b.get("v", (0, 0, 0)), b.get("w", (0, 0, 0)))
            if k > 0:
                g.set_pose(b["id"], Qp, tp, b.get("v", (0, 0, 0)), b.get("w", (0, 0, 0)))
        o.map()
        if k == 0 or k == steps - 1:
            Bo, ido, co, _ = o.fractions()
            Bg, idg, cg = g.fractions()
            assert np.array_equal(co, cg), f"count mismatch at step {k}: {(co != cg).sum()} cells"
            assert np.array_equal(ido, idg)
            assert np.array_equal(Bo, Bg)
        o.step(1)
        g.step(1)
        if ft_every or k == steps - 1:
            for b in bodies:
                ok, info = _ft_close(g.force_torque(b["id"]), o.force_torque(b["id"]), ft_rel)
                assert ok, (k, info)
    return o, g


def _static(Q=np.eye(3), t=(16.0, 16.0, 16.0)):
    return lambda k: (Q, t)


@pytest.mark.parametrize("sc", [1, 2, 3])
@pytest.mark.parametrize("bmode", [0, 1])
def test_c1_stationary_sphere_fp64_100_steps(sc, bmode):
    """BASELINE config c1: D3Q19 fp64, 32^3 periodic, sphere r=6 at (16,16,16), tau=0.8, s=2."""
    c = pi.CONFIGS["c1"]
    o, g = _run_pair(32, 32, 32, 19, 0.8, (0, 0, 0), sc, bmode, "f64", "two_array",
                     [dict(id=1, kind="sphere", r=6.0, s=2, pose=_static())], 100, c["seed"])
    d = np.max(np.abs(o.pdfs() - g.pdfs()))
    assert d <= F64_TOL, d


@pytest.mark.parametrize("pattern", ["two_array", "aa"])
@pytest.mark.parametrize("Q", [19, 27])
def test_ragged_walls_rotating_mesh(pattern, Q):
    """Ragged grid (not a multiple of the 32x4x2 tile), y/z walls, a rotating + translating mesh
    body remapped every step: fp64 parity, fractions bit-exact, F/T every step."""
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.0, 0.0, 0.03])
    vv = np.array([0.02, 0.0, 0.0])
    Q0 = pi.rotation_about([1, 1, 0], 0.4)

    def pose(k):
        Qk, tk = oracle.pose_advance(Q0, [20.3, 10.6, 9.2], vv, w, k, [45, 21, 19], [1, 0, 0])
        return Qk, tk

    o, g = _run_pair(45, 21, 19, Q, 0.65, (0, 1, 1), 1, 1, "f64", pattern,
                     [dict(id=3, kind="mesh", verts=v, tris=tr, s=1, pose=pose, v=vv, w=w)], 40,
                     77, u0=(0.02, 0.01, 0.0))
    d = np.max(np.abs(o.pdfs() - g.pdfs()))
    assert d <= F64_TOL, d


def test_c2_translating_sphere_channel_fp64_and_fp32():
    """BASELINE config c2 geometry: 128x64x64, x periodic, y/z walls, sphere r=6 translating at
    v=(1/32,0,0), tau=0.575, SC2, weighted B; 100 steps (explicit dyadic poses)."""
    c = pi.CONFIGS["c2"]
    v = np.array(c["v"])
    body = dict(id=1, kind="sphere", r=6.0, s=2, v=v,
                pose=lambda k: (np.eye(3), tuple(np.array(c["t"]) + k * v)))
    o, g = _run_pair(128, 64, 64, 19, 0.575, (0, 1, 1), 2, 1, "f64", "two_array", [body], 100,
                     c["seed"], u0=(0.0, 0.0, 0.0), ft_every=False)
    ref = o.pdfs()
    d = np.max(np.abs(ref - g.pdfs()))
    assert d <= F64_TOL, d
    # fp32 variant of the same run: <= 2e-5 against the fp64 oracle, fractions bit-exact
    g32 = _sim(nx=128, ny=64, nz=64, Q=19, tau=0.575, bc=(0, 1, 1), prec="f32", sc=2, bmode=1)
    rho, u = pi.perturbed_flow((64, 64, 128), c["seed"], u0=(0.0, 0.0, 0.0))
    g32.init_equilibrium(rho, u)
    g32.set_sphere(1, 6.0, 2, np.eye(3), c["t"], v)
    for k in range(100):
        if k > 0:
            g32.set_pose(1, np.eye(3), tuple(np.array(c["t"]) + k * v), v)
        g32.step(1)
    d32 = np.max(np.abs(ref - g32.pdfs()))
    assert d32 <= F32_TOL, d32
    Bo, ido, co, _ = o.fractions()
    assert np.array_equal(g32.fractions()[2], co)


def test_internal_pose_advance_matches_explicit_poses():
    """psm_step(n) advancing a translating body itself (dyadic velocity: exact poses) gives the
    same state and fractions as feeding the poses explicitly."""
    c = pi.CONFIGS["c2"]
    v = np.array(c["v"])
    a = _sim(nx=128, ny=64, nz=64, Q=19, tau=0.575, bc=(0, 1, 1), sc=2, bmode=1)
    b = _sim(nx=128, ny=64, nz=64, Q=19, tau=0.575, bc=(0, 1, 1), sc=2, bmode=1)
    for s in (a, b):
        s.init_equilibrium()
        s.set_sphere(1, 6.0, 2, np.eye(3), c["t"], v)
    a.step(40)
    for k in range(40):
        if k > 0:
            b.set_pose(1, np.eye(3), tuple(np.array(c["t"]) + k * v), v)
        b.step(1)
    assert np.array_equal(a.pdfs(), b.pdfs())
    assert a.step_count == 40
    fa, fb = a.force_torque(1), b.force_torque(1)
    assert np.array_equal(fa[0], fb[0])


@pytest.mark.parametrize("Q", [19, 27])
def test_two_array_and_aa_give_the_same_state(Q):
    v, tr = pi.propeller_mesh(n_blades=4, scale=0.08, n_st=8, n_pts=16, hub_seg=16)
    w = (0.02, -0.01, 0.0)
    runs = []
    for pattern in ("two_array", "aa"):
        s = _sim(nx=48, ny=40, nz=36, Q=Q, tau=0.7, bc=(0, 0, 0), pattern=pattern, sc=1)
        rho, u = pi.perturbed_flow((36, 40, 48), 5)
        s.init_equilibrium(rho, u)
        s.set_mesh(2, v, tr, 1, np.eye(3), (24.0, 20.0, 18.0), (0.01, 0, 0), w)
        for n in (1, 6, 10):  # odd and even step counts
            s.step(n)
        runs.append((s.pdfs(), s.force_torque(2)))
    d = np.max(np.abs(runs[0][0] - runs[1][0]))
    assert d <= 1e-15, d
    assert np.allclose(runs[0][1][0], runs[1][1][0], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("sc", [1, 2, 3])
def test_debug_fields_random_B(sc):
    """Random B in [0,1] and u_s through psm_debug_set_fields (P4 on the GPU)."""
    shape = (11, 9, 37)
    n = int(np.prod(shape))
    rho, u = pi.perturbed_flow(shape, 21)
    B = pi.random_unit(22, n).reshape(shape)
    B[B < 0.3] = 0.0
    us = 0.05 * pi.uniform_pm1(23, 3 * n).reshape((3,) + shape)
    bid = np.where(B > 0, 1 + (np.arange(n).reshape(shape) % 3), 0).astype(np.uint8)
    o = oracle.Oracle(37, 9, 11, 19, 0.9, (0, 0, 0), sc, 1)
    g = _sim(nx=37, ny=9, nz=11, Q=19, tau=0.9, sc=sc, bmode=1)
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    o.set_fields(B, us, bid)
    g.debug_set_fields(B, us, bid)
    for _ in range(5):
        o.step(1)
        g.step(1)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL
    for b in (1, 2, 3):
        ok, info = _ft_close(g.force_torque(b), o.force_torque(b))
        assert ok, info


def test_body_force_with_sphere_and_walls():
    g0 = (2e-5, 1e-6, 0.0)
    body = dict(id=1, kind="sphere", r=4.0, s=1, pose=_static(t=(12.0, 10.0, 8.0)))
    o, g = _run_pair(24, 20, 16, 19, 0.8, (0, 1, 0), 2, 1, "f64", "two_array", [body], 60, 9,
                     u0=(0.0, 0.0, 0.0), force=g0)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


def test_error_word_reports_invalid_state():
    import paper_2502_20049_b200 as psm
    s = _sim(nx=32, ny=8, nz=8)
    f = np.broadcast_to(oracle.stencil(19)[1][:, None, None, None], (19, 8, 8, 32)).copy()
    f[:, 3, 2, 5] = -1.0  # rho < 0 at cell (5, 2, 3)
    s.write_pdfs(f)
    with pytest.raises(psm.PSMError) as e:
        s.step(1)
    assert e.value.code == psm.PSM_E_STATE
    assert "(5,2,3)" in str(e.value)


def test_write_read_roundtrip_and_equilibrium():
    s = _sim(nx=35, ny=6, nz=5, bc=(0, 1, 1), Q=27)
    f = pi.random_pdfs(27, (5, 6, 35), 3, w=oracle.stencil(27)[1])
    s.write_pdfs(f)
    assert np.array_equal(s.pdfs(), f)
    rho, u = pi.perturbed_flow((5, 6, 35), 4)
    s.init_equilibrium(rho, u)
    r2, u2 = s.velocity()
    assert np.allclose(r2, rho, atol=1e-14) and np.allclose(u2, u, atol=1e-14)


@pytest.mark.parametrize("mapping", ["R1", "R2"])
@pytest.mark.parametrize("s", [1, 2, 3])
def test_mesh_band_pass_exact_on_geometry_cell_faces(s, mapping):
    """The mesh band pass (k_remap_l3_mesh) transforms one sub-sample per 8 in fp64 and the
    others in fp32, falling back to the exact per-sample arithmetic within 1e-5 of a
    geometry-cell face.  Poses that put every sub-sample exactly on a face (identity rotation,
    t offset by half a sub-sample spacing), within ~1e-4 of one (a 3e-6 rad rotation) and a
    generic pose: counts bit-exact against the oracle's per-sample A14 arithmetic (reading R1).
    R2 (reading A12): the centre-only block count, by per-brick popcount masks in the library
    (r2_block_count) and cell by cell in the oracle; the identity pose puts every block exactly on
    one brick, the others make blocks straddle up to 2 x 2 x 2 bricks."""
    import psm_inputs.meshgen as mg
    n = 48
    h = 0.5 ** s
    meshes = [pi.box_mesh([-9.0, -7.0, -8.0], [8.0, 9.0, 7.0]), mg.uv_sphere_mesh(12.3, 24, 16),
              pi.propeller_mesh(n_blades=4, scale=0.16, n_st=10, n_pts=16, hub_seg=24)]
    c = np.array([24.0, 23.0, 25.0]) + h / 2
    poses = [(np.eye(3), c), (pi.rotation_about([1.0, -2.0, 0.5], 3e-6), c),
             (pi.rotation_about([0.3, 1.0, -0.7], 0.61), c + [0.17, -0.29, 0.05])]
    g = _sim(nx=n, ny=n, nz=n, Q=19, tau=0.8, prec="f32")
    for v, tr in meshes:
        o = oracle.Oracle(n, n, n, 19, 0.8, (0, 0, 0), 1, 1)
        o.set_mesh(1, v, tr, s)
        o.set_mapping(1, mapping)
        for k, (Q, t) in enumerate(poses):
            if k == 0:
                g.set_mesh(1, v, tr, s, Q, t, mapping=mapping)
            else:
                g.set_pose(1, Q, t)
            o.set_pose(1, Q, t)
            o.map()
            co = o.fractions()[2]
            cg = g.fractions()[2]
            assert co.sum() > 0
            assert np.array_equal(co, cg), (s, k, int((co != cg).sum()))
        g.remove_body(1)
    g.close()


@pytest.mark.parametrize("s", [1, 2])
def test_cror_rotor_fractions_bit_exact_large(s):
    """A 12-blade rotor (tip 55 cells, coarse CROR recipe) rotating about x in a 128^3 box: the
    remap's tile-level (18-brick reach) and cell-level early-outs must reproduce the oracle's
    brute-force counts bit for bit at several poses; then 3 coupled steps."""
    v, tr = pi.propeller_mesh(n_blades=12, scale=55.0 / 110.0, n_st=16, n_pts=24, hub_seg=32)
    n = 128
    w = (0.004, 0.0, 0.0)
    o = oracle.Oracle(n, n, n, 19, 0.6, (0, 0, 0), 1, 1)
    g = _sim(nx=n, ny=n, nz=n, Q=19, tau=0.6, prec="f32", sc=1, bmode=1)
    o.set_mesh(1, v, tr, s)
    rho, u = pi.perturbed_flow((n, n, n), 3, u0=(0.02, 0, 0), u_amp=0.001)
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    t = (60.3, 64.0, 63.7)
    for k, ang in enumerate((0.0, 0.37, 1.1 - 0.004)):
        Q = pi.rotation_about([1, 0, 0], ang) @ pi.rotation_about([0.2, 1, 0], 0.05)
        o.set_pose(1, Q, t, (0, 0, 0), w)
        o.map()
        if k == 0:
            g.set_mesh(1, v, tr, s, Q, t, (0, 0, 0), w)
        else:
            g.set_pose(1, Q, t, (0, 0, 0), w)
        Bo, ido, co, _ = o.fractions()
        Bg, idg, cg = g.fractions()
        assert np.array_equal(co, cg), (k, int((co != cg).sum()))
        assert np.array_equal(Bo, Bg)
        assert co.sum() > 1000
    for k in range(3):  # explicit poses on both sides (A13); k = 0 is the last checked pose
        if k > 0:
            Q = (pi.rotation_about([1, 0, 0], 1.1 - 0.004 + 0.004 * k)
                 @ pi.rotation_about([0.2, 1, 0], 0.05))
            o.set_pose(1, Q, t, (0, 0, 0), w)
            o.map()
            g.set_pose(1, Q, t, (0, 0, 0), w)
        o.step(1)
        g.step(1)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F32_TOL
    ok, info = _ft_close(g.force_torque(1), o.force_torque(1), rel=1e-4)
    assert ok, info


def test_two_bodies_with_overlapping_boxes():
    """Two bodies whose remap boxes overlap (a sphere passing next to a rotating mesh): those
    boxes go through the general multi-body remap kernel; max-eps / lower-id rule (A18)."""
    v, tr = pi.propeller_mesh(n_blades=4, scale=0.09, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.0, 0.03, 0.0])

    def pose_mesh(k):
        return oracle.pose_advance(np.eye(3), [24.0, 20.0, 18.2], [0, 0, 0], w, k,
                                   [48, 40, 36], [1, 1, 1])

    vs = np.array([0.0, 0.0, 1.0 / 16])
    bodies = [dict(id=2, kind="mesh", verts=v, tris=tr, s=1, pose=pose_mesh, w=w),
              dict(id=5, kind="sphere", r=4.0, s=2, v=vs,
                   pose=lambda k: (np.eye(3), tuple(np.array([24.0, 20.0, 28.0]) + k * vs)))]
    o, g = _run_pair(48, 40, 36, 19, 0.7, (0, 0, 0), 3, 1, "f64", "two_array", bodies, 24, 13,
                     u0=(0.02, 0.0, 0.0))
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


@pytest.mark.parametrize("pattern,Q,sc", [("two_array", 19, 1), ("aa", 27, 3),
                                          ("two_array", 27, 2)])
def test_trt_psm_rotating_mesh(pattern, Q, sc):
    """TRT fluid operator (NEXT rank 2) inside the PSM update with a rotating mesh and walls."""
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.025, 0.0, 0.0])

    def pose(k):
        return oracle.pose_advance(np.eye(3), [20.0, 11.0, 9.5], [0, 0, 0], w, k, [40, 22, 19],
                                   [1, 0, 0])

    o, g = _run_pair(40, 22, 19, Q, 0.62, (0, 1, 1), sc, 1, "f64", pattern,
                     [dict(id=1, kind="mesh", verts=v, tris=tr, s=1, pose=pose, w=w)], 30, 17,
                     u0=(0.02, 0.0, 0.01), collision="trt", magic=0.1)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


def test_trt_forced_channel_with_sphere():
    body = dict(id=1, kind="sphere", r=3.5, s=1, pose=_static(t=(10.0, 8.0, 6.0)))
    o, g = _run_pair(20, 16, 12, 19, 0.7, (0, 1, 0), 1, 1, "f64", "two_array", [body], 40, 3,
                     u0=(0.0, 0.0, 0.0), force=(1e-5, 0.0, 2e-6), collision="trt")
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


@pytest.mark.parametrize("world_bc", [(0, 0, 0), (0, 1, 1)])
def test_two_way_coupled_bodies(world_bc):
    """NEXT rank 1: dynamic bodies driven by their own Eq.(10)-(11) force/torque every step
    (semi-implicit Euler on the host), vs the oracle's independent integrator."""
    n = (40, 36, 32)
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    o = oracle.Oracle(*n, 19, 0.7, world_bc, 1, 1)
    g = _sim(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.7, bc=world_bc, sc=1, bmode=1)
    rho, u = pi.perturbed_flow(n[::-1], 29, u0=(0.02, 0.0, 0.0))
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    I_mesh = np.array([[900.0, 20.0, 0.0], [20.0, 700.0, 5.0], [0.0, 5.0, 800.0]])
    o.set_sphere(1, 4.0, 1)
    o.set_pose(1, np.eye(3), (12.0, 18.0, 16.0), (0.0, 0.0, 0.01), (0, 0, 0))
    o.set_dynamics(1, 2500.0, np.eye(3) * 16000.0, (0.0, -0.5, 0.0))
    g.set_sphere(1, 4.0, 1, np.eye(3), (12.0, 18.0, 16.0), (0.0, 0.0, 0.01), (0, 0, 0))
    g.set_dynamics(1, 2500.0, np.eye(3) * 16000.0, (0.0, -0.5, 0.0))
    Q0 = pi.rotation_about([1, 0, 1], 0.3)
    o.set_mesh(2, v, tr, 1)
    o.set_pose(2, Q0, (28.0, 18.0, 16.0), (0, 0, 0), (0.0, 0.02, 0.0))
    o.set_dynamics(2, 3000.0, I_mesh, (0, 0, 0), (0.0, 0.0, 0.3))
    g.set_mesh(2, v, tr, 1, Q0, (28.0, 18.0, 16.0), (0, 0, 0), (0.0, 0.02, 0.0))
    g.set_dynamics(2, 3000.0, I_mesh, (0, 0, 0), (0.0, 0.0, 0.3))
    for k in range(30):
        o.map()
        o.step(1)
        o.integrate()
        g.step(1)
        for b in (1, 2):
            so, sg = o.body_state(b), g.body_state(b)
            for a, c in zip(so, sg):
                assert np.allclose(a, c, rtol=1e-11, atol=1e-14), (k, b, a, c)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL
    assert not np.allclose(g.body_state(1)[2], (0.0, 0.0, 0.01))  # it really was coupled


def test_dynamic_body_back_to_prescribed_motion_with_remap_ahead():
    """psm_set_dynamics(id, NULL) after coupled steps: the body continues in closed form from its
    integrated state, the remap-ahead spare buffer (which followed the dynamic pose) is rebuilt,
    and a pipelined psm_step(n) equals the oracle fed the closed-form poses from that state
    (fractions bit-exact, PDFs <= 1e-12, F/T of the last step)."""
    n = (40, 36, 32)
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    I_mesh = np.array([[900.0, 20.0, 0.0], [20.0, 700.0, 5.0], [0.0, 5.0, 800.0]])
    Q0 = pi.rotation_about([1, 0, 1], 0.3)
    t0 = (20.0, 18.0, 16.0)
    o = oracle.Oracle(*n, 19, 0.7, (0, 0, 0), 1, 1)
    g = _sim(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.7, sc=1, bmode=1)
    rho, u = pi.perturbed_flow(n[::-1], 31, u0=(0.02, 0.0, 0.0))
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    v0, w0 = (0.01, 0.0, 0.0), (0.0, 0.02, 0.0)
    o.set_mesh(2, v, tr, 1)
    g.set_mesh(2, v, tr, 1, Q0, t0, v0, w0)
    # prescribed phase in one pipelined call: the spare word buffer is in use
    g.step(5)
    for k in range(5):
        Qk, tk = oracle.pose_advance(Q0, t0, v0, w0, k, list(n), [1, 1, 1])
        o.set_pose(2, Qk, tk, v0, w0)
        o.map()
        o.step(1)
    Q5, t5 = oracle.pose_advance(Q0, t0, v0, w0, 5, list(n), [1, 1, 1])
    o.set_pose(2, Q5, t5, v0, w0)
    o.set_dynamics(2, 3000.0, I_mesh, (0.5, 0.0, 0.0), (0.0, 0.0, 0.3))
    g.set_dynamics(2, 3000.0, I_mesh, (0.5, 0.0, 0.0), (0.0, 0.0, 0.3))
    for _ in range(4):
        o.map()
        o.step(1)
        o.integrate()
        g.step(1)
    g.set_dynamics(2, None)  # back to prescribed motion from the integrated state
    Qs, ts, vs, ws = g.body_state(2)
    so = o.body_state(2)
    for a, c in zip(so, (Qs, ts, vs, ws)):
        assert np.allclose(a, c, rtol=1e-11, atol=1e-14)
    g.step(9)  # remap-ahead pipeline over the prescribed phase
    for k in range(9):
        Qk, tk = oracle.pose_advance(Qs, ts, vs, ws, k, list(n), [1, 1, 1])
        o.set_pose(2, Qk, tk, vs, ws)
        o.map()
        o.step(1)
    assert np.array_equal(o.fractions()[2], g.fractions()[2])
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL
    ok, info = _ft_close(g.force_torque(2), o.force_torque(2), 1e-9)
    assert ok, info


def test_neighbouring_bodies_sharing_tiles_keep_their_fractions():
    """Regression: two bodies whose cell boxes are disjoint but share 32x4x2 tiles; remapping
    one (single-body fast path) must not clear the other's words."""
    n = (64, 24, 24)
    o = oracle.Oracle(*n, 19, 0.7, (0, 0, 0), 1, 1)
    g = _sim(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.7, sc=1, bmode=1)
    g.init_equilibrium()
    for sim in (g,):
        sim.set_sphere(1, 3.0, 2, np.eye(3), (6.0, 12.0, 12.0))
        sim.set_sphere(2, 3.0, 2, np.eye(3), (20.0, 12.0, 12.0), (1 / 32, 0, 0))
    o.set_sphere(1, 3.0, 2)
    o.set_sphere(2, 3.0, 2)
    for k in range(5):
        o.set_pose(1, np.eye(3), (6.0, 12.0, 12.0))
        o.set_pose(2, np.eye(3), (20.0 + k / 32, 12.0, 12.0), (1 / 32, 0, 0))
        o.map()
        if k:
            g.step(1)       # collides step k-1, then the body sits at pose k
            g.map_fractions()  # fractions at the current pose
        assert np.array_equal(o.fractions()[2], g.fractions()[2]), k
        assert np.array_equal(o.fractions()[1], g.fractions()[1]), k


@pytest.mark.parametrize("s", [1, 2])
def test_r2_centre_only_mapping_rotating_mesh(s):
    """NEXT rank 3: the paper-literal centre-only mapping (R2) on a rotating mesh, both remap
    paths (single-body pipeline and, with a second body sharing tiles, the general kernel)."""
    v, tr = pi.propeller_mesh(n_blades=4, scale=0.09, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.0, 0.03, 0.01])

    def pose(k):
        return oracle.pose_advance(pi.rotation_about([1, 0, 0], 0.2), [20.3, 18.0, 17.6],
                                   [0, 0, 0], w, k, [48, 36, 34], [1, 1, 1])

    bodies = [dict(id=1, kind="mesh", verts=v, tris=tr, s=s, pose=pose, w=w, mapping="R2"),
              dict(id=2, kind="sphere", r=3.0, s=1, pose=_static(t=(36.0, 18.0, 17.0)))]
    o, g = _run_pair(48, 36, 34, 19, 0.7, (0, 0, 0), 1, 1, "f64", "two_array", bodies, 25, 8,
                     u0=(0.02, 0.0, 0.0))
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("pattern,bc,prec", [("two_array", (0, 0, 0), "f64"),
                                             ("aa", (0, 1, 1), "f64"),
                                             ("aa", (0, 0, 0), "f64"),
                                             ("two_array", (0, 1, 0), "f32"),
                                             ("aa", (0, 0, 1), "f32")])
def test_cumulant_psm_rotating_mesh(pattern, bc, prec, Q):
    """Cumulant fluid operator (the paper's performance operator) inside the PSM
    update: D3Q27 (A29, kernel factorised back-transform) and D3Q19 (A32, kernel closed-form
    raw-moment inverse) against the oracle's moment solve (27x27 / 19x19).  D3Q19 + AA +
    periodic + fp64 + SC1 + rotation is the paper's own performance configuration."""
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.025, 0.0, 0.0])

    def pose(k):
        return oracle.pose_advance(np.eye(3), [20.0, 11.0, 9.5], [0, 0, 0], w, k, [40, 22, 19],
                                   [1, 1, 1])

    o, g = _run_pair(40, 22, 19, Q, 0.62, bc, 1, 1, prec, pattern,
                     [dict(id=1, kind="mesh", verts=v, tris=tr, s=1, pose=pose, w=w)], 30, 19,
                     u0=(0.03, 0.0, 0.01), collision="cumulant", ft_every=(prec == "f64"),
                     ft_rel=FT_REL if prec == "f64" else 1e-4)  # fp32: ~30 steps of 1e-7 drift
    tol = F64_TOL if prec == "f64" else F32_TOL
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= tol


# ---- open boundaries (reading A30): velocity inflow at x = 0, pressure outflow at x = nx-1 ----
OPEN = ((0.05, 0.01, -0.005), 1.002)


@pytest.mark.parametrize("sc", [1, 2])
def test_open_channel_moving_sphere_fp64(sc):
    """Channel with inflow/outflow on x, no-slip walls on y (domain edges: x faces win), periodic
    z; a sphere crosses the channel; D3Q19 fp64, 100 steps, F/T every step."""
    o, g = _run_pair(48, 20, 18, 19, 0.7, (2, 1, 0), sc, 1, "f64", "two_array",
                     [dict(id=1, kind="sphere", r=5.0, s=1, v=(0.02, 0.0, 0.0),
                           pose=lambda k: (np.eye(3), (14.0 + 0.02 * k, 10.3, 9.1)))],
                     100, 31, u0=(0.05, 0.0, 0.0), open_bc=OPEN)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


@pytest.mark.parametrize("collision,Q", [("trt", 19), ("cumulant", 27), ("srt", 27),
                                         ("cumulant", 19)])
def test_open_channel_rotating_mesh_operators(collision, Q):
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.07, n_st=8, n_pts=16, hub_seg=16)
    w = np.array([0.025, 0.0, 0.0])

    def pose(k):
        return oracle.pose_advance(np.eye(3), [20.0, 11.0, 9.5], [0, 0, 0], w, k, [40, 22, 19],
                                   [0, 1, 0])

    o, g = _run_pair(40, 22, 19, Q, 0.62, (2, 1, 1), 1, 1, "f64", "two_array",
                     [dict(id=1, kind="mesh", verts=v, tris=tr, s=1, pose=pose, w=w)], 30, 23,
                     u0=(0.04, 0.0, 0.0), collision=collision, open_bc=OPEN)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


def test_open_channel_fp32():
    o, g = _run_pair(64, 16, 12, 19, 0.6, (2, 1, 0), 1, 1, "f32", "two_array",
                     [dict(id=1, kind="sphere", r=4.0, s=2,
                           pose=lambda k: (np.eye(3), (20.0, 8.0, 6.0)))],
                     60, 37, u0=(0.05, 0.0, 0.0), ft_every=False, ft_rel=1e-4,
                     open_bc=((0.05, 0.0, 0.0), 1.0))
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F32_TOL


def test_open_state_roundtrip():
    """write_pdfs inverts the face rules (A30) exactly: reading back gives the state written."""
    for Q in (19, 27):
        s = _sim(nx=9, ny=6, nz=5, bc=(2, 1, 0), Q=Q)
        s.set_open_boundary((0.03, -0.01, 0.02), 0.98)
        f = pi.random_pdfs(Q, (5, 6, 9), 5, w=oracle.stencil(Q)[1])
        s.write_pdfs(f)
        assert np.max(np.abs(s.pdfs() - f)) <= 1e-15


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_open_x_only_periodic_yz(prec):
    """Open x faces with periodic y, z: the launcher's x-only wall variant."""
    o, g = _run_pair(40, 12, 12, 19, 0.65, (2, 0, 0), 1, 1, prec, "two_array",
                     [dict(id=1, kind="sphere", r=3.5, s=1, v=(0.0, 0.01, 0.0),
                           pose=lambda k: (np.eye(3), (20.0, 3.0 + 0.01 * k, 6.0)))],
                     40, 41, u0=(0.05, 0.0, 0.0), ft_every=(prec == "f64"),
                     ft_rel=FT_REL if prec == "f64" else 1e-4, open_bc=OPEN)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= (F64_TOL if prec == "f64" else F32_TOL)


def test_remap_ahead_pipeline_equals_stepwise():
    """psm_step(n > 1) remaps step k+1 into the spare word buffer while step k collides; the
    result must be bitwise the same as n calls of psm_step(1) (no pipeline), including after
    body changes that invalidate the spare buffer (set_body, remove_body) and a body crossing
    the periodic boundary."""
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.09, n_st=8, n_pts=16, hub_seg=16)
    kw = dict(nx=64, ny=40, nz=36, Q=19, tau=0.62, prec="f64", sc=1, bmode=1)
    rho, u = pi.perturbed_flow((36, 40, 64), 61, u0=(0.03, 0.0, 0.01))
    sims = [_sim(**kw), _sim(**kw)]
    for s in sims:
        s.init_equilibrium(rho, u)
        s.set_mesh(1, v, tr, 1, pi.rotation_about([0, 1, 1], 0.3), (20.0, 20.0, 18.0),
                   (0.02, 0.0, 0.0), (0.03, 0.0, 0.01))
        s.set_sphere(2, 4.5, 2, np.eye(3), (50.0, 20.0, 1.0), (0.0, 0.05, -0.1))
    a, b = sims

    def run(n):
        a.step(n)
        for _ in range(n):
            b.step(1)
        assert np.array_equal(a.pdfs(), b.pdfs())
        for i in range(3):
            assert np.array_equal(a.fractions()[i], b.fractions()[i])
        for bid in (1, 2):
            if bid in present:
                for x, y in zip(a.force_torque(bid), b.force_torque(bid)):
                    assert np.array_equal(x, y)

    present = {1, 2}
    run(7)
    for s in sims:  # new pose/velocity of the sphere: the spare buffer is stale
        s.set_sphere(2, 4.5, 2, np.eye(3), (40.0, 30.0, 30.0), (0.1, 0.0, 0.0))
    run(5)
    for s in sims:
        s.remove_body(1)
    present = {2}
    run(4)
    for s in sims:
        s.set_mesh(3, v, tr, 1, np.eye(3), (15.0, 15.0, 15.0), (0.0, 0.0, 0.0), (0.0, 0.02, 0.0))
    present = {2, 3}
    run(6)


@pytest.mark.parametrize("s", [0, 1, 2, 3])
def test_gpu_voxelizer_equals_host_bricks_and_flags(s, monkeypatch):
    """The GPU voxeliser (k_voxelize.cu, default in psm_set_body) and the host implementation of
    reading A15 produce identical brick words and early-out flags (PSM_VOXELIZE_CHECK compares
    them inside the library), for a cube, a UV sphere, a propeller and the large CROR rotor."""
    import time
    import psm_inputs.meshgen as mg
    monkeypatch.setenv("PSM_VOXELIZE_CHECK", "1")
    meshes = [pi.box_mesh([-5.3, -4.1, -6.2], [5.7, 4.9, 3.3]),
              mg.uv_sphere_mesh(7.3, 24, 16),
              pi.propeller_mesh(n_blades=5, scale=0.15, n_st=12, n_pts=16, hub_seg=24)]
    g = _sim(nx=64, ny=64, nz=64, Q=19, prec="f32")
    for k, (v, tr) in enumerate(meshes):
        g.set_mesh(1, v, tr, s, pi.rotation_about([1, 2, 3], 0.4), (32.0, 31.0, 30.5))
        g.remove_body(1)
    g.close()
    if s <= 2:  # the ~0.6 M-face rotor (tip radius 200 cells) in a grid that holds it
        v, tr = pi.cror_rotor(True)
        g = _sim(nx=448, ny=448, nz=448, Q=19, prec="f32")
        t0 = time.perf_counter()
        g.set_mesh(1, v, tr, s, np.eye(3), (224.0, 224.0, 224.0))
        print(f"CROR rotor s={s}: GPU + host voxelisation and compare {time.perf_counter() - t0:.2f} s")
        g.close()


def test_gpu_voxelizer_speed_large_rotor(monkeypatch):
    """Setup cost of the ~0.6 M-face rotor at s = 3 (7.7e9 geometry cells): GPU vs host."""
    import time
    v, tr = pi.cror_rotor(True)
    g = _sim(nx=448, ny=448, nz=448, Q=19, prec="f32")
    t0 = time.perf_counter()
    g.set_mesh(1, v, tr, 3, np.eye(3), (224.0, 224.0, 224.0))
    t_gpu = time.perf_counter() - t0
    _, _, cnt_gpu = g.fractions()
    g.remove_body(1)
    monkeypatch.setenv("PSM_VOXELIZE", "host")
    t0 = time.perf_counter()
    g.set_mesh(1, v, tr, 3, np.eye(3), (224.0, 224.0, 224.0))
    t_host = time.perf_counter() - t0
    _, _, cnt_host = g.fractions()
    print(f"set_mesh s=3, {len(tr)} faces: GPU voxeliser {t_gpu:.2f} s, host {t_host:.2f} s")
    assert np.array_equal(cnt_gpu, cnt_host)
    g.close()


def test_two_way_coupled_light_body_with_virtual_mass():
    """A light body (density ratio 1.1) with the virtual-mass stabilisation (psm.h
    psm_dynamics.added_mass / added_inertia, A28), closed box, SC2: library integrator vs the
    oracle's, body states <= 1e-11 relative, PDFs <= 1e-12 over 60 coupled steps."""
    n, r, ratio, gz = (28, 26, 30), 4.0, 1.1, 2e-4
    o = oracle.Oracle(*n, 19, 0.8, (1, 1, 1), 2, 1)
    g = _sim(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.8, bc=(1, 1, 1), sc=2, bmode=1)
    rho, u = pi.perturbed_flow(n[::-1], 31, u0=(0.0, 0.0, 0.0))
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    V = 4.0 / 3.0 * np.pi * r ** 3
    m = ratio * V
    I = 0.4 * m * r * r * np.eye(3)
    kw = dict(added_mass=V, added_inertia=I / ratio)
    o.set_sphere(1, r, 1)
    o.set_pose(1, np.eye(3), (14.2, 13.1, 17.4), (0, 0, 0), (0, 0, 0.001))
    o.set_dynamics(1, m, I, (0.0, 0.0, -(m - V) * gz), **kw)
    g.set_sphere(1, r, 1, np.eye(3), (14.2, 13.1, 17.4), (0, 0, 0), (0, 0, 0.001))
    g.set_dynamics(1, m, I, (0.0, 0.0, -(m - V) * gz), **kw)
    for k in range(60):
        o.map()
        o.step(1)
        o.integrate()
        g.step(1)
        so, sg = o.body_state(1), g.body_state(1)
        for a, c in zip(so, sg):
            assert np.allclose(a, c, rtol=1e-11, atol=1e-14), (k, a, c)
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL
    assert g.body_state(1)[2][2] < 0  # sinking


@pytest.mark.parametrize("Q", [19, 27])
def test_cumulant_with_body_force(Q):
    """Cumulant operator with a Guo-type body force (reading A31) in a walled channel with a
    moving sphere: fp64 <= 1e-12 and F/T every step against the oracle."""
    o, g = _run_pair(36, 20, 18, Q, 0.7, (0, 1, 0), 2, 1, "f64", "two_array",
                     [dict(id=1, kind="sphere", r=4.5, s=1, v=(0.02, 0.0, 0.0),
                           pose=lambda k: (np.eye(3), (12.0 + 0.02 * k, 10.3, 9.1)))],
                     40, 47, u0=(0.02, 0.0, 0.0), force=(2e-5, 0.0, 1e-5),
                     collision="cumulant")
    assert np.max(np.abs(o.pdfs() - g.pdfs())) <= F64_TOL


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_degenerate_one_cell_thick_grids(prec):
    """Edge case: extents of 1 (the periodic neighbour of a cell is itself) and a ragged y/z:
    a forced 1 x 37 x 1 channel between walls, and a 1 x 1 x 1 periodic box, against the oracle."""
    tol = F64_TOL if prec == "f64" else F32_TOL
    for (nx, ny, nz, bc) in [(1, 37, 1, (0, 1, 0)), (1, 1, 1, (0, 0, 0)), (3, 5, 2, (0, 0, 1))]:
        rho, u = pi.perturbed_flow((nz, ny, nx), 91, u0=(0.01, 0.0, 0.0))
        o = oracle.Oracle(nx, ny, nz, 19, 0.8, bc, 1, 1)
        o.set_force((1e-5, 0.0, 0.0))
        g = _sim(nx=nx, ny=ny, nz=nz, Q=19, tau=0.8, bc=bc, prec=prec, sc=1, bmode=1,
                 body_force=(1e-5, 0.0, 0.0))
        o.init_equilibrium(rho, u)
        g.init_equilibrium(rho, u)
        o.step(50)
        g.step(50)
        assert np.max(np.abs(o.pdfs() - g.pdfs())) <= tol, (nx, ny, nz, bc)


@pytest.mark.parametrize("sc", [1, 2, 3])
def test_paper_configuration_d3q19_cumulant_aa_rotating_100_steps(sc):
    """The paper's performance configuration: D3Q19, cumulant (A32), AA
    in-place streaming, fp64, prescribed rotation of a triangle-mesh propeller, 100 steps,
    fully periodic, with the library advancing the pose itself (psm_step(n) in chunks, so the
    remap-ahead pipeline and the cached band run too) against the oracle fed
    oracle.pose_advance poses: PDFs <= 1e-12, counts bit-exact, F/T of the last step."""
    import paper_2502_20049_b200 as psm
    nx, ny, nz = 44, 38, 36
    v, tr = pi.propeller_mesh(n_blades=4, scale=0.13, n_st=10, n_pts=16, hub_seg=16)
    w = np.array([0.02, 0.0, 0.0])
    t0 = [21.3, 19.1, 17.7]
    rho, u = pi.perturbed_flow((nz, ny, nx), 53, u0=(0.03, 0.0, 0.0))
    o = oracle.Oracle(nx, ny, nz, 19, 0.55, (0, 0, 0), sc, 1)
    o.set_collision("cumulant")
    g = psm.Simulation(nx, ny, nz, Q=19, tau=0.55, prec="f64", pattern="aa", sc=sc, bmode=1,
                       collision="cumulant")
    o.init_equilibrium(rho, u)
    g.init_equilibrium(rho, u)
    o.set_mesh(1, v, tr, 1)
    g.set_mesh(1, v, tr, 1, np.eye(3), t0, (0, 0, 0), w)
    for k in range(100):
        Qk, tk = oracle.pose_advance(np.eye(3), t0, (0, 0, 0), w, k, [nx, ny, nz], [1, 1, 1])
        o.set_pose(1, Qk, tk, (0, 0, 0), w)
        o.map()
        o.step(1)
    for n in (1, 7, 25, 33, 34):  # odd and even AA step counts, pipelined calls
        g.step(n)
    assert g.step_count == 100
    assert np.array_equal(o.fractions()[2], g.fractions()[2])
    d = np.max(np.abs(o.pdfs() - g.pdfs()))
    assert d <= F64_TOL, d
    ok, info = _ft_close(g.force_torque(1), o.force_torque(1))
    assert ok, info


@pytest.mark.parametrize("pattern,collision", [("two_array", "srt"), ("aa", "cumulant")])
def test_fp64_occupancy_variants_bitwise_identical(pattern, collision):
    """The fp64 D3Q19 collide exists at two occupancies (chosen at run time from the PSM-tile
    fraction): both give the same bits, and equal the oracle."""
    import os
    n = (40, 36, 32)
    v, tr = pi.propeller_mesh(n_blades=4, scale=0.1, n_st=8, n_pts=16, hub_seg=16)
    rho, u = pi.perturbed_flow(n[::-1], 61, u0=(0.02, 0.0, 0.01))
    w = (0.03, 0.0, 0.0)
    runs = []
    for h in ("0", "1"):
        old = os.environ.get("PSM_HIOCC")
        os.environ["PSM_HIOCC"] = h
        try:
            g = _sim(nx=n[0], ny=n[1], nz=n[2], Q=19, tau=0.6, prec="f64", pattern=pattern,
                     collision=collision)
        finally:
            if old is None:
                os.environ.pop("PSM_HIOCC", None)
            else:
                os.environ["PSM_HIOCC"] = old
        g.init_equilibrium(rho, u)
        g.set_mesh(1, v, tr, 1, np.eye(3), (20.0, 18.0, 16.0), (0, 0, 0), w)
        for k in (1, 6, 9):
            g.step(k)
        runs.append((g.pdfs(), g.force_torque(1)[0]))
        g.close()
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    o = oracle.Oracle(*n, 19, 0.6, (0, 0, 0), 1, 1)
    o.set_collision(collision)
    o.init_equilibrium(rho, u)
    o.set_mesh(1, v, tr, 1)
    for k in range(16):
        Qk, tk = oracle.pose_advance(np.eye(3), (20.0, 18.0, 16.0), (0, 0, 0), w, k, list(n),
                                     [1, 1, 1])
        o.set_pose(1, Qk, tk, (0, 0, 0), w)
        o.map()
        o.step(1)
    assert np.max(np.abs(o.pdfs() - runs[0][0])) <= F64_TOL
