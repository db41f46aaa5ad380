"""Full-size check in the launch configuration bench.py times (BASELINE config c5, N=1: 512^3
fp32, CROR-like rotor pair with the full ~0.6 M-face meshes, two-array pull, SC1, weighted B).
The oracle cannot run 134 M cells, so: (a) sampled fluid cells are recomputed one by one by the
oracle's one-cell operator and compared with the pushed post-step populations; (b) total mass is
conserved; (c) the mapped solid volume matches the meshes' own volume (divergence theorem)."""
import os
import sys

import numpy as np
import pytest

import oracle
import psm_inputs as pi

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mesh_volume(v, t):
    return np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6.0


def test_c5w_full_size_sampled_cells_and_invariants():
    sys.path.insert(0, ROOT)
    import bench
    import paper_2502_20049_b200 as psm
    wl = bench.WORKLOADS["c5w"]
    sim, poses, nb, _ = bench.build_workload(psm, wl, 0, 1)
    sim.step(4)  # let the rotors stir the rest fluid
    n = wl["nx"]
    # (c) mapped solid volume vs mesh volume (s = 1: eps = cnt / 8)
    _, bid, cnt = sim.fractions()
    for b, front in ((1, True), (2, False)):
        v, t = pi.cror_rotor(front)
        vol = _mesh_volume(v, t)
        got = cnt[bid == b].sum() / 8.0
        assert abs(got / vol - 1) < 0.01, (b, got, vol)
    # (b) mass before/after
    rho0, _ = sim.velocity()
    m0 = rho0.sum(dtype=np.float64)
    # (a) sampled fluid cells: planes 250..262 read before and after one step
    z0, nzp = 250, 13
    before = sim.pdfs_planes(z0, nzp)
    sim.step(1)
    after = sim.pdfs_planes(z0, nzp)
    rho1, _ = sim.velocity()
    assert abs(rho1.sum(dtype=np.float64) / m0 - 1) < 1e-7
    c, w, _ = oracle.stencil(19)
    rng = np.random.default_rng(5)
    rb = [np.max(np.linalg.norm(pi.cror_rotor(f)[0], axis=1)) for f in (True, False)]
    checked = 0
    worst = 0.0
    while checked < 400:
        x, y, z = rng.integers(1, n - 1), rng.integers(1, n - 1), rng.integers(1, nzp - 1)
        xc = np.array([x + 0.5, y + 0.5, z0 + z + 0.5])
        # certainly fluid (B = 0, independent of the GPU fractions): outside both bounding spheres
        if any(np.linalg.norm(xc - np.array(p[1])) <= r + 2.0 for p, r in zip(poses, rb)):
            continue
        fs, _, err = oracle.collide_cell(19, before[:, z, y, x], wl["tau"], wl["sc"], 0.0,
                                         [0, 0, 0])
        assert err == 0
        for i in range(19):
            got = after[i, z + c[i, 2], y + c[i, 1], x + c[i, 0]]
            worst = max(worst, abs(got - fs[i]))
        checked += 1
    assert worst <= 2e-6, worst  # fp32 storage and arithmetic vs fp64 oracle, one step
    # the rotors are in the sampled planes too: nonzero forces on both
    for b in (1, 2):
        F, T, aF, aT = sim.force_torque(b)
        assert aF.max() > 0


def test_c5w_shaped_256_rotor_pair_full_parity():
    """The measured configuration's hard paths at a size the oracle can follow: c5w scaled to
    256^3 (D3Q19 fp32, SRT + SC1, weighted B, tau = 0.55, two-array, rest start), the
    counter-rotating rotor pair of the c5 recipe at half size (12 + 10 blades, tips 100 / 90,
    ~57 k faces together, s = 1), advanced by the library itself in ONE psm_step(20) call
    (closed-form poses, remap-ahead pipeline, cached narrow band) against the oracle fed
    oracle.pose_advance poses: counts bit-exact after the run, fp32 PDFs within 2e-5 of the
    fp64 oracle on every cell (PSM cells included), F/T of the last step within fp32 bounds."""
    import paper_2502_20049_b200 as psm
    n, steps, tau, om = 256, 20, 0.55, 0.05 / 110.0
    rot = [(pi.propeller_mesh(n_blades=12, scale=100 / 110, n_st=40, n_pts=32, hub_seg=64),
            (100.0, 128.0, 128.0), (om, 0.0, 0.0)),
           (pi.propeller_mesh(n_blades=10, scale=90 / 110, n_st=40, n_pts=32, hub_seg=64),
            (165.0, 128.0, 128.0), (-om, 0.0, 0.0))]
    g = psm.Simulation(n, n, n, Q=19, tau=tau, prec="f32", sc=1, bmode=1)
    o = oracle.Oracle(n, n, n, 19, tau, (0, 0, 0), 1, 1)
    g.init_equilibrium(None, None)
    o.init_equilibrium(None, None)
    for b, ((v, t), pos, w) in enumerate(rot):
        g.set_mesh(b + 1, v, t, 1, np.eye(3), pos, (0, 0, 0), w)
        o.set_mesh(b + 1, v, t, 1)
    for k in range(steps):
        for b, (_, pos, w) in enumerate(rot):
            Qk, tk = oracle.pose_advance(np.eye(3), pos, (0, 0, 0), w, k, [n] * 3, [1] * 3)
            o.set_pose(b + 1, Qk, tk, (0, 0, 0), w)
        o.map()
        o.step(1)
    g.step(steps)
    _, ido, co, _ = o.fractions()
    _, idg, cg = g.fractions()
    assert np.array_equal(co, cg) and np.array_equal(ido, idg)
    fo = o.pdfs()
    fg = g.pdfs()
    d = np.abs(fo - fg).max(axis=0)
    psm_cells = co > 0
    assert psm_cells.sum() > 10000
    assert d[psm_cells].max() <= 2e-5, d[psm_cells].max()
    assert d.max() <= 2e-5, d.max()
    for b in (1, 2):
        Fg, Tg, _, _ = g.force_torque(b)
        Fo, To, aF, aT = o.force_torque(b)
        assert np.all(np.abs(Fg - Fo) <= 1e-4 * aF + 1e-12), (b, Fg, Fo, aF)
        assert np.all(np.abs(Tg - To) <= 1e-4 * aT + 1e-12), (b, Tg, To, aT)
    g.close()
