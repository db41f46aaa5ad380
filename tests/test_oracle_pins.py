"""Pins of the CPU oracle against what the paper and mathematics fix (P1-P13).

None of these re-types an oracle formula and compares it with itself: each checks a closed form,
an invariant, a special case that reduces to a textbook result, or a brute force computed here
by an independent method.  All run on CPU (`-m "not gpu"`).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import psm_inputs as pi


# ----------------------------------------------------------------------------- P1 stencils ---
@pytest.mark.parametrize("Q", [19, 27])
def test_p1_stencil_tables(Q):
    c, w, opp = oracle.stencil(Q)
    # Independent construction: D3Q27 = {-1,0,1}^3 with w = prod_a w1(c_a), w1(0)=2/3,
    # w1(+-1)=1/6 (tensor product of D1Q3); D3Q19 = {|c|^2 <= 2} with 1/3, 1/18, 1/36.
    vecs = {tuple(int(x) for x in row) for row in c}
    assert len(vecs) == Q
    allv = {(a, b, d) for a in (-1, 0, 1) for b in (-1, 0, 1) for d in (-1, 0, 1)}
    expect = allv if Q == 27 else {v for v in allv if sum(x * x for x in v) <= 2}
    assert vecs == expect
    for i in range(Q):
        n = int(np.sum(np.abs(c[i])))
        if Q == 27:
            wf = Fraction(1)
            for x in c[i]:
                wf *= Fraction(2, 3) if x == 0 else Fraction(1, 6)
        else:
            wf = [Fraction(1, 3), Fraction(1, 18), Fraction(1, 36)][n]
        assert w[i] == float(wf)
        assert np.all(c[opp[i]] == -c[i])
        assert opp[opp[i]] == i
    assert tuple(c[0]) == (0, 0, 0)
    assert abs(w.sum() - 1.0) < 1e-15
    # isotropy up to 4th order: sum w c_a c_b = delta/3; sum w c_a^2 c_b^2 = 1/9 (a != b);
    # sum w c_a^4 = 1/3; odd moments vanish
    cf = c.astype(np.float64)
    M2 = np.einsum("i,ia,ib->ab", w, cf, cf)
    assert np.allclose(M2, np.eye(3) / 3.0, atol=1e-15)
    assert np.allclose(np.einsum("i,ia->a", w, cf), 0.0, atol=1e-16)
    assert np.allclose(np.einsum("i,ia,ib,ic->abc", w, cf, cf, cf), 0.0, atol=1e-16)
    for a in range(3):
        assert abs(np.sum(w * cf[:, a] ** 4) - 1 / 3) < 1e-15
        for b in range(3):
            if a != b:
                assert abs(np.sum(w * cf[:, a] ** 2 * cf[:, b] ** 2) - 1 / 9) < 1e-15


# --------------------------------------------------------------------------- P2 equilibrium --
@pytest.mark.parametrize("Q", [19, 27])
def test_p2_equilibrium_moments(Q):
    """sum f^eq = rho, sum f^eq c = rho u, sum f^eq c c = rho (u u + I/3): the last one fixes
    both the magnitude and the SIGN of the u^2 term (reading A1: with the printed '+',
    sum f^eq = rho (1 + 3u^2))."""
    c, w, _ = oracle.stencil(Q)
    cf = c.astype(np.float64)
    xi = pi.uniform_pm1(7, 4 * 20).reshape(20, 4)
    for k in range(20):
        rho = 1.0 + 0.2 * xi[k, 0]
        u = 0.1 * xi[k, 1:]
        feq = oracle.equilibrium(Q, rho, u)
        assert abs(feq.sum() - rho) < 1e-15 * 4
        assert np.allclose(feq @ cf, rho * u, atol=1e-16 * 8, rtol=0)
        M2 = np.einsum("i,ia,ib->ab", feq, cf, cf)
        assert np.allclose(M2, rho * (np.outer(u, u) + np.eye(3) / 3), atol=5e-16, rtol=0)
    # rest state: f^eq = w rho exactly
    assert np.array_equal(oracle.equilibrium(Q, 1.0, [0, 0, 0]), w)


# ------------------------------------------------------------------------------- P3 BGK -----
def test_p3_bgk_fixed_point_and_full_relaxation():
    Q = 19
    c, w, _ = oracle.stencil(Q)
    feq = oracle.equilibrium(Q, 1.03, [0.04, -0.02, 0.01])
    out, m, err = oracle.collide_cell(Q, feq, 0.7, 1, 0.0, [0, 0, 0])
    assert err == 0 and np.allclose(out, feq, atol=1e-17, rtol=0)
    f = pi.random_pdfs(Q, (1,), 3, w=w)[:, 0]
    rho = f.sum()
    u = (f @ c.astype(float)) / rho
    out, _, _ = oracle.collide_cell(Q, f, 1.0, 1, 0.0, [0, 0, 0])
    assert np.allclose(out, oracle.equilibrium(Q, rho, u), atol=1e-16, rtol=0)


def test_p3_shear_wave_decay():
    """Decaying shear wave u_x = U sin(2 pi y_c / L) e^{-nu k^2 t}, nu = (tau - 1/2)/3
    (closed-form Navier-Stokes solution; L=64, U=1e-3, tau=0.8)."""
    L, U, tau, steps = 64, 1e-3, 0.8, 2000
    o = oracle.Oracle(1, L, 1, 19, tau, (0, 0, 0), 1, 1)
    yc = np.arange(L) + 0.5
    u = np.zeros((3, 1, L, 1))
    u[0, 0, :, 0] = U * np.sin(2 * np.pi * yc / L)
    o.init_equilibrium(np.ones((1, L, 1)), u)
    o.step(steps)
    _, uu = o.velocity()
    amp = 2.0 / L * np.sum(uu[0, 0, :, 0] * np.sin(2 * np.pi * yc / L))
    nu = (tau - 0.5) / 3.0
    k = 2 * np.pi / L
    rate_meas = -math.log(amp / U) / steps
    assert abs(rate_meas / (nu * k * k) - 1.0) < 0.01


# --------------------------------------------------------- P4 PSM blend / plain LBM at B=0 ---
def _numpy_bgk_push(f, c, w, tau):
    """Independent vectorised BGK collide + periodic push (np.roll), 3cu/4.5cu^2/1.5u^2 form."""
    cf = c.astype(np.float64)
    rho = f.sum(0)
    u = np.einsum("i...,ia->a...", f, cf) / rho
    cu = np.einsum("ia,a...->i...", cf, u)
    usq = (u * u).sum(0)
    feq = w[:, None, None, None] * rho * (1 + 3 * cu + 4.5 * cu * cu - 1.5 * usq)
    fs = f - (f - feq) / tau
    out = np.empty_like(f)
    for i in range(len(w)):
        out[i] = np.roll(fs[i], shift=(c[i, 2], c[i, 1], c[i, 0]), axis=(0, 1, 2))
    return out


@pytest.mark.parametrize("Q", [19, 27])
def test_p4_zero_fraction_is_plain_lbm(Q):
    c, w, _ = oracle.stencil(Q)
    shape = (5, 6, 7)
    rho, u = pi.perturbed_flow(shape, 11)
    o = oracle.Oracle(7, 6, 5, Q, 0.8, (0, 0, 0), 1, 1)
    o.init_equilibrium(rho, u)
    f0 = o.pdfs()
    o.step(1)
    ref = _numpy_bgk_push(f0, c, w, 0.8)
    assert np.max(np.abs(o.pdfs() - ref)) < 2e-16


@pytest.mark.parametrize("sc", [1, 2, 3])
def test_p4_step_equals_cellwise_blend_then_push(sc):
    """Random B in [0,1] and u_s through the test-only field setter: one simulation step equals
    the one-cell Eq.(4) operator applied cell by cell, then pushed by np.roll."""
    Q = 19
    c, w, _ = oracle.stencil(Q)
    shape = (4, 5, 6)
    n = int(np.prod(shape))
    rho, u = pi.perturbed_flow(shape, 21)
    B = pi.random_unit(22, n).reshape(shape)
    B[B < 0.3] = 0.0
    us = 0.05 * pi.uniform_pm1(23, 3 * n).reshape((3,) + shape)
    bid = (B > 0).astype(np.uint8)
    o = oracle.Oracle(6, 5, 4, Q, 0.9, (0, 0, 0), sc, 1)
    o.init_equilibrium(rho, u)
    o.set_fields(B, us, bid)
    f0 = o.pdfs()
    o.step(1)
    fs = np.empty_like(f0)
    for k in range(shape[0]):
        for j in range(shape[1]):
            for i in range(shape[2]):
                out, _, err = oracle.collide_cell(Q, f0[:, k, j, i], 0.9, sc, B[k, j, i],
                                                  us[:, k, j, i])
                assert err == 0
                fs[:, k, j, i] = out
    ref = np.empty_like(f0)
    for q in range(Q):
        ref[q] = np.roll(fs[q], shift=(c[q, 2], c[q, 1], c[q, 0]), axis=(0, 1, 2))
    assert np.array_equal(o.pdfs(), ref)


# ---------------------------------------------------------------- P5 solid operators ---------
@pytest.mark.parametrize("sc", [1, 2, 3])
def test_p5_rest_fluid_invariant_any_B(sc):
    Q = 19
    shape = (6, 6, 6)
    n = int(np.prod(shape))
    o = oracle.Oracle(6, 6, 6, Q, 0.7, (0, 0, 0), sc, 1)
    rho0 = 1.0
    o.init_equilibrium(np.full(shape, rho0), None)
    f0 = o.pdfs()
    B = pi.random_unit(31, n).reshape(shape)
    o.set_fields(B, np.zeros((3,) + shape), np.ones(shape, np.uint8))
    o.step(200)
    assert np.max(np.abs(o.pdfs() - f0)) < 1e-13


@pytest.mark.parametrize("sc", [1, 2, 3])
def test_p5_comoving_body_leaves_uniform_flow_unchanged(sc):
    """f = f^eq(rho, U) everywhere and a sphere translating at v = U, remapped every step
    (periodic, no walls): both brackets of Eqs.(7)-(9) vanish, so the state is unchanged."""
    U = np.array([1.0 / 32, 1.0 / 64, 0.0])
    o = oracle.Oracle(16, 16, 16, 19, 0.8, (0, 0, 0), sc, 1)
    o.set_sphere(1, 3.5, 1)
    o.init_equilibrium(None, np.broadcast_to(U[:, None, None, None], (3, 16, 16, 16)).copy())
    f0 = o.pdfs()
    t0 = np.array([8.0, 8.0, 8.0])
    for k in range(20):
        o.set_pose(1, np.eye(3), t0 + k * U, U, (0, 0, 0))
        o.map()
        o.step(1)
    B, _, _, _ = o.fractions()
    assert B.max() == 1.0 and (B > 0).sum() > 100
    assert np.max(np.abs(o.pdfs() - f0)) < 1e-13


def test_p5_special_cases_of_sc_operators():
    Q = 19
    c, w, opp = oracle.stencil(Q)
    cf = c.astype(float)
    f = pi.random_pdfs(Q, (1,), 41, w=w)[:, 0]
    rho = f.sum()
    j = f @ cf
    tau = 0.8
    us = np.array([0.02, -0.01, 0.03])
    # SC3, B = 1, u_s = 0: f*_i = f_ibar (exact bounce-back)
    out, _, _ = oracle.collide_cell(Q, f, tau, 3, 1.0, [0, 0, 0])
    assert np.allclose(out, f[opp], atol=2e-16, rtol=0)
    # Cell momentum after a B = 1 collision (A25):
    # SC1 -> rho u_s ; SC2 -> (1 - 1/tau) j + rho u_s / tau ; SC3 -> 2 rho u_s - j
    expect = {1: rho * us, 2: (1 - 1 / tau) * j + rho * us / tau, 3: 2 * rho * us - j}
    for sc, mom in expect.items():
        out, m, _ = oracle.collide_cell(Q, f, tau, sc, 1.0, us)
        assert np.allclose(out @ cf, mom, atol=1e-16, rtol=0)
        assert abs(out.sum() - rho) < 1e-15          # mass: sum_i Omega^S_i = 0
        assert np.allclose(m, mom - j, atol=1e-16, rtol=0)  # m = momentum the fluid gains
    # SC2 literal form == -(f - f^eq(rho,u_s))/tau (reading A2); B=1 => f* = f + Omega^S
    out, _, _ = oracle.collide_cell(Q, f, tau, 2, 1.0, us)
    fs = oracle.equilibrium(Q, rho, us)
    assert np.allclose(out - f, -(f - fs) / tau, atol=2e-16, rtol=0)
    # SC3 with f = f^eq(rho, u_s): Omega^S = 0, so f* = f + (1-B) Omega^F
    out, _, _ = oracle.collide_cell(Q, fs, tau, 3, 0.4, us)
    u = (fs @ cf) / fs.sum()
    feq = oracle.equilibrium(Q, fs.sum(), u)
    assert np.allclose(out, fs - 0.6 * (fs - feq) / tau, atol=2e-16, rtol=0)


# ----------------------------------------------------------------------------- P8 Eq.(6) ----
def test_p8_weighted_fraction_values():
    for tau in (0.51, 0.6, 0.8, 1.0, 1.7):
        for mode in (0, 1):
            assert oracle.weight_fraction(0.0, tau, mode) == 0.0
            assert oracle.weight_fraction(1.0, tau, mode) == 1.0
    assert oracle.weight_fraction(0.5, 1.0, 1) == 0.25
    assert abs(oracle.weight_fraction(0.5, 0.8, 1) - 3 / 16) <= 2 ** -52 * 3 / 16 * 2
    assert oracle.weight_fraction(0.37, 0.8, 0) == 0.37
    # monotone in eps, and below eps for tau - 1/2 < 1/2... (B/eps = (tau-1/2)/(1-eps+tau-1/2))
    e = np.linspace(0, 1, 101)
    b = np.array([oracle.weight_fraction(x, 0.8, 1) for x in e])
    assert np.all(np.diff(b) > 0)


# --------------------------------------------------------------------------- P11 pose -------
def test_p11_pose_closed_form():
    L = [64.0, 64.0, 64.0]
    per = [1, 1, 1]
    Q0 = pi.rotation_about([1, 2, 3], 0.3)
    t0 = [10.0, 20.0, 30.0]
    w = np.array([0.0, 0.0, 2 * np.pi / 40])
    Qn, tn = oracle.pose_advance(Q0, t0, [0.5, 0, 0], w, 40, L, per)
    assert np.allclose(Qn, Q0, atol=1e-13)           # Rot(w, 2 pi) = I
    assert np.allclose(tn, [(10 + 20) % 64, 20, 30])  # 10 + 40 * 0.5 = 30
    # Rotation about z by theta in closed form
    th = 7 * 0.013
    Qn, _ = oracle.pose_advance(np.eye(3), [0, 0, 0], [0, 0, 0], [0, 0, 0.013], 7, L, per)
    Rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    assert np.allclose(Qn, Rz, atol=1e-15)
    # composition, orthonormality, det
    w = np.array([0.01, -0.02, 0.015])
    Qa, _ = oracle.pose_advance(Q0, t0, [0, 0, 0], w, 5, L, per)
    Qb, _ = oracle.pose_advance(Qa, t0, [0, 0, 0], w, 9, L, per)
    Qc, _ = oracle.pose_advance(Q0, t0, [0, 0, 0], w, 14, L, per)
    assert np.allclose(Qb, Qc, atol=1e-14)
    assert np.allclose(Qc.T @ Qc, np.eye(3), atol=1e-14)
    assert abs(np.linalg.det(Qc) - 1) < 1e-14
    # wrapping on periodic axes: t in [0, L)
    _, tn = oracle.pose_advance(np.eye(3), [63.0, 1.0, 0.0], [1.0, -1.5, 0.0], [0, 0, 0], 3,
                                L, per)
    assert np.allclose(tn, [2.0, 60.5, 0.0])  # 63+3=66->2 ; 1-4.5=-3.5->60.5


# ---------------------------------------------------------------- TRT (NEXT rank 2) ---
def test_trt_reduces_to_srt_and_conserves():
    """tau_- = tau (magic = (tau - 1/2)^2) is SRT; TRT conserves mass and momentum per cell."""
    Q = 19
    c, w, _ = oracle.stencil(Q)
    cf = c.astype(float)
    f = pi.random_pdfs(Q, (1,), 61, w=w)[:, 0]
    tau = 0.73
    a, _, _ = oracle.collide_cell(Q, f, tau, 1, 0.0, [0, 0, 0])
    b, _, _ = oracle.collide_cell_trt(Q, f, tau, (tau - 0.5) ** 2, 1, 0.0, [0, 0, 0])
    assert np.allclose(a, b, atol=2e-16, rtol=0)
    for magic in (3 / 16, 1 / 4, 1 / 12):
        out, _, _ = oracle.collide_cell_trt(Q, f, tau, magic, 1, 0.0, [0, 0, 0])
        assert abs(out.sum() - f.sum()) < 1e-15
        assert np.allclose(out @ cf, f @ cf, atol=1e-16, rtol=0)
        assert np.max(np.abs(out - a)) > 1e-6  # the antisymmetric rate really differs


def test_trt_poiseuille_is_exact_at_magic_3_16():
    """Half-way bounce-back + Guo force + TRT with Lambda = 3/16: the parabolic profile is
    reproduced to round-off (the known exact-wall property of TRT), with u = (j + g/2)/rho."""
    H, tau, g = 16, 0.8, 1e-6
    o = oracle.Oracle(1, H, 1, 19, tau, (0, 1, 0), 1, 1)
    o.set_collision("trt", 3 / 16)
    o.init_equilibrium(None, None)
    o.set_force([g, 0, 0])
    o.step(60000)
    rho, u = o.velocity()
    ux = u[0, 0, :, 0] + 0.5 * g / rho[0, :, 0]
    yc = np.arange(H) + 0.5
    ref = g * yc * (H - yc) / (2 * (tau - 0.5) / 3)
    assert np.max(np.abs(ux - ref)) / ref.max() < 1e-9


# ------------------------------------------------- cumulant (NEXT rank 2) ---
@pytest.mark.parametrize("Q", [19, 27])
def test_cumulant_conservation_idempotence_and_fixed_point(Q):
    c, w, _ = oracle.stencil(Q)
    cf = c.astype(float)
    f = pi.random_pdfs(Q, (1,), 63, w=w, amp=0.2)[:, 0]
    out, _, err = oracle.collide_cell_cum(Q, f, 0.7, 1, 0.0, [0, 0, 0])
    assert err == 0
    assert abs(out.sum() - f.sum()) < 1e-15 * 4
    assert np.allclose(out @ cf, f @ cf, atol=2e-16 * 8, rtol=0)
    # full relaxation (tau = 1) is idempotent, and its result is a fixed point for any tau
    e1, _, _ = oracle.collide_cell_cum(Q, f, 1.0, 1, 0.0, [0, 0, 0])
    e2, _, _ = oracle.collide_cell_cum(Q, e1, 1.0, 1, 0.0, [0, 0, 0])
    e3, _, _ = oracle.collide_cell_cum(Q, e1, 0.63, 1, 0.0, [0, 0, 0])
    assert np.allclose(e2, e1, atol=1e-15, rtol=0) and np.allclose(e3, e1, atol=1e-15, rtol=0)
    # at rest with rho = 1 the cumulant equilibrium is the lattice weights
    r, _, _ = oracle.collide_cell_cum(Q, w * 1.0, 0.9, 1, 0.0, [0, 0, 0])
    assert np.allclose(r, w, atol=1e-16 if Q == 27 else 4e-16, rtol=0)  # (19x19 elimination)


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("U0", [0.0, 0.1])
def test_cumulant_shear_wave_viscosity_and_galilean_invariance(U0, Q):
    """Decay rate nu k^2 with nu = (tau - 1/2)/3, also for a wave advected at U0 = 0.1."""
    L, U, tau, steps = 64, 1e-3, 0.8, 1000
    o = oracle.Oracle(1, L, 1, Q, tau, (0, 0, 0), 1, 1)
    o.set_collision("cumulant")
    yc = np.arange(L) + 0.5
    u = np.zeros((3, 1, L, 1))
    u[0, 0, :, 0] = U0 + U * np.sin(2 * np.pi * yc / L)
    o.init_equilibrium(np.ones((1, L, 1)), u)
    o.step(steps)
    _, uu = o.velocity()
    amp = 2.0 / L * np.sum((uu[0, 0, :, 0] - U0) * np.sin(2 * np.pi * yc / L))
    nu = (tau - 0.5) / 3.0
    k = 2 * np.pi / L
    assert abs(-math.log(amp / U) / steps / (nu * k * k) - 1.0) < 0.01


@pytest.mark.parametrize("Q", [19, 27])
def test_cumulant_forcing_momentum_and_poiseuille(Q):
    """Reading A31: with a body force the first-order central moments about u = (j + g/2)/rho flip
    sign in the collision, so every cell gains exactly g of momentum (mass unchanged); a forced
    channel between resting walls gives the Poiseuille parabola (D3Q27 and D3Q19 cumulant)."""
    c, w, _ = oracle.stencil(Q)
    cf = c.astype(float)
    g = np.array([2e-4, -1e-4, 5e-5])
    f = pi.random_pdfs(Q, (1,), 64, w=w, amp=0.2)[:, 0]
    out, _, err = oracle.collide_cell_cum(Q, f, 0.7, 1, 0.0, [0, 0, 0], g=g)
    assert err == 0
    assert abs(out.sum() - f.sum()) < 1e-15 * 4
    assert np.allclose(out @ cf, f @ cf + g, atol=2e-16 * 8, rtol=0)
    H, tau, gx = 16, 0.8, 1e-6
    o = oracle.Oracle(1, H, 1, Q, tau, (0, 1, 0), 1, 1)
    o.set_collision("cumulant")
    o.init_equilibrium(None, None)
    o.set_force([gx, 0, 0])
    o.step(6000)
    rho, u = o.velocity()
    ux = u[0, 0, :, 0] + 0.5 * gx / rho[0, :, 0]
    yc = np.arange(H) + 0.5
    ref = gx * yc * (H - yc) / (2 * (tau - 0.5) / 3)
    assert np.max(np.abs(ux - ref)) / ref.max() < 0.02


def _set_partitions(items):
    """All set partitions of a list (Bell(6) = 203 for a sixth-order multi-index)."""
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for p in _set_partitions(rest):
        for i in range(len(p)):
            yield p[:i] + [[first] + p[i]] + p[i + 1:]
        yield [[first]] + p


def _cumulant(f, c, abc):
    """Joint cumulant of the velocity distribution f / rho for the multi-index (a, b, c), from
    its raw moments by the textbook set-partition formula
    kappa(X_1..X_n) = sum_pi (|pi| - 1)! (-1)^(|pi|-1) prod_B E[prod_{i in B} X_i] — no central
    moments, no Wick products, nothing shared with the oracle's transform."""
    rho = f.sum()
    vs = [0] * abc[0] + [1] * abc[1] + [2] * abc[2]

    def mom(block):
        pr = np.ones(len(f))
        for i in block:
            pr = pr * c[:, vs[i]]
        return float((f * pr).sum() / rho)

    tot = 0.0
    for p in _set_partitions(list(range(len(vs)))):
        k = len(p)
        tot += (-1) ** (k - 1) * math.factorial(k - 1) * np.prod([mom(B) for B in p])
    return tot


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("tau", [0.6, 0.8, 1.7])
def test_cumulant_relaxes_each_cumulant_as_a29_states(tau, Q):
    """Reading A29 pinned cumulant by cumulant on a strongly sheared,
    anisotropic, moving random f: after the collision every cumulant of order >= 3 of f/rho
    vanishes; the off-diagonal second cumulants and the two deviatoric differences are
    multiplied by 1 - 1/tau; the trace is its equilibrium 3 c_s^2 = 1; rho and j are kept.
    The cumulants come from raw moments by the set-partition formula (numpy, independent of the
    oracle's central-moment/Wick arithmetic), so a wrong coefficient in any Wick product
    (e.g. kappa_xxyy = rho (C_xx C_yy + 2 C_xy^2)) leaves a nonzero post-collision cumulant.
    D3Q19 (reading A32): the 19 multi-indices with at least one zero order, the moments the
    velocity set carries (xyz, x^2yz, ... are not independent on it and are not checked)."""
    c, w, _ = oracle.stencil(Q)
    cf = c.astype(float)
    u = np.array([0.05, -0.03, 0.02])
    cu = cf @ u
    f = w * (1 + 3 * cu + 4.5 * cu ** 2 - 1.5 * (u @ u))
    f += w * 9 * (0.03 * cf[:, 0] * cf[:, 1] + 0.02 * cf[:, 1] * cf[:, 2] +
                  0.015 * cf[:, 0] * cf[:, 2])
    f += w * 0.06 * (cf[:, 0] ** 2 - cf[:, 1] ** 2)
    f *= 1 + 0.1 * pi.uniform_pm1(5, Q)
    assert f.min() > 0
    out, _, err = oracle.collide_cell_cum(Q, f, tau, 1, 0.0, [0, 0, 0])
    assert err == 0
    idx = [(a, b, k) for a in range(3) for b in range(3) for k in range(3) if a + b + k > 0 and
           (Q == 27 or min(a, b, k) == 0)]
    assert len(idx) == Q - 1
    pre = {m: _cumulant(f, cf, m) for m in idx}
    post = {m: _cumulant(out, cf, m) for m in idx}
    r = 1.0 - 1.0 / tau
    assert max(abs(pre[m]) for m in idx if sum(m) >= 3) > 1e-3  # far from equilibrium
    for m in idx:
        if sum(m) >= 3:
            assert abs(post[m]) < 1e-15, (m, pre[m], post[m])
    for m in [(1, 0, 0), (0, 1, 0), (0, 0, 1)]:
        assert abs(post[m] - pre[m]) < 1e-16, m
    for m in [(1, 1, 0), (1, 0, 1), (0, 1, 1)]:
        assert abs(post[m] - r * pre[m]) < 1e-15, (m, pre[m], post[m])
    assert abs(post[(1, 1, 0)]) > 1e-3 or tau == 1.0  # the sheared state survives the collision
    for a, b in [((2, 0, 0), (0, 2, 0)), ((2, 0, 0), (0, 0, 2))]:
        assert abs((post[a] - post[b]) - r * (pre[a] - pre[b])) < 1e-15
    assert abs(post[(2, 0, 0)] + post[(0, 2, 0)] + post[(0, 0, 2)] - 1.0) < 1e-15
    assert abs(out.sum() - f.sum()) < 1e-15


def test_integrator_world_inertia_is_q_i_qt():
    """Two-way coupling integrator (reading A28) with an anisotropic,
    non-diagonal body-frame inertia and a rotated initial pose: a body at rest in fluid at rest
    feels no fluid force (rest state invariant, P5), so one step gives exactly
    dv = F_e / m, t1 = t0 + dv (semi-implicit), dw = (Q0 I Q0^T)^-1 T_e (numpy.linalg.solve, not
    the oracle's adjugate) and Q1 = exp([dw]x) Q0 (scipy rotation vector, not Rodrigues as
    coded).  Q0^T I Q0 (the other convention) differs by ~2x here."""
    from scipy.spatial.transform import Rotation
    n = 12
    o = oracle.Oracle(n, n, n, 19, 0.8, (0, 0, 0), 1, 1)
    o.init_equilibrium(None, None)
    o.set_sphere(1, 3.0, 1)
    Q0 = pi.rotation_about([1, 2, 3], 0.8)
    t0 = np.array([6.2, 5.9, 6.4])
    o.set_pose(1, Q0, t0, (0, 0, 0), (0, 0, 0))
    inertia = np.array([[300.0, 20.0, -15.0], [20.0, 450.0, 35.0], [-15.0, 35.0, 700.0]])
    Fe = np.array([1e-3, -2e-3, 5e-4])
    Te = np.array([2e-3, -1e-3, 3e-3])
    m = 500.0
    o.set_dynamics(1, m, inertia, Fe, Te)
    o.map()
    o.step(1)
    F, T, _, _ = o.force_torque(1)
    assert np.all(F == 0) and np.all(T == 0)
    o.integrate()
    Q, t, v, w = o.body_state(1)
    w_ref = np.linalg.solve(Q0 @ inertia @ Q0.T, Te)
    assert np.allclose(w, w_ref, rtol=1e-13, atol=0)
    assert not np.allclose(w, np.linalg.solve(Q0.T @ inertia @ Q0, Te), rtol=0.1, atol=0)
    assert np.allclose(v, Fe / m, rtol=1e-15, atol=0)
    assert np.allclose(t, t0 + Fe / m, rtol=0, atol=1e-15)
    Q_ref = Rotation.from_rotvec(w_ref).as_matrix() @ Q0
    assert np.abs(Q - Q_ref).max() < 1e-14
