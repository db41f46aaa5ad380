"""Pins of the oracle's dynamics (P6, P7, P12, P13): exact conservation and
momentum-exchange identities that fix the force/torque of Eqs.(10)-(11)
independently of the reduction code, forced momentum balance, and Poiseuille flow."""
import numpy as np
import pytest

import oracle
import psm_inputs as pi


def _momentum(f, cf):
    return cf.T @ f.reshape(f.shape[0], -1).sum(axis=1)


def _abs_momentum(f, cf):
    return np.abs(cf).T @ np.abs(f).reshape(f.shape[0], -1).sum(axis=1)


def _rotor_sim(sc, n=20, steps=None):
    v, tr = pi.propeller_mesh(n_blades=3, scale=0.06, n_st=8, n_pts=16, hub_seg=16)
    o = oracle.Oracle(n, n, n, 19, 0.7, (0, 0, 0), sc, 1)
    o.set_mesh(1, v, tr, 1)
    rho, u = pi.perturbed_flow((n, n, n), 51, u0=(0.03, 0.0, 0.0))
    o.init_equilibrium(rho, u)
    return o


def _pose(k, w, t0):
    return oracle.pose_advance(pi.rotation_about([0, 1, 0], 0.2), t0, [0.01, 0, 0], w, k,
                               [20.0] * 3, [1, 1, 1])


@pytest.mark.parametrize("sc", [1, 2, 3])
def test_p6_p7_momentum_and_angular_exchange_identities(sc):
    """Periodic, no forcing.  Per step n:
       P^{n+1} - P^n = S_F^n = -F^n                    (momentum gained by the fluid, A6)
       S_T^n = sum_x mi(x_c - R) x m(x),  m(x) = sum_i [f_i^{n+1}(x + c_i) - f_i^n(x)] c_i
    with mass conserved; body rotating and translating, remapped every step."""
    c, w, _ = oracle.stencil(19)
    cf = c.astype(float)
    o = _rotor_sim(sc)
    wv = np.array([0.02, 0.01, -0.015])
    t0 = np.array([10.3, 9.6, 10.1])
    f = o.pdfs()
    mass0 = f.sum()
    n = 20
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    xc = np.stack([x, y, z], 0) + 0.5
    for k in range(12):
        Qk, tk = _pose(k, wv, t0)
        o.set_pose(1, Qk, tk, [0.01, 0, 0], wv)
        o.map()
        o.step(1)
        fn = o.pdfs()
        F, T, AF, AT = o.force_torque(1)
        assert AF.max() > 1e-6
        dP = _momentum(fn, cf) - _momentum(f, cf)
        # rounding scale of the momentum sums: eps * sum |f_i c_i| (summation error bound)
        rnd = 16 * np.finfo(float).eps * _abs_momentum(fn, cf)
        assert np.all(np.abs(dP + F) <= 1e-12 * AF + rnd), (dP, F, AF, rnd)
        m = np.zeros((3, n, n, n))
        for i in range(19):
            back = np.roll(fn[i], shift=(-c[i, 2], -c[i, 1], -c[i, 0]), axis=(0, 1, 2))
            m += (back - f[i])[None] * cf[i][:, None, None, None]
        r = xc - tk[:, None, None, None]
        r = r - n * np.rint(r / n) * (np.abs(r) >= n / 2)
        ST = np.cross(r, m, axis=0).sum(axis=(1, 2, 3))
        absfc = np.einsum("iz...,ia->az...", np.abs(fn)[:, None], np.abs(cf))[:, 0]
        rndT = 16 * np.finfo(float).eps * (np.abs(r).sum(0) * absfc.sum(0)).sum()
        assert np.all(np.abs(ST + T) <= 1e-12 * AT + rndT), (ST, T, AT, rndT)
        f = fn
    assert abs(f.sum() / mass0 - 1) < 1e-13


def test_p6_mass_conservation_long_run():
    o = _rotor_sim(1)
    mass0 = o.pdfs().sum()
    wv = np.array([0.0, 0.03, 0.0])
    for k in range(200):
        Qk, tk = _pose(k, wv, np.array([10.0, 10.0, 10.0]))
        o.set_pose(1, Qk, tk, [0.01, 0, 0], wv)
        o.map()
        o.step(1)
    assert abs(o.pdfs().sum() / mass0 - 1) < 1e-10


def test_p12_forced_momentum_balance_and_drag_direction():
    """Guo body force g on the fluid part ((1-B) weighted): every step
    P^{n+1} - P^n = sum_x (1 - B) g - F^n exactly; and the drag on a stationary sphere points
    along the driven flow."""
    c, _, _ = oracle.stencil(19)
    cf = c.astype(float)
    n = 16
    g = np.array([2e-5, 0.0, 0.0])
    o = oracle.Oracle(n, n, n, 19, 0.8, (0, 0, 0), 2, 1)
    o.set_force(g)
    o.set_sphere(1, 3.0, 2)
    o.set_pose(1, np.eye(3), (8.0, 8.0, 8.0))
    o.map()
    B = o.fractions()[0]
    o.init_equilibrium(None, None)
    f = o.pdfs()
    for k in range(300):
        o.step(1)
        fn = o.pdfs()
        F, _, AF, _ = o.force_torque(1)
        dP = _momentum(fn, cf) - _momentum(f, cf)
        expect = (1 - B).sum() * g - F
        rnd = 16 * np.finfo(float).eps * _abs_momentum(fn, cf)
        assert np.all(np.abs(dP - expect) <= 1e-12 * AF + rnd)
        f = fn
    assert F[0] > 0 and abs(F[1]) < 1e-3 * F[0] and abs(F[2]) < 1e-3 * F[0]


def test_p13_poiseuille_and_resting_walls():
    """Half-way bounce-back walls at y = 0 and y = H, Guo force g_x:
    u(y_c) = g y_c (H - y_c) / (2 nu), nu = (tau - 1/2)/3 (closed form); rest state with walls
    is invariant."""
    H, tau, g = 32, 0.8, 1e-6
    o = oracle.Oracle(1, H, 1, 19, tau, (0, 1, 0), 1, 1)
    o.init_equilibrium(None, None)
    f0 = o.pdfs()
    o.step(50)
    assert np.max(np.abs(o.pdfs() - f0)) < 1e-15
    o.set_force([g, 0, 0])
    o.step(15000)
    _, u = o.velocity()
    yc = np.arange(H) + 0.5
    nu = (tau - 0.5) / 3
    ref = g * yc * (H - yc) / (2 * nu)
    assert np.max(np.abs(u[0, 0, :, 0] - ref)) / ref.max() < 0.02
    assert np.max(np.abs(u[1:])) < 1e-12
