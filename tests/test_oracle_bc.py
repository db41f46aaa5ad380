"""Pins of the oracle's open boundaries (reading A30): velocity inflow at x = 0
(moving-wall bounce-back, rho_w = 1) and pressure outflow at x = nx-1 (anti-bounce-back with
rho_out and the normal velocity u_x = (S_0 + 2 S_+)/rho_out - 1 of the known populations).  The paper only names "boundary handling for
inflow and outflow"; the pins fix the reading by what it must satisfy:
  B1  a uniform normal stream f^eq(1, U) with u_in = U, rho_out = 1 is an exact fixed point
      (both stencils, SRT and TRT) — a wrong sign, factor or density in either rule breaks it;
  B2  a closed inlet (u_in = 0) and an open outlet relax the density of a fluid at rest to
      rho_out (the outflow fixes the pressure);
  B3  channel with no-slip walls: the steady mass flux is the same through every x plane and
      equals the inflow flux H * U; far from the inlet the profile is Poiseuille's parabola.
"""
import numpy as np
import pytest

import oracle


def _uniform(shape, U, rho=1.0):
    nz, ny, nx = shape
    r = np.full(shape, rho)
    u = np.empty((3,) + shape)
    for a in range(3):
        u[a] = U[a]
    return r, u


@pytest.mark.parametrize("Q", [19, 27])
@pytest.mark.parametrize("coll", ["srt", "trt"])
def test_b1_uniform_stream_is_a_fixed_point(Q, coll):
    U = (0.05, 0.0, 0.0)  # the outflow assumes a normal stream (u_y = u_z = 0, A30)
    nx, ny, nz = 12, 4, 3
    o = oracle.Oracle(nx, ny, nz, Q, 0.7, (2, 0, 0), 1, 1)
    o.set_collision(coll)
    o.set_open_boundary(U, 1.0)
    rho, u = _uniform((nz, ny, nx), U)
    o.init_equilibrium(rho, u)
    f0 = o.pdfs()
    o.step(40)
    assert np.max(np.abs(o.pdfs() - f0)) < 2e-15
    # the same state with a wrong inflow velocity is not a fixed point (the pin has teeth)
    o2 = oracle.Oracle(nx, ny, nz, Q, 0.7, (2, 0, 0), 1, 1)
    o2.set_open_boundary((0.04, 0.0, 0.0), 1.0)
    o2.init_equilibrium(rho, u)
    o2.step(1)
    assert np.max(np.abs(o2.pdfs() - f0)) > 1e-4


def test_b2_outflow_fixes_the_density():
    nx = 8
    o = oracle.Oracle(nx, 1, 1, 19, 1.5, (2, 0, 0), 1, 1)
    o.set_open_boundary((0.0, 0.0, 0.0), 1.0)
    rho, u = _uniform((1, 1, nx), (0.0, 0.0, 0.0), rho=1.01)
    o.init_equilibrium(rho, u)
    o.step(1500)
    r, v = o.velocity()
    assert np.max(np.abs(r - 1.0)) < 1e-6
    assert np.max(np.abs(v)) < 1e-6
    # a different outlet density is reached just as well
    o.set_open_boundary((0.0, 0.0, 0.0), 0.995)
    o.step(1500)
    r, _ = o.velocity()
    assert np.max(np.abs(r - 0.995)) < 1e-6


def test_b3_channel_flux_and_poiseuille_profile():
    nx, H, tau, U = 96, 16, 0.8, 0.02
    o = oracle.Oracle(nx, H, 1, 19, tau, (2, 1, 0), 1, 1)
    o.set_open_boundary((U, 0.0, 0.0), 1.0)
    rho, u = _uniform((1, H, nx), (U, 0.0, 0.0))
    o.init_equilibrium(rho, u)
    o.step(12000)
    r, v = o.velocity()
    flux = (r[0] * v[0, 0]).sum(axis=0)  # per x plane
    inner = flux[2:-2]
    assert np.max(np.abs(inner - inner.mean())) / inner.mean() < 1e-4  # steady: same everywhere
    assert abs(inner.mean() / (H * U) - 1) < 0.01                     # = the inflow flux
    # far from the inlet: parabola with the same mean velocity
    yc = np.arange(H) + 0.5
    prof = v[0, 0, :, 3 * nx // 4]
    ref = 6.0 * prof.mean() * (yc / H) * (1 - yc / H)
    assert np.max(np.abs(prof - ref)) / ref.max() < 0.03
    # developed flow between the inlet and outlet regions: no cross flow
    assert np.max(np.abs(v[1, 0, :, nx // 4:3 * nx // 4])) < 1e-4 * U
