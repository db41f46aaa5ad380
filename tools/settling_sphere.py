#!/usr/bin/env python
"""Settling sphere (the paper's two-way coupling validation class; NEXT rank 1)
on the B200 path: a sphere of density ratio rho_s/rho_f falls under gravity in a closed box,
integrated every step from its own PSM force/torque (Eqs.(10)-(11)) by the library's coupling
(DESIGN.md §12).  The paper compares with ten Cate et al.'s measured curves, which are not
available offline; this reports the terminal velocity against the Schiller-Naumann drag
correlation for an unbounded fluid, C_D = 24/Re (1 + 0.15 Re^0.687) — a context number (the box
walls at 4 diameters slow the sphere by O(10 %)), not a pin.  Needs a GPU.

usage: python tools/settling_sphere.py [--out profiles/r01_settling_sphere.md]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def schiller_naumann_velocity(r, nu, ratio, g):
    """Terminal velocity from (ratio - 1) V g = C_D(Re) pi r^2 U^2 / 2 (fixed-point iteration)."""
    d = 2 * r
    U = 1e-3
    for _ in range(200):
        Re = U * d / nu
        cd = 24.0 / Re * (1 + 0.15 * Re ** 0.687)
        U = np.sqrt((ratio - 1) * (4.0 / 3.0) * np.pi * r ** 3 * g / (0.5 * cd * np.pi * r ** 2))
    return U, U * d / nu


def run(nx=96, nz=320, r=6.0, tau=0.65, ratio=1.5, g=3.8e-4, steps=6000, every=100, s=2,
        prec="f64"):
    import paper_2502_20049_b200 as psm
    sim = psm.Simulation(nx, nx, nz, Q=19, tau=tau, bc=(1, 1, 1), prec=prec, sc=1, bmode=1)
    sim.init_equilibrium()
    vol = 4.0 / 3.0 * np.pi * r ** 3
    m = ratio * vol
    z0 = nz - 3 * 2 * r
    sim.set_sphere(1, r, s, np.eye(3), (nx / 2, nx / 2, z0))
    sim.set_dynamics(1, m, 0.4 * m * r * r * np.eye(3),
                     ext_force=(0.0, 0.0, -(m - vol) * g))
    hist = []
    for k in range(0, steps, every):
        sim.step(every)
        _, t, v, _ = sim.body_state(1)
        hist.append((k + every, float(t[2]), float(v[2])))
        if hist[-1][1] < 3 * 2 * r:  # stop before the bottom wall
            break
    sim.close()
    return hist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    r, tau, ratio, g = 6.0, 0.65, 1.5, 3.8e-4
    nu = (tau - 0.5) / 3
    hist = run(r=r, tau=tau, ratio=ratio, g=g)
    U_sn, Re_sn = schiller_naumann_velocity(r, nu, ratio, g)
    w = np.array([h[2] for h in hist])
    U_t = -float(np.mean(w[-5:]))
    drift = float(np.std(w[-5:]) / max(abs(np.mean(w[-5:])), 1e-30))
    lines = ["# Settling sphere (two-way coupled PSM, B200 path)", "",
             f"D3Q19 fp64, 96x96x320 closed box, sphere d = {2 * r:g} cells (s = 2), "
             f"rho_s/rho_f = {ratio}, tau = {tau} (nu = {nu:.4f}), g = {g:g} (lattice units)", "",
             "| step | z_c | w |", "|---|---|---|"]
    for k, z, v in hist:
        lines.append(f"| {k} | {z:.3f} | {v:.6f} |")
    lines += ["", f"terminal velocity (mean of the last 5 samples): {U_t:.5f} "
              f"(relative spread {drift:.1e}); Re = {U_t * 2 * r / nu:.2f}",
              f"Schiller-Naumann, unbounded fluid: {U_sn:.5f} (Re = {Re_sn:.2f}); "
              f"ratio {U_t / U_sn:.3f} (walls at 4 d and the PSM resolution lower it)"]
    text = "\n".join(lines) + "\n"
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    print(text)


if __name__ == "__main__":
    main()
