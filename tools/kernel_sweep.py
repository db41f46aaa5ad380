#!/usr/bin/env python
"""Collide-kernel sweep (no bodies: every tile takes the fluid path, so this isolates the
stream-collide of each operator / stencil / precision / streaming pattern).  Prints one JSON
line per variant: MLUPS and the fraction of the measured HBM bandwidth at 2*Q*S bytes/update.

usage: python tools/kernel_sweep.py [--n 384] [--steps 40] [--only srt19f64aa,cum19f64aa]
Under ncu --metrics gpu__time_duration.sum the AA even/odd launches alternate in the list.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {}
for q in (19, 27):
    for prec in ("f32", "f64"):
        for pat in ("two_array", "aa"):
            for coll in ("srt", "trt", "cumulant"):
                name = f"{coll[:3]}{q}{prec}{'aa' if pat == 'aa' else ''}"
                VARIANTS[name] = (q, prec, pat, coll)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=384)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pads", default="", help="comma list of PSM_PLANE_PAD values to cycle")
    ap.add_argument("--only", default="srt19f64,srt19f64aa,cum19f64,cum19f64aa,srt19f32aa,"
                                      "cum27f32,cum27f64,cum19f32aa")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2502_20049_b200 as psm
    peak, _ = bench.load_peak()
    n = a.n
    pads = a.pads.split(",") if a.pads else [None]
    for name, pad in [(nm, pd) for nm in a.only.split(",") for pd in pads]:
        Q, prec, pat, coll = VARIANTS[name]
        if pad is not None:
            os.environ["PSM_PLANE_PAD"] = pad
        sim = psm.Simulation(n, n, n, Q=Q, tau=0.6, prec=prec, pattern=pat, collision=coll)
        sim.init_equilibrium(None, None)
        sim.step(4)
        st = torch.cuda.current_stream()
        times = []
        clk = bench.ClockSampler(torch.cuda.current_device())
        clk.__enter__()
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            sim.step(a.steps)
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / a.steps)
        clk.__exit__()
        sim.close()
        del sim
        torch.cuda.empty_cache()
        ms = float(np.median(times))
        mlups = n ** 3 / (ms / 1e3) / 1e6
        S = 8 if prec == "f64" else 4
        print(json.dumps({"variant": name, "n": n, "pad": pad, "ms_per_step": ms, "mlups": mlups,
                          "frac": mlups * 1e6 * 2 * Q * S / (peak * 1e9),
                          "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
