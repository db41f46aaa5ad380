#!/usr/bin/env python
"""BASELINE config c3 — the paper's GPU node-level experiment on one B200.

One 256^3 block per GPU (the paper: four A100s with one 256^3 block each), fp64, the two
scenarios of P:478-479 / Fig. blockstructures:
  A  rotating geometry over the whole domain: four coaxial 6-blade rotors (tip 118, wide chord
     60 -> 50 cells, ~0.3 M faces each, ~1.2 M faces together — the paper's CROR face count,
     P:284) spaced 64 cells along the rotation axis x, so their swept boxes cover ~88 % of the
     cells (each rotor's bounding radius 122 < 127, the minimum-image limit of a 256-cell axis)
  B  rotating geometry in a small part of the domain: one 6-blade propeller of the c3 recipe
     scaled x0.4 (tip 44), ~0.3 M faces
and the paper's kernel variants:
  V0 LBM (no PSM bodies: every tile takes the fluid path)
  V1 PSM, static geometry (mapped once)
  V2/V3/V4 PSM, geometry rotating at Omega = 0.05/r_tip rad/step, remapped every step, s = 0/1/2
Each figure: median of `--reps` repetitions of `--steps` steps (CUDA events on the library's
stream, after warm-up), MLUPS, fraction of the measured HBM bandwidth (2*Q*S bytes per update,
the paper's roofline model P:504-507), and the overhead 1 - V/V0 next to the paper's
-8 % (B) / -10 % (A) for rotation on A100.

usage: python tools/c3_node_level.py [--ops srt27,cum27,cum19aa] [--out profiles/r02_c3.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OPS = {  # name -> (Q, collision, pattern)
    "srt27": (27, "srt", "two_array"),
    "cum27": (27, "cumulant", "two_array"),
    "cum19aa": (19, "cumulant", "aa"),  # the paper's own performance operator
    "cum19": (19, "cumulant", "two_array"),
    "srt19aa": (19, "srt", "aa"),
    "srt19": (19, "srt", "two_array"),
    "srt27aa": (27, "srt", "aa"),
}
N = 256
_MESH = {}


def meshes(scen):
    import psm_inputs as pi
    if scen not in _MESH:
        if scen == "A":
            v, t = pi.propeller_mesh(n_blades=6, hub_r=12.0, hub_len=48.0, r_tip=118.0,
                                     chord=(60.0, 50.0), pitch=(25.0, 15.0), thick=4.0,
                                     n_st=160, n_pts=160, hub_seg=128)
            _MESH[scen] = [((v, t), (32.0 + 64.0 * k, N / 2, N / 2), 118.0) for k in range(4)]
        else:
            v, t = pi.propeller_mesh(n_blades=6, scale=0.4, n_st=160, n_pts=160, hub_seg=128)
            _MESH[scen] = [((v, t), (N / 2, N / 2, N / 2), 44.0)]
    return _MESH[scen]


def run(op, scen, var, steps, warmup, reps, mapping="R1"):
    import torch
    import paper_2502_20049_b200 as psm
    Q, coll, pattern = OPS[op]
    sim = psm.Simulation(N, N, N, Q=Q, tau=0.6, prec="f64", pattern=pattern, sc=1, bmode=1,
                         collision=coll)
    sim.init_equilibrium(None, None)
    faces = 0
    cover = 0.0
    if var != "V0":
        s = {"V1": 1, "V2": 0, "V3": 1, "V4": 2}[var]
        for b, ((v, t), pos, tip) in enumerate(meshes(scen)):
            w = (0.0, 0.0, 0.0) if var == "V1" else ((-1) ** b * 0.05 / tip, 0.0, 0.0)
            sim.set_mesh(b + 1, v, t, s, np.eye(3), pos, (0, 0, 0), w, mapping=mapping)
            faces += len(t)
    sim.step(warmup)
    torch.cuda.synchronize()
    if var != "V0":
        _, bid, _ = sim.fractions()
        cover = float((bid > 0).mean())
    st = torch.cuda.current_stream()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        sim.step(steps)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / steps)
    sim.close()
    del sim
    torch.cuda.empty_cache()
    ms = float(np.median(times))
    mlups = N ** 3 / (ms / 1e3) / 1e6
    return {"op": op, "scen": scen, "var": var, "mapping": mapping, "ms_per_step": ms,
            "mlups": mlups,
            "faces": faces, "solid_cell_fraction": cover, "reps_ms": times}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="srt27,cum27,cum19aa")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--json", default=None)
    ap.add_argument("--scen", default="A,B")
    ap.add_argument("--vars", default="V0,V1,V2,V3,V4")
    ap.add_argument("--mapping", default="R1", choices=["R1", "R2"],
                    help="R1: every sub-sample (default); R2: the paper's literal centre-only "
                         "block average (reading A12)")
    a = ap.parse_args()
    import bench
    peak, _ = bench.load_peak()
    rows = []
    for op in a.ops.split(","):
        for scen in a.scen.split(","):
            for var in a.vars.split(","):
                t0 = time.time()
                r = run(op, scen, var, a.steps, a.warmup, a.reps, a.mapping)
                r["frac"] = r["mlups"] * 1e6 * 2 * OPS[op][0] * 8 / (peak * 1e9)
                rows.append(r)
                print(json.dumps(r), f"({time.time() - t0:.0f} s)", flush=True)
    paper = {"A": -0.10, "B": -0.08}
    lines = ["# c3 node-level experiment on one B200 (PAPER.md:556-565; tools/c3_node_level.py)",
             "", f"256^3 cells, fp64, tau = 0.6, SC1, weighted B; {a.steps} steps x {a.reps} "
             f"repetitions (median); fraction = MLUPS x 2QS / {peak:g} GB/s (measured HBM). "
             "Paper (A100, D3Q19 cumulant AA fp64): rotation -10 % (A), -8 % (B) vs LBM, "
             "static PSM = LBM (B) or faster (A), s adds no cost (P:562-565).", "",
             "| operator | scen. | variant | MLUPS | % of HBM | vs V0 | faces | solid cells |",
             "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        v0 = next((x for x in rows if x["op"] == r["op"] and x["scen"] == r["scen"] and
                   x["var"] == "V0"), r)
        ov = r["mlups"] / v0["mlups"] - 1.0
        lines.append(f"| {r['op']} | {r['scen']} | {r['var']} | {r['mlups']:.0f} | "
                     f"{100 * r['frac']:.1f} | {100 * ov:+.1f} % | {r['faces']} | "
                     f"{100 * r['solid_cell_fraction']:.1f} % |")
    lines += ["", "paper overhead of rotation: " + ", ".join(f"{k} {100 * v:+.0f} %"
                                                          for k, v in paper.items())]
    text = "\n".join(lines) + "\n"
    print(text)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
