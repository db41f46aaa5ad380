#!/usr/bin/env python
"""Benchmark of the B200 PSM hot path (arXiv 2502.20049): MLUPS and % of the HBM roofline.

Default workload: BASELINE config c5 (weak scaling) — D3Q19 PSM fp32, 512^3 periodic cells per
GPU stacked along z (global 512 x 512 x 512N), one CROR-like counter-rotating rotor pair per GPU
(triangle meshes of ~0.6 M faces each, voxelised once, remapped every step at s=1), SRT + SC1,
weighted B (Eq.(6)), two-array pull streaming, NCCL halo exchange for N>1.  A "step" is one pass
of the whole hot path: closed-form pose advance, fraction remap (GPU), fused PSM stream-collide
with force/torque partials (GPU), halo exchange (N>1), and the per-call force/torque reduction.
Other workloads: --config c4 (moving sphere r=64, 512^3), c4aa, c4f64, c3f64.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config c5w]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ...
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "MLUPS per GPU and % of HBM roofline at 1/2/4/8 B200 (PSM moving geometry)"
UNIT = "MLUPS"

WORKLOADS = {
    # c5 weak scaling: 512^3 per GPU stacked in z, one CROR-like counter-rotating rotor pair per
    # GPU (front 12 blades tip 200 at x=200, +Omega; rear 10 blades tip 180 at x=330, -Omega;
    # Omega = 0.05/220 rad/step; ~0.6 M faces each; s=1), D3Q19 fp32 SRT+SC1, weighted B
    "c5w": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.55, rotors=True, s=1,
                omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1,
                desc="c5 weak: D3Q19 PSM fp32, 512^3 per GPU, CROR-like counter-rotating rotor "
                     "pair per GPU (12+10 blades, ~1.1 M faces, s=1, remapped every step), SC1, "
                     "weighted B"),
    # the same at the paper's precision (fp64): the default bench line
    "c5w64": dict(nx=512, ny=512, nz=512, Q=19, prec="f64", tau=0.55, rotors=True, s=1,
                  omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1,
                  desc="c5 weak, fp64: D3Q19 PSM fp64 (the paper's precision), 512^3 per GPU, "
                       "CROR-like counter-rotating rotor pair per GPU (12+10 blades, ~1.1 M "
                       "faces, s=1, remapped every step), SC1, weighted B"),
    # the paper's own performance configuration: D3Q19, cumulant (reading A32), AA
    # in-place streaming, SC1, fp64, prescribed rotation — on the c5w rotor pair
    "c5wpap": dict(nx=512, ny=512, nz=512, Q=19, prec="f64", tau=0.55, rotors=True, s=1,
                   omega=0.05 / 220.0, pattern="aa", sc=1, bmode=1, collision="cumulant",
                   desc="c5 weak, the paper's operator: D3Q19 cumulant AA fp64 PSM, 512^3 per "
                        "GPU, CROR-like counter-rotating rotor pair per GPU (s=1, remapped every "
                        "step), SC1, weighted B"),
    # c5w as an application run: inflow U = 0.05 at x = 0, pressure outflow at
    # x = nx-1 (reading A30), flow starting from rest
    "c5app": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.55, rotors=True, s=1,
                  omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1, bc=(2, 0, 0),
                  open_bc=((0.05, 0.0, 0.0), 1.0),
                  desc="c5 weak + open boundaries: c5w with velocity inflow U=0.05 at x=0 and "
                       "pressure outflow rho=1 at x=nx-1 (A30), y/z periodic"),
    # c5 strong scaling: the whole ~1e9-cell CROR-like domain split over the GPUs (rotor axis x:
    # front 12 blades tip 220 at x=760, +Omega; rear 10 blades tip 200 at x=900, -Omega)
    "c5s": dict(nx=2048, ny=704, nz=704, Q=19, prec="f32", tau=0.55, rotors=True, s=1,
                omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1, strong=True,
                rotor_x=(760.0, 900.0), rotor_tip=(220.0, 200.0),
                desc="c5 strong: D3Q19 PSM fp32, 2048x704x704 = 1.015e9 cells split over the "
                     "GPUs, CROR-like counter-rotating rotor pair (12+10 blades, s=1, remapped "
                     "every step), SC1, weighted B"),
    "c4": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.6, r=64.0, s=1,
               v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1,
               desc="c4: D3Q19 PSM fp32 512^3/GPU periodic, sphere r=64 translating "
                    "v=(1/32,0,0), s=1, remapped every step, SC1, weighted B"),
    # NEXT-row workloads: TRT fluid operator, two-way coupled sphere, paper-literal R2 mapping
    "c4trt": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.6, r=64.0, s=1,
                  v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1, collision="trt",
                  desc="c4 TRT: D3Q19 PSM fp32 512^3, moving sphere r=64, s=1, TRT (magic 3/16)"),
    "c4dyn": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.6, r=64.0, s=1,
                  v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1,
                  dynamic=(2.0, -1e-5),
                  desc="c4 two-way coupled: D3Q19 PSM fp32 512^3, sphere r=64 (density ratio 2, "
                       "gravity -1e-5 x) integrated from its own force/torque every step"),
    "c5wr2": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.55, rotors=True, s=1,
                  omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1, mapping="R2",
                  desc="c5 weak with the paper-literal centre-only mapping R2 (A12)"),
    "c4aa": dict(nx=512, ny=512, nz=512, Q=19, prec="f32", tau=0.6, r=64.0, s=1,
                 v=(1.0 / 32.0, 0.0, 0.0), pattern="aa", sc=1, bmode=1,
                 desc="c4 (AA pattern): D3Q19 PSM fp32 512^3, moving sphere r=64, s=1"),
    "c4f64": dict(nx=512, ny=512, nz=512, Q=19, prec="f64", tau=0.6, r=64.0, s=1,
                  v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1,
                  desc="c4 fp64: D3Q19 PSM fp64 512^3, moving sphere r=64, s=1"),
    # the paper's performance operator (cumulant) on D3Q27 with the c3-shaped geometry
    "c3cum": dict(nx=256, ny=256, nz=256, Q=27, prec="f64", tau=0.6, r=48.0, s=1,
                  v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1,
                  collision="cumulant",
                  desc="c3-shaped, cumulant: D3Q27 PSM fp64 256^3, moving sphere r=48, s=1"),
    "c5w27": dict(nx=512, ny=512, nz=512, Q=27, prec="f32", tau=0.55, rotors=True, s=1,
                  omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1,
                  desc="c5 weak, D3Q27: D3Q27 PSM fp32 SRT, 512^3 per GPU, CROR-like rotor pair "
                       "per GPU, s=1, SC1, weighted B"),
    "c5wcum": dict(nx=512, ny=512, nz=512, Q=27, prec="f32", tau=0.55, rotors=True, s=1,
                   omega=0.05 / 220.0, pattern="two_array", sc=1, bmode=1, collision="cumulant",
                   desc="c5 weak, cumulant: D3Q27 PSM fp32, 512^3 per GPU, CROR-like rotor pair "
                        "per GPU, s=1, SC1, weighted B"),
    "c3f64": dict(nx=256, ny=256, nz=256, Q=27, prec="f64", tau=0.6, r=48.0, s=1,
                  v=(1.0 / 32.0, 0.0, 0.0), pattern="two_array", sc=1, bmode=1,
                  desc="c3-shaped: D3Q27 PSM fp64 256^3, moving sphere r=48, s=1"),
}


def bytes_per_update(Q: int, S: int) -> int:
    """Algorithmic bytes per cell update: one read + one write per population, 2*Q*S
    (the paper's roofline model)."""
    return 2 * Q * S


def load_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def profiles_traffic(workload: str):
    """dram bytes per collide launch from the committed ncu summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------------ CPU oracle leg ---
def oracle_sample(wl: dict, steps, budget_s: float, seed: int, warmup: int = 0,
                  threads: int | None = None):
    """Time the CPU oracle (as it stands) on a bounded sub-box of the same workload: same
    stencil/tau/operator, bodies scaled with the box, moving, remapped every step.  `warmup`
    untimed steps first; steps=None sizes the timed steps to about `budget_s` seconds."""
    cores = threads or os.cpu_count() or 1
    # torchrun pins OMP_NUM_THREADS=1 per rank; the sample runs on rank 0 alone and may use the
    # whole host (set before the oracle library, and with it libgomp, is loaded)
    if "oracle" not in sys.modules:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import ctypes
    import oracle
    import psm_inputs as pi
    oracle.lib()
    # the thread count of this sample (libgomp's runtime call; the oracle is unchanged)
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(cores))
    # oracle throughput is ~0.6-1 MLUPS per core for D3Q19; size the box for the budget
    est = 0.6e6 * cores * (19.0 / wl["Q"])
    per_step = budget_s / max(1, steps or 10)
    cells = max(32 ** 3, min(256 ** 3, int(per_step * est)))
    n = max(32, int(round(cells ** (1 / 3) / 16)) * 16)
    scale = n / wl["nx"]
    o = oracle.Oracle(n, n, n, wl["Q"], wl["tau"], (0, 0, 0), wl["sc"], wl["bmode"])
    o.set_collision(wl.get("collision", "srt"))
    rho, u = pi.perturbed_flow((n, n, n), seed, u0=(0.02, 0.0, 0.0), u_amp=0.001)
    o.init_equilibrium(rho, u)
    if wl.get("rotors"):
        bodies = []
        for k, (nbl, tip, xc) in enumerate(((12, 200.0, 200.0), (10, 180.0, 330.0))):
            v, t = pi.propeller_mesh(n_blades=nbl, scale=tip / 110.0 * scale, n_st=16,
                                     n_pts=24, hub_seg=32)
            o.set_mesh(k + 1, v, t, wl["s"])
            w = (wl["omega"] / scale * (1 if k == 0 else -1), 0.0, 0.0)
            bodies.append((k + 1, (xc * scale, n / 2, n / 2), w))
        what = "CROR-like rotor pair (12+10 blades, coarse meshes)"
    else:
        o.set_sphere(1, max(2.0, wl["r"] * scale), wl["s"])
        bodies = [(1, None, None)]
        what = f"sphere r={max(2.0, wl['r'] * scale):g}"

    def one(k):
        for bid, pos, w in bodies:
            if pos is None:
                o.set_pose(1, np.eye(3), (n / 2 + k * wl["v"][0], n / 2, n / 2), wl["v"])
            else:
                Qk, _ = oracle.pose_advance(np.eye(3), pos, (0, 0, 0), w, k, [n] * 3, [1] * 3)
                o.set_pose(bid, Qk, pos, (0, 0, 0), w)
        o.map()
        o.step(1)

    k = 0
    t_w = time.perf_counter()
    for _ in range(max(warmup, 0 if steps else 1)):
        one(k)
        k += 1
    if steps is None:  # size the timed run from the measured warm-up step
        t1 = (time.perf_counter() - t_w) / max(1, k)
        steps = int(min(200, max(2, budget_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(steps):
        one(k)
        k += 1
    dt = time.perf_counter() - t0
    mlups = n ** 3 * steps / dt / 1e6
    sample = (f"oracle fp64 on a {n}^3 periodic sub-box of {wl['desc'].split(':')[0]} "
              f"({what}, scaled by {scale:g}, moving, remap+collide every step), "
              f"{steps} timed steps after {k - steps} untimed, {dt:.1f} s")
    return {"value": mlups, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
            "ms_per_step": 1e3 * dt / steps}


def run_reference(args, wl, rank, world):
    if rank != 0:
        return 0
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    cb = oracle_sample(wl, max(1, args.steps), per_step_budget * args.steps, 7,
                       warmup=args.warmup)
    ms = cb.pop("ms_per_step")
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if wl.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(wl, world),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def workload_config(wl: dict, world: int) -> dict:
    nx, ny = wl["nx"], wl["ny"]
    nzg = wl["nz"] if wl.get("strong") else wl["nz"] * world
    return {"workload": wl["desc"], "grid": [nx, ny, nzg],
            "cells_per_gpu": nx * ny * nzg // world, "global_cells": nx * ny * nzg,
            "stencil": f"D3Q{wl['Q']}", "pattern": wl["pattern"],
            "parallelism": f"z-slab x{world}" + (" + NCCL halo" if world > 1 else ""),
            "l2": "inputs larger than L2 (PDF arrays >> 126 MB)"}


_MESHES = {}


def _rotor_mesh(blades: int, tip: float):
    """The CROR-like rotor meshes (~0.6 M faces), generated once per process: at N GPUs every
    rank holds all 2N rotors, which share two shapes."""
    import psm_inputs as pi
    key = (blades, tip)
    if key not in _MESHES:
        _MESHES[key] = pi.propeller_mesh(n_blades=blades, scale=tip / 110.0, n_st=200, n_pts=128,
                                         hub_seg=256)
    return _MESHES[key]


def build_workload(psm, wl: dict, rank: int, world: int, nccl_id=None):
    """The bench's simulation: the grid of `wl` (nz per GPU stacked in z), rest fluid, and the
    bodies (a CROR-like rotor pair or one moving sphere per GPU slab; every rank holds every
    body so the force/torque allreduce is consistent).  Returns (sim, body_poses, nbodies, S)."""
    import psm_inputs as pi
    nx, ny = wl["nx"], wl["ny"]
    nzg = wl["nz"] if wl.get("strong") else wl["nz"] * world
    S = 8 if wl["prec"] == "f64" else 4
    sim = psm.Simulation(nx, ny, nzg, Q=wl["Q"], tau=wl["tau"], bc=wl.get("bc", (0, 0, 0)),
                         prec=wl["prec"], pattern=wl["pattern"], sc=wl["sc"], bmode=wl["bmode"],
                         rank=rank, world=world, nccl_id=nccl_id,
                         collision=wl.get("collision", "srt"))
    if wl.get("open_bc"):
        sim.set_open_boundary(*wl["open_bc"])
    sim.init_equilibrium(None, None)
    nbodies = 0
    body_poses = []  # (Q0, t0, v, w) per body, in id order
    for r in range(1 if wl.get("strong") else world):
        zc = (nzg * r) // world + ((nzg * (r + 1)) // world - (nzg * r) // world) / 2
        if wl.get("strong"):
            zc = nzg / 2
        if wl.get("rotors"):
            for k, front in enumerate((True, False)):
                tip = wl.get("rotor_tip", (200.0, 180.0))[k]
                v, t = _rotor_mesh(12 if front else 10, tip)
                w = (wl["omega"] if front else -wl["omega"], 0.0, 0.0)
                tpos = (wl.get("rotor_x", (200.0, 330.0))[k], ny / 2, zc)
                sim.set_mesh(1 + 2 * r + k, v, t, wl["s"], np.eye(3), tpos, (0, 0, 0), w,
                             mapping=wl.get("mapping", "R1"))
                body_poses.append((np.eye(3), tpos, (0.0, 0.0, 0.0), w))
                nbodies += 1
        else:
            sim.set_sphere(1 + r, wl["r"], wl["s"], np.eye(3), (nx / 2, ny / 2, zc), wl["v"])
            body_poses.append((np.eye(3), (nx / 2, ny / 2, zc), wl["v"], (0.0, 0.0, 0.0)))
            nbodies += 1
            if wl.get("dynamic"):
                # two-way coupled (NEXT rank 1): density ratio rho_s/rho_f, gravity along -x
                ratio, gx = wl["dynamic"]
                vol = 4.0 / 3.0 * np.pi * wl["r"] ** 3
                m = ratio * vol
                sim.set_dynamics(1 + r, m, 0.4 * m * wl["r"] ** 2 * np.eye(3),
                                 ext_force=((m - vol) * gx, 0.0, 0.0))
    return sim, body_poses, nbodies, S


# ---------------------------------------------------------------------------- GPU leg -----
def _json_out():
    """The driver reads ONE JSON line from stdout; libraries (NCCL prints its version banner)
    must not write there.  Route fd 1 to stderr and keep a private handle for the result."""
    saved = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(saved, "w")


OUT = None


def emit(line: dict):
    OUT.write(json.dumps(line) + "\n")
    OUT.flush()


def main():
    global OUT
    OUT = _json_out()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5w64", choices=sorted(WORKLOADS))
    ap.add_argument("--extra", default=None,
                    help="comma list of further workloads measured in the same run, each under "
                         "its own key (default with c5w64: c5w -> 'f32', c5wpap -> "
                         "'paper_config'); 'none' for none")
    ap.add_argument("--reps", type=int, default=5,
                    help="timed repetitions of exactly K steps; value = their median")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--s", type=int, default=None, help="override the super-sampling exponent")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.config])
    if args.s is not None:
        wl["s"] = args.s
        wl["desc"] += f" [s overridden to {args.s}]"

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, wl, rank, world)

    import torch
    import paper_2502_20049_b200 as psm
    import psm_inputs as pi

    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(psm.psm_nccl_get_unique_id()),
                                       dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())

    # further workloads measured in the same run, each under its own key: by default the fp32
    # twin of the fp64 line ("f32") and the paper's own performance configuration ("paper_config":
    # D3Q19 cumulant AA fp64) on the same rotor-pair geometry
    if args.extra is not None:
        extras = [e for e in args.extra.split(",") if e and e != "none"]
    else:
        extras = ["c5w", "c5wpap"] if args.config == "c5w64" else []
    extras = [e for e in extras if e != args.config]
    stream_gbs = stream_copy_gbs(torch) if rank == 0 else None
    res = measure(psm, torch, dist, wl, args, rank, world, local, nccl_id, e2e=not args.no_e2e,
                  config_name=args.config)
    extra_res = []
    for extra in extras:
        nccl_id2 = None
        if world > 1:
            idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(psm.psm_nccl_get_unique_id()),
                                           dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nccl_id2 = bytes(idt.cpu().numpy().tobytes())
        extra_res.append(measure(psm, torch, dist, dict(WORKLOADS[extra]), args, rank, world,
                                 local, nccl_id2, e2e=False, config_name=extra))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(wl, None, 12.0, 7)
        cpu.pop("ms_per_step", None)
        one = oracle_sample(wl, None, 8.0, 7, threads=1)
        cpu["single_thread"] = {"value": one["value"], "unit": UNIT, "cores": 1,
                                "sample": one["sample"]}
        cpu["cpu_model"] = cpu_model()

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["mlups"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "strong" if wl.get("strong") else "weak",
            "vs_baseline": None, "dtype": wl["prec"], "data": "synthetic",
            "config": res["config"],
            "mlups_per_gpu": res["mlups"] / world,
            "reps": res["reps"],
            "roofline_frac_step": res["step_frac"],
            "roofline": roofline_block(res, stream_gbs),
            "phases_ms": res["phases_ms"],
            "nvlink_rank0": res["nvlink"],
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "e2e": res["e2e"],
            "cpu_baseline": cpu,
        }
        for er in extra_res:
            key = {"c5w": "f32", "c5wpap": "paper_config"}.get(er["name"], er["name"])
            line[key] = {
                "config": er["name"], "workload": er["config"]["workload"],
                "dtype": er["prec"], "pattern": er["config"]["pattern"],
                "value": er["mlups"], "unit": UNIT, "ms_per_step": er["ms_per_step"],
                "reps": er["reps"], "roofline_frac_step": er["step_frac"],
                "roofline": roofline_block(er, stream_gbs),
                "phases_ms": er["phases_ms"], "gpu_launches": er["launches"],
                "clocks": er["clocks"]}
        emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


NOMINAL_GBS = 8000.0  # B200 HBM3e nominal (north_star "~8 TB/s")


def roofline_block(res, stream_gbs):
    peak, peak_src = load_peak()
    a = res["achieved"]
    out = {"bound": "hbm", "kernel": "k_collide (fused PSM stream-collide)",
           "achieved": a, "peak": peak, "unit": "GB/s", "frac": (a / peak) if a else None,
           "traffic": profiles_traffic(res["name"]), "bytes_per_update": res["bpu"],
           "peak_source": peak_src, "avg_launch_ms": res["avg_launch_ms"],
           "launches_timed": res["launches_timed"],
           # the same achieved bandwidth against the other two denominators SURVEY §8(d) names
           "peaks": {"measured_json": peak, "stream_copy_same_run": stream_gbs,
                     "nominal": NOMINAL_GBS},
           "frac_vs_stream_copy_same_run": (a / stream_gbs) if (a and stream_gbs) else None,
           "frac_vs_nominal": (a / NOMINAL_GBS) if a else None,
           "step_frac_vs": {"measured_json": res["step_gbs"] / peak,
                            "stream_copy_same_run": (res["step_gbs"] / stream_gbs)
                            if stream_gbs else None,
                            "nominal": res["step_gbs"] / NOMINAL_GBS}}
    return out


def stream_copy_gbs(torch, nbytes=4 << 30, reps=10):
    """Same-run STREAM-copy bandwidth (the paper's roofline practice): a
    device-to-device copy of a 4 GiB buffer, read + write bytes over the best of `reps` launches
    timed with CUDA events on the current stream."""
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1)
    best = None
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    del a, b
    torch.cuda.empty_cache()
    return 2 * nbytes / (best / 1e3) / 1e9


def nvlink_bytes(index: int):
    """(tx, rx) NVLink data bytes of GPU `index` since the driver started, from NVML's
    throughput counters (KiB; aggregate over links), or None where unsupported."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        fids = [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
        tot = [0, 0]
        for link in range(18):
            vals = nv.nvmlDeviceGetFieldValues(h, [(f, link) for f in fids])
            for k, v in enumerate(vals):
                if v.nvmlReturn == 0:
                    tot[k] += int(v.value.ullVal)
        return tot[0] * 1024, tot[1] * 1024
    except Exception:
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def measure(psm, torch, dist, wl, args, rank, world, local, nccl_id, e2e=True, config_name=""):
    """Build the workload, warm up, time `args.reps` repetitions of exactly `args.steps` steps
    (each bracketed by barrier + synchronize, device time on the library's stream, max over
    ranks) and, optionally, the end-to-end loop through the public API."""
    import math
    import psm_inputs as pi
    sim, body_poses, nbodies, S = build_workload(psm, wl, rank, world, nccl_id)
    nx, ny = wl["nx"], wl["ny"]
    nzg = wl["nz"] if wl.get("strong") else wl["nz"] * world
    z0, nzl = sim.z0, sim.nzl
    stream = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sim.step(max(3, args.warmup))
    barrier()
    l0 = sim.launches
    sim.profile(True)
    times = []
    nvl0 = nvlink_bytes(local) if world > 1 else None
    with ClockSampler(local) as clk:
        for _ in range(max(1, args.reps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            sim.step(args.steps)
            e1.record(stream)
            barrier()
            ms = e0.elapsed_time(e1)
            if dist is not None:
                t = torch.tensor([ms], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            times.append(ms)
    nvl1 = nvlink_bytes(local) if world > 1 else None
    sim.profile(False)
    prof = sim.profile_read()
    reps = max(1, args.reps)
    nvlink = None
    if nvl0 and nvl1:
        nsteps = reps * args.steps
        # halo volume per rank and step: the c_z = +-1 populations of one nx*ny plane to each
        # of the two z neighbours (5 of 19 / 9 of 27 directions)
        qz = 5 if wl["Q"] == 19 else 9
        nvlink = {"tx_bytes_per_step": (nvl1[0] - nvl0[0]) / nsteps,
                  "rx_bytes_per_step": (nvl1[1] - nvl0[1]) / nsteps,
                  "halo_bytes_per_step_expected": 2 * qz * nx * ny * S,
                  "source": "NVML NVLink data throughput counters of this rank's GPU "
                            "around the timed repetitions"}
    launches = (sim.launches - l0) // reps
    ms_med = float(np.median(times))
    cells_local = nx * ny * nzl
    cells_total = nx * ny * nzg
    mlups = cells_total * args.steps / (ms_med / 1e3) / 1e6
    bpu = bytes_per_update(wl["Q"], S)
    coll_ms, coll_n = prof["collide"]
    avg = coll_ms / max(1, coll_n)
    achieved = bpu * cells_local / (avg / 1e3) / 1e9 if coll_n else None
    step_gbs = bpu * cells_local * args.steps / (ms_med / 1e3) / 1e9

    # end-to-end through the public API with host buffers (the coupled-simulation loop a user
    # runs): every step the host computes each body's pose in closed form and hands it to
    # psm_set_body (H2D, 144 B per body: pose + velocity), runs psm_step(1), and reads every
    # body's force/torque back (D2H, 96 B per body + the 8 B error word).  The one-off field
    # upload (psm_init_equilibrium from pinned host rho/u) and readback (psm_read_velocity) are
    # timed separately and reported as setup_ms / readback_ms.
    e2e_line = None
    if e2e:
        shape = (nzl, ny, nx)
        rho_h = torch.ones(shape, dtype=torch.float64).pin_memory().numpy()
        u_h = torch.zeros((3,) + shape, dtype=torch.float64).pin_memory().numpy()
        u_h[0] = 0.02
        barrier()
        t_a = time.perf_counter()
        sim.init_equilibrium(rho_h, u_h)
        barrier()
        t_b = time.perf_counter()
        for k in range(args.steps):
            for b, (Q0, t0, v, w) in enumerate(body_poses):
                if wl.get("dynamic"):
                    break  # the library integrates two-way coupled bodies itself
                ang = k * math.sqrt(w[0] ** 2 + w[1] ** 2 + w[2] ** 2)
                Qk = pi.rotation_about(w, ang) @ Q0 if ang else Q0
                tk = tuple(t0[a] + k * v[a] for a in range(3))
                sim.set_pose(1 + b, Qk, tk, v, w)
            sim.step(1)
            for b in range(nbodies):
                sim.force_torque(1 + b)
        barrier()
        t_c = time.perf_counter()
        rho_o = np.empty(shape)
        u_o = np.empty((3,) + shape)
        psm.psm_read_velocity(sim.ctx, rho_o, u_o)
        barrier()
        t_d = time.perf_counter()
        dt = t_c - t_b
        if dist is not None:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e_line = {"value": cells_total * args.steps / dt / 1e6, "unit": UNIT,
                    "h2d_bytes_per_step": 144 * nbodies, "d2h_bytes_per_step": 96 * nbodies + 8,
                    "ms_per_step": dt / args.steps * 1e3,
                    "setup_ms": (t_b - t_a) * 1e3,
                    "setup_h2d_bytes": int(rho_h.nbytes + u_h.nbytes),
                    "readback_ms": (t_d - t_c) * 1e3,
                    "readback_d2h_bytes": int(rho_o.nbytes + u_o.nbytes),
                    "what": "K x [host closed-form pose -> psm_set_body (each body), "
                            "psm_step(1), psm_force_torque (each body)], wall clock, max over "
                            "ranks"}
    halo_cfg = {}
    if world > 1:
        hm = psm.psm_halo_mode(sim.ctx)
        halo_cfg = {"parallelism": f"z-slab x{world} + " + (
            "fused halo (k_collide stores into the neighbours' ghost planes over NVLink)"
            if hm == 2 else "NCCL send/recv halo")}
    if dist is not None:
        dist.barrier()
    sim.close()
    del sim
    torch.cuda.empty_cache()
    return {"name": config_name, "prec": wl["prec"], "mlups": mlups,
            "ms_per_step": ms_med / args.steps,
            "reps": {"n": len(times), "ms_per_step": [t / args.steps for t in times],
                     "value_is": "median"},
            "step_frac": step_gbs / load_peak()[0], "step_gbs": step_gbs,
            "achieved": achieved, "bpu": bpu, "avg_launch_ms": avg, "launches_timed": coll_n,
            "phases_ms": {k: v[0] / (max(1, args.steps) * reps) for k, v in prof.items()},
            "launches": launches, "clocks": clk.summary(), "e2e": e2e_line, "nvlink": nvlink,
            "config": dict(workload_config(wl, world), **halo_cfg)}


if __name__ == "__main__":
    sys.exit(main())
