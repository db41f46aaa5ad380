"""Multi-rank worker (launched by tests/test_multigpu.py under torchrun, one rank per GPU).

Checks the z-slab decomposition with NCCL halo exchange against a single-GPU run of the same
problem on the same device: PDFs bitwise identical (per-cell arithmetic does not depend on the
partition), fractions bit-exact, force/torque within 1e-12 relative (only the
allreduce order differs).  Exit code 0 = pass.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_20049_b200 as psm  # noqa: E402
import psm_inputs as pi  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    failures = []
    for (bc, Q, prec, coll, pattern) in [
            ((0, 0, 0), 19, "f64", "srt", "two_array"), ((0, 1, 1), 27, "f64", "srt", "two_array"),
            ((0, 0, 0), 19, "f32", "srt", "two_array"),
            ((2, 1, 0), 19, "f64", "srt", "two_array"),  # open x faces (A30) + y walls
            ((0, 0, 1), 27, "f64", "cumulant", "two_array"),
            ((0, 1, 0), 19, "f64", "trt", "two_array"),
            ((0, 0, 0), 19, "f64", "srt", "aa"), ((0, 1, 1), 27, "f32", "srt", "aa")]:
        # an ncclUniqueId serves exactly one communicator: a fresh one per context
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(psm.psm_nccl_get_unique_id()),
                                       dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
        nx, ny, nz = 40, 36, 16 * world + 6
        kw = dict(Q=Q, tau=0.7, bc=bc, prec=prec, sc=1, bmode=1, collision=coll, pattern=pattern)
        dsim = psm.Simulation(nx, ny, nz, rank=rank, world=world, nccl_id=nid, **kw)
        ref = psm.Simulation(nx, ny, nz, **kw)
        if bc[0] == 2:
            for s in (ref, dsim):
                s.set_open_boundary((0.03, 0.0, 0.01), 1.0)
        rho, u = pi.perturbed_flow((nz, ny, nx), 99, u0=(0.03, 0.0, 0.01))
        z0, nzl = dsim.z0, dsim.nzl
        ref.init_equilibrium(rho, u)
        dsim.init_equilibrium(np.ascontiguousarray(rho[z0:z0 + nzl]),
                              np.ascontiguousarray(u[:, z0:z0 + nzl]))
        v, tr = pi.propeller_mesh(n_blades=3, scale=0.09, n_st=8, n_pts=16, hub_seg=16)
        Q0 = pi.rotation_about([0, 1, 1], 0.3)
        # the mesh body straddles the slab boundaries; the sphere wraps periodic z when bc_z = 0
        for s in (ref, dsim):
            s.set_mesh(1, v, tr, 1, Q0, (20.0, 18.0, nz / 2 + 0.3), (0.01, 0.0, 0.02),
                       (0.0, 0.02, 0.01))
            s.set_sphere(2, 4.5, 2, np.eye(3), (10.0, 9.0, 2.0 if bc[2] == 0 else 6.0),
                         (0.0, 0.0, -1.0 / 32))
        for n in (1, 2, 5):
            ref.step(n)
            dsim.step(n)
            for b in (1, 2):
                Fr, Tr, aF, aT = ref.force_torque(b)
                Fd, Td, _, _ = dsim.force_torque(b)
                if not (np.all(np.abs(Fr - Fd) <= 1e-12 * np.maximum(np.abs(Fr), aF)) and
                        np.all(np.abs(Tr - Td) <= 1e-12 * np.maximum(np.abs(Tr), aT))):
                    failures.append(f"F/T body {b} {bc} Q{Q} {prec} {pattern}: {Fr} {Fd} {Tr} {Td}")
        if rank == 0:
            print(f"halo mode {psm.psm_halo_mode(dsim.ctx)} ({bc} Q{Q} {prec} {coll} {pattern})",
                  flush=True)
        fr = ref.pdfs()[:, z0:z0 + nzl]
        fd = dsim.pdfs()
        if not np.array_equal(fr, fd):
            failures.append(f"pdfs {bc} Q{Q} {prec} {pattern}: max diff {np.max(np.abs(fr - fd))}")
        cr = ref.fractions()[2][z0:z0 + nzl]
        if not np.array_equal(cr, dsim.fractions()[2]):
            failures.append(f"fractions {bc} Q{Q} {prec}")
        dsim.close()
        ref.close()
    # body-free (no F/T allreduce syncs the ranks): a readback straight after psm_step and a
    # state write followed by a step must see the neighbours' final peer stores (fused halo)
    for prec in ("f64", "f32"):
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(psm.psm_nccl_get_unique_id()),
                                       dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
        nx, ny, nz = 40, 36, 16 * world + 6
        kw = dict(Q=19, tau=0.7, bc=(0, 0, 0), prec=prec)
        dsim = psm.Simulation(nx, ny, nz, rank=rank, world=world, nccl_id=nid, **kw)
        ref = psm.Simulation(nx, ny, nz, **kw)
        z0, nzl = dsim.z0, dsim.nzl
        rho, u = pi.perturbed_flow((nz, ny, nx), 7, u0=(0.02, 0.01, 0.03))
        ref.init_equilibrium(rho, u)
        dsim.init_equilibrium(np.ascontiguousarray(rho[z0:z0 + nzl]),
                              np.ascontiguousarray(u[:, z0:z0 + nzl]))
        for n in (1, 3, 2):
            ref.step(n)
            dsim.step(n)
            if not np.array_equal(ref.pdfs()[:, z0:z0 + nzl], dsim.pdfs()):
                failures.append(f"body-free read after step {prec} n={n}")
        f = ref.pdfs()
        f = f * (1.0 + 0.001 * pi.uniform_pm1(8, f.size).reshape(f.shape))
        ref.write_pdfs(f)
        dsim.write_pdfs(np.ascontiguousarray(f[:, z0:z0 + nzl]))
        ref.step(3)
        dsim.step(3)
        if not np.array_equal(ref.pdfs()[:, z0:z0 + nzl], dsim.pdfs()):
            failures.append(f"body-free write then step {prec}")
        dsim.close()
        ref.close()
    ok = torch.tensor([0 if failures else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    for f in failures:
        print(f"rank {rank}: FAIL {f}", flush=True)
    dist.destroy_process_group()
    if rank == 0:
        print("multigpu", "PASS" if ok.item() == 1 else "FAIL", flush=True)
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
