"""N>1 z-slab decomposition on real GPUs (>= 2 visible): the fused peer-store halo (default when
the GPUs can reach each other) and the NCCL send/recv halo (PSM_HALO=nccl) must both reproduce
the single-GPU run bitwise (tests/mp_worker.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("halo", ["auto", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_slabs_bitwise_identical_to_single_gpu(world, halo):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ)
    if halo == "nccl":
        env["PSM_HALO"] = "nccl"
    else:
        env.pop("PSM_HALO", None)
    port = 29611 + world * 2 + (halo == "nccl")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "multigpu PASS" in r.stdout
    if halo == "nccl":
        assert "halo mode 1" in r.stdout and "halo mode 2" not in r.stdout
    elif all(torch.cuda.can_device_access_peer(0, k) for k in range(1, world)):
        # fused for every two-array case; the AA pattern exchanges its ghost planes over NCCL
        two_array = [l for l in r.stdout.splitlines() if "halo mode" in l and "two_array" in l]
        assert two_array and all("halo mode 2" in l for l in two_array), r.stdout[-2000:]
