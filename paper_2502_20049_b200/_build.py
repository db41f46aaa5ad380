"""Build the product library libpsm.so (sm_100a CUDA kernels + C ABI) in-tree with nvcc.

No fast-math: IEEE division/sqrt and denormals are kept (the fraction remap is bit-exact with
the method definition, reading A14); explicit __fma_rn/__dmul_rn fix the operation
order where it matters.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libpsm.so")
CSRC = os.path.join(HERE, "csrc")


def nccl_dir() -> str:
    import nvidia.nccl  # torch-bundled NCCL 2.28 (same library torch.distributed loads)
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(
        nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(
        os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "psm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nccl = nccl_dir()
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC,-fopenmp,-O2", "-shared", "-Xptxas", "-warn-spills",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-I", os.path.join(nccl, "include"),
           "-o", LIB + ".tmp"] + sources() + [
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nccl, "lib"), "-lgomp"]
    extra = os.environ.get("PSM_NVCC_EXTRA")  # tuning experiments only, e.g. -DPSM_CUM32_BLOCKS=4
    if extra:
        cmd[1:1] = extra.split()
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
