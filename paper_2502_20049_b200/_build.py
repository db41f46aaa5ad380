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


STAMP = LIB + ".flags"  # the extra nvcc flags the library was built with (PSM_NVCC_EXTRA)


def _extra() -> str:
    return os.environ.get("PSM_NVCC_EXTRA", "").strip()


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    built = open(STAMP).read().strip() if os.path.exists(STAMP) else ""
    if built != _extra():  # e.g. a PSM_BOUNDS_CHECK build must not be reused silently
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(
        os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "psm.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          extra_flags: str | None = None) -> str:
    """Compile libpsm.so in-tree.  out / extra_flags: a variant library for kernel-tuning
    experiments (loaded with PSM_LIB=<path>), never the default one."""
    if out is not None:
        return _build_to(out, extra_flags or "", verbose)
    if not force and not needs_build():
        return LIB
    _build_to(LIB, _extra(), verbose)
    with open(STAMP, "w") as fh:
        fh.write(_extra() + "\n")
    return LIB


def _build_to(lib: str, extra: str, verbose: bool) -> str:
    from concurrent.futures import ThreadPoolExecutor
    nccl = nccl_dir()
    nvcc = os.environ.get("NVCC", "nvcc")
    # extra: diagnostics only, e.g. -DPSM_BOUNDS_CHECK (device-side bounds asserts)
    flags = [nvcc, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
             "-Xcompiler", "-fPIC,-fopenmp,-O2", "-Xptxas", "-warn-spills",
             "-I", os.path.join(ROOT, "include"), "-I", CSRC,
             "-I", os.path.join(nccl, "include")] + extra.split()
    objdir = os.path.join(HERE, "build", os.path.basename(lib))
    os.makedirs(objdir, exist_ok=True)
    objs, cmds = [], []
    for src in sources():  # one nvcc per translation unit, in parallel
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmds.append(flags + ["-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        results = list(ex.map(run, cmds))
    for cmd, r in zip(cmds, results):
        if r.stderr:
            sys.stderr.write(r.stderr)
        if r.returncode != 0:
            raise subprocess.CalledProcessError(r.returncode, cmd, r.stdout, r.stderr)
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib + ".tmp"] + \
        objs + ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                "-Xlinker", "-rpath," + os.path.join(nccl, "lib"), "-lgomp"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
