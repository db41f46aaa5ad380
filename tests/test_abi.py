"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/psm.h
declares, and host-side validation returns the documented error codes (no GPU needed: these
calls fail before touching the device)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2502_20049_b200 as psm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "psm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psm_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = psm.load()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(psm.EXPORTED)


def test_struct_layouts_match_header():
    # psm_options: 4 int32 + 3 double + 2 int32 + 2 pointers + int32 (+4 pad) + double
    assert C.sizeof(psm.psm_grid) == 3 * 8 + 3 * 4 + 4
    assert C.sizeof(psm.psm_options) == 16 + 24 + 8 + 16 + 8 + 8
    assert C.sizeof(psm.psm_pose) == 12 * 8
    assert C.sizeof(psm.psm_velocity) == 6 * 8
    assert C.sizeof(psm.psm_shape) == 8 + 8 + 8 + 8 + 8 + 8 + 8
    assert psm.load().psm_nccl_id_bytes() == 128


def _opts(**kw):
    o = dict(prec=psm.PSM_F64, pattern=psm.PSM_TWO_ARRAY, sc=1, bmode=1, rank=0, world=1)
    o.update(kw)
    return psm.psm_options(o["prec"], o["pattern"], o["sc"], o["bmode"],
                           (C.c_double * 3)(*o.get("force", (0, 0, 0))), o["rank"], o["world"],
                           None, None, o.get("coll", 0), o.get("magic", 0.1875))


def _grid(nx=8, ny=8, nz=8, bc=(0, 0, 0)):
    return psm.psm_grid(nx, ny, nz, (C.c_int32 * 3)(*bc))


@pytest.mark.parametrize("tau", [0.5, 0.2, float("nan"), float("inf")])
def test_create_rejects_bad_tau(tau):
    with pytest.raises(psm.PSMError) as e:
        psm.psm_create(_grid(), 19, tau, _opts())
    assert e.value.code == psm.PSM_E_ARG


def test_create_validation_codes():
    cases = [
        (dict(), _grid(0, 8, 8), 19, psm.PSM_E_ARG),
        (dict(), _grid(), 15, psm.PSM_E_ARG),
        (dict(sc=4), _grid(), 19, psm.PSM_E_ARG),
        (dict(prec=7), _grid(), 19, psm.PSM_E_ARG),
        (dict(pattern=psm.PSM_AA, force=(1e-5, 0, 0)), _grid(), 19, psm.PSM_E_UNSUPPORTED),
        (dict(world=2, rank=0), _grid(), 19, psm.PSM_E_UNSUPPORTED if False else psm.PSM_E_ARG),
        (dict(world=2, rank=2), _grid(), 19, psm.PSM_E_ARG),
        (dict(), _grid(8, 8, 8, (0, 3, 0)), 19, psm.PSM_E_ARG),
        (dict(coll=3), _grid(), 27, psm.PSM_E_ARG),
        (dict(coll=1, magic=0.0), _grid(), 19, psm.PSM_E_ARG),
        (dict(), _grid(8, 8, 8, (0, 2, 0)), 19, psm.PSM_E_UNSUPPORTED),  # open faces: x only
        (dict(), _grid(2, 8, 8, (2, 0, 0)), 19, psm.PSM_E_UNSUPPORTED),  # nx >= 3
        (dict(pattern=psm.PSM_AA), _grid(8, 8, 8, (2, 0, 0)), 19, psm.PSM_E_UNSUPPORTED),
        # AA across ranks needs a periodic x axis
        (dict(pattern=psm.PSM_AA, world=2, rank=0), _grid(8, 8, 8, (1, 0, 0)), 19,
         psm.PSM_E_UNSUPPORTED),
    ]
    for kw, g, q, code in cases:
        with pytest.raises(psm.PSMError) as e:
            psm.psm_create(g, q, 0.8, _opts(**kw))
        assert e.value.code == code, (kw, e.value)


def test_open_boundary_setter_codes():
    ctx = psm.psm_create(_grid(8, 8, 8), 19, 0.7, _opts())
    try:
        with pytest.raises(psm.PSMError) as e:
            psm.psm_set_open_boundary(ctx, (0.01, 0, 0), 1.0)
        assert e.value.code == psm.PSM_E_UNSUPPORTED  # bc[0] is periodic
    finally:
        psm.psm_destroy(ctx)
    ctx = psm.psm_create(_grid(8, 8, 8, (2, 1, 0)), 19, 0.7, _opts())
    try:
        psm.psm_set_open_boundary(ctx, (0.01, 0, 0), 1.0)
        for u, r in (((0.01, 0, 0), 0.0), ((float("nan"), 0, 0), 1.0), ((0, 0, 0), float("inf"))):
            with pytest.raises(psm.PSMError) as e:
                psm.psm_set_open_boundary(ctx, u, r)
            assert e.value.code == psm.PSM_E_ARG
    finally:
        psm.psm_destroy(ctx)


def test_create_succeeds_host_only_and_reports_layout():
    ctx = psm.psm_create(_grid(40, 12, 10), 19, 0.7, _opts())
    try:
        z0, nzl = psm.psm_local_extent(ctx)
        assert (z0, nzl) == (0, 10)
        nbytes = psm.psm_required_bytes(ctx)
        # two fp64 PDF arrays dominate: 2 * 19 * N * 8
        assert nbytes >= 2 * 19 * 40 * 12 * 10 * 8
    finally:
        psm.psm_destroy(ctx)


def test_simulation_refuses_to_run_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        psm.Simulation(8, 8, 8)


@pytest.mark.parametrize("s", [0, 1, 2])
def test_product_voxelizer_matches_oracle_bit_exact(s):
    """The library's row-binned voxelizer (csrc/voxelize.cpp) and the oracle's plain per-row
    one implement reading A15 independently; their geometry fields must agree bit for bit."""
    import oracle
    import psm_inputs as pi
    for v, t in (pi.propeller_mesh(n_blades=5, scale=0.12, n_st=10, n_pts=20, hub_seg=20),
                 pi.uv_sphere_mesh(4.3, 12, 24), pi.box_mesh([-2.5, -1.0, -3.0], [2.0, 3.0, 1.5])):
        o1, b1 = psm.psm_voxelize(v, t, s)
        o2, b2 = oracle.voxelize(v, t, s)
        assert np.array_equal(o1, o2)
        assert b1.shape == b2.shape and np.array_equal(b1, b2)
        assert b1.sum() > 0


def test_voxelize_rejects_open_mesh():
    import psm_inputs as pi
    v, t = pi.box_mesh([0, 0, 0], [1, 1, 1])
    with pytest.raises(psm.PSMError) as e:
        psm.psm_voxelize(v, t[:-1], 1)
    assert e.value.code == psm.PSM_E_MESH
    t2 = t.copy()
    t2[0, 0] = 99
    with pytest.raises(psm.PSMError) as e:
        psm.psm_voxelize(v, t2, 1)
    assert e.value.code == psm.PSM_E_MESH


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """sizeof and field offsets of every ABI struct as gcc sees include/psm.h == the ctypes
    binding's (catches a header change the binding did not follow)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    checks = {
        "psm_grid": ["nx", "bc"], "psm_options": ["body_force", "rank", "cuda_stream",
                                                  "collision", "trt_magic"],
        "psm_shape": ["radius", "verts", "tris", "mapping"], "psm_pose": ["t"],
        "psm_velocity": ["omega"],
        "psm_dynamics": ["inertia", "ext_torque", "added_mass", "added_inertia"],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "psm.h"', "int main(void) {"]
    for st, fields in checks.items():
        lines.append(f'  printf("{st} %zu\\n", sizeof({st}));')
        for f in fields:
            lines.append(f'  printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for st, fields in checks.items():
        cls = getattr(psm, st)
        assert int(out[st]) == C.sizeof(cls), st
        for f in fields:
            assert int(out[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)


def test_size_limits_are_checked_host_side():
    """Maximum sizes: a local slab beyond 32-bit in-plane indexing (2^31 cells per direction
    plane set; the limit is per rank) is rejected at psm_create with PSM_E_ARG; the largest
    bench grid (c5 strong, 1.015e9 cells) fits one rank."""
    with pytest.raises(psm.PSMError) as e:
        psm.psm_create(_grid(2048, 2048, 600), 19, 0.6, _opts(prec=psm.PSM_F32))
    assert e.value.code == psm.PSM_E_ARG
    ctx = psm.psm_create(_grid(2048, 704, 704), 19, 0.55, _opts(prec=psm.PSM_F32))
    try:
        assert psm.psm_required_bytes(ctx) > 150e9  # two fp32 D3Q19 arrays of 1.015e9 cells
    finally:
        psm.psm_destroy(ctx)
