"""Host emulation (numpy, no GPU) of the fp32 sub-sample arithmetic of the mesh band pass
(psm_map_common.cuh, mesh_count8_t): sample si0 of an 8-sample chunk is transformed in fp64,
split into base = floor(f0) and the fraction; the other seven are fraction - 1/2 plus the rotated
lattice offsets in fp32, rounded with the magic-number add.  The kernel's exactness argument is
that whenever the fp32 value lies farther than kTol = 1e-5 from a half-integer, its rounding
equals floor() of the exact coordinate (error < 2e-6 cells).  Checked here against the exact
coordinate in extended precision for random rotations, poses and cells, s = 1, 2, 3; the
fallback (samples within kTol of a face) must be rare."""
import numpy as np
import pytest

K_MAGIC = np.float32(12582912.0)
K_TOL = np.float32(1e-5)


def _rot(rng):
    a = rng.normal(size=3)
    a /= np.linalg.norm(a)
    th = rng.uniform(0, 2 * np.pi)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


def _chunk_check(s, near_face, tol=K_TOL):
    """(mismatches among 'safe' samples, fallbacks, samples) over random chunks; near_face:
    tiny rotations of a pose whose sub-samples sit on geometry-cell faces (the values then land
    within ~1e-5 of half-integers, where fp32 rounding can flip)"""
    rng = np.random.default_rng(11 + s + 100 * near_face)
    n = 1 << s
    h = 1.0 / n
    ld = np.longdouble
    mism = fallback = total = 0
    for trial in range(40):
        if near_face:
            Q = _rot_small(rng, rng.uniform(1e-7, 3e-6))
            t = np.floor(rng.uniform(0, 512, size=3)) + h / 2
        else:
            Q = _rot(rng)
            t = rng.uniform(0, 512, size=3)
        o = np.floor(rng.uniform(-300, -100, size=3))
        cells = rng.integers(0, 512, size=(4000, 3))
        si0 = 8 * rng.integers(0, max(1, n ** 3 // 8), size=4000)
        gy0 = (si0 >> s) & (n - 1)
        gz0 = si0 >> (2 * s)
        p0 = np.stack([cells[:, 0] + 0.5 * h, cells[:, 1] + (gy0 + 0.5) * h,
                       cells[:, 2] + (gz0 + 0.5) * h], axis=1)
        # sample si0 in fp64 (the kernel's exact A14 transform), then base and fraction
        d0 = p0 - t
        q0 = d0 @ Q  # q_a = sum_b Q[b, a] d_b  (Q^T d)
        f0 = (q0 - o) * n
        base = np.floor(f0)
        rh = ((f0 - base).astype(np.float32) - np.float32(0.5)).astype(np.float32)
        Qf = Q.astype(np.float32)
        for j in range(1, 8):
            dg = np.array([j & (n - 1), (j >> s) & (n - 1), j >> (2 * s)])
            # fp32: v = rh + dgx*Q[0, a] + dgy*Q[1, a] + dgz*Q[2, a]  (each step rounded)
            v = rh.copy()
            for b in range(3):
                if dg[b]:
                    v = (v + np.float32(dg[b]) * Qf[b]).astype(np.float32)
            tm = (v + K_MAGIC).astype(np.float32)
            i = (tm - K_MAGIC).astype(np.float32)
            fr = (v - i).astype(np.float32)
            safe = np.all(np.abs(fr) < np.float32(0.5) - tol, axis=1)
            g_fast = base + i.astype(np.float64)
            # exact coordinate of sample j in extended precision
            pj = p0.astype(ld) + (dg * h).astype(ld)
            fj = ((pj - t.astype(ld)) @ Q.astype(ld) - o.astype(ld)) * ld(n)
            g_exact = np.floor(fj).astype(np.float64)
            ok = np.all(g_fast == g_exact, axis=1)
            mism += int(np.sum(safe & ~ok))
            fallback += int(np.sum(~safe))
            total += len(safe)
    return mism, fallback, total


def _rot_small(rng, th):
    a = rng.normal(size=3)
    a /= np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


@pytest.mark.parametrize("s", [1, 2, 3])
def test_fp32_chunk_rounding_matches_exact_floor(s):
    mism, fallback, total = _chunk_check(s, near_face=False)
    assert mism == 0
    assert fallback / total < 1e-3, fallback / total


@pytest.mark.parametrize("s", [1, 2, 3])
def test_fp32_chunk_rounding_near_faces_needs_the_tolerance(s):
    """Sub-samples within ~1e-5 of faces: with kTol = 1e-5 no sample is misrounded (they take
    the exact fallback); with no tolerance some are — the fallback is what makes it exact."""
    mism, fallback, total = _chunk_check(s, near_face=True)
    assert mism == 0 and fallback > 0
    mism0, _, _ = _chunk_check(s, near_face=True, tol=np.float32(0.0))
    assert mism0 > 0
