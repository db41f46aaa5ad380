"""Deterministic closed triangle meshes (body frame, lattice units, no randomness).

Input generators only: vertices/triangles consumed identically by the oracle and the CUDA path.
All meshes are watertight (every edge shared by exactly two triangles) and consistently
oriented (outward normals), so ray parity classifies them (reading A15).
"""
from __future__ import annotations

import numpy as np


def box_mesh(lo, hi):
    """Axis-aligned box [lo, hi] as 8 vertices / 12 outward-oriented triangles."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    v = np.array([[lo[0] if i & 1 == 0 else hi[0], lo[1] if i & 2 == 0 else hi[1],
                   lo[2] if i & 4 == 0 else hi[2]] for i in range(8)])
    t = np.array([
        [0, 2, 1], [1, 2, 3],  # z = lo (normal -z)
        [4, 5, 6], [5, 7, 6],  # z = hi
        [0, 1, 4], [1, 5, 4],  # y = lo
        [2, 6, 3], [3, 6, 7],  # y = hi
        [0, 4, 2], [2, 4, 6],  # x = lo
        [1, 3, 5], [3, 7, 5],  # x = hi
    ], np.int32)
    return v, t


def uv_sphere_mesh(r: float, n_lat: int = 16, n_lon: int = 32):
    """Closed UV sphere of radius r centred at the origin."""
    verts = [[0.0, 0.0, r]]
    for i in range(1, n_lat):
        th = np.pi * i / n_lat
        for j in range(n_lon):
            ph = 2 * np.pi * j / n_lon
            verts.append([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph),
                          r * np.cos(th)])
    verts.append([0.0, 0.0, -r])
    tris = []
    south = len(verts) - 1

    def ring(i, j):
        return 1 + (i - 1) * n_lon + (j % n_lon)

    for j in range(n_lon):
        tris.append([0, ring(1, j), ring(1, j + 1)])
    for i in range(1, n_lat - 1):
        for j in range(n_lon):
            a, b = ring(i, j), ring(i, j + 1)
            c, d = ring(i + 1, j), ring(i + 1, j + 1)
            tris.append([a, c, d])
            tris.append([a, d, b])
    for j in range(n_lon):
        tris.append([south, ring(n_lat - 1, j + 1), ring(n_lat - 1, j)])
    return np.array(verts, np.float64), np.array(tris, np.int32)


def cylinder_mesh(radius: float, x0: float, x1: float, n_seg: int = 48):
    """Closed cylinder along x from x0 to x1 (hub)."""
    ang = 2 * np.pi * np.arange(n_seg) / n_seg
    ring0 = np.stack([np.full(n_seg, x0), radius * np.cos(ang), radius * np.sin(ang)], 1)
    ring1 = np.stack([np.full(n_seg, x1), radius * np.cos(ang), radius * np.sin(ang)], 1)
    verts = np.concatenate([ring0, ring1, [[x0, 0, 0]], [[x1, 0, 0]]])
    c0, c1 = 2 * n_seg, 2 * n_seg + 1
    tris = []
    for j in range(n_seg):
        a, b = j, (j + 1) % n_seg
        tris.append([a, n_seg + b, n_seg + a])  # outward (radial) normals
        tris.append([a, b, n_seg + b])
        tris.append([c0, b, a])
        tris.append([c1, n_seg + a, n_seg + b])
    return verts, np.array(tris, np.int32)


def _naca_section(n_pts: int, thickness: float, chord: float):
    """Closed symmetric airfoil polygon (NACA 4-digit thickness law, closed trailing edge),
    n_pts points, counter-clockwise in (chordwise, normal), centred at mid-chord."""
    half = n_pts // 2
    beta = np.linspace(0.0, np.pi, half + 1)
    xs = 0.5 * (1 - np.cos(beta))  # cosine spacing 0..1
    t = thickness / chord
    yt = 5 * t * (0.2969 * np.sqrt(xs) - 0.1260 * xs - 0.3516 * xs ** 2 + 0.2843 * xs ** 3
                  - 0.1036 * xs ** 4)
    upper = np.stack([xs, yt], 1)[::-1]          # TE -> LE on top
    lower = np.stack([xs, -yt], 1)[1:-1]         # LE -> TE on bottom (skip duplicate LE/TE)
    pts = np.concatenate([upper, lower])
    pts[:, 0] = (pts[:, 0] - 0.5) * chord
    pts[:, 1] = pts[:, 1] * chord
    return pts  # shape (n_pts, 2)


def _blade(r0, r1, n_st, n_pts, chord0, chord1, pitch0, pitch1, thick, phi, sweep=0.0):
    """One blade: closed tube of airfoil sections from radius r0 to r1 with end caps."""
    er = np.array([0.0, np.cos(phi), np.sin(phi)])
    et = np.array([0.0, -np.sin(phi), np.cos(phi)])
    ex = np.array([1.0, 0.0, 0.0])
    f = np.arange(n_st) / (n_st - 1)
    r = r0 + (r1 - r0) * f
    ch = chord0 + (chord1 - chord0) * f
    b = np.deg2rad(pitch0 + (pitch1 - pitch0) * f)
    verts = np.empty((n_st, n_pts, 3))
    for k in range(n_st):
        sec = _naca_section(n_pts, thick, ch[k])
        dc = np.cos(b[k]) * ex + np.sin(b[k]) * et     # chordwise direction
        dn = -np.sin(b[k]) * ex + np.cos(b[k]) * et    # thickness direction
        verts[k] = r[k] * er + sec[:, :1] * dc + sec[:, 1:] * dn + sweep * f[k] * ex
    verts = verts.reshape(-1, 3)
    m = n_pts
    caps = np.stack([verts[:m].mean(0), verts[(n_st - 1) * m:].mean(0)])
    base = len(verts)
    k = np.arange(n_st - 1)[:, None]
    j = np.arange(m)[None, :]
    a = k * m + j
    bb = k * m + (j + 1) % m
    c = (k + 1) * m + j
    d = (k + 1) * m + (j + 1) % m
    side = np.concatenate([np.stack([a, bb, d], -1).reshape(-1, 3),
                           np.stack([a, d, c], -1).reshape(-1, 3)])
    jj = np.arange(m)
    cap0 = np.stack([np.full(m, base), (jj + 1) % m, jj], -1)
    cap1 = np.stack([np.full(m, base + 1), (n_st - 1) * m + jj, (n_st - 1) * m + (jj + 1) % m], -1)
    return np.concatenate([verts, caps]), np.concatenate([side, cap0, cap1]).astype(np.int64)


def _orient_outward(verts, tris):
    """Flip every triangle of a closed component if its signed volume is negative."""
    v0, v1, v2 = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    vol = np.einsum("ij,ij->i", v0, np.cross(v1, v2)).sum() / 6.0
    if vol < 0:
        tris = tris[:, [0, 2, 1]]
    return tris


def propeller_mesh(n_blades=6, hub_r=12.0, hub_len=48.0, r_tip=110.0, chord=(28.0, 12.0),
                   pitch=(55.0, 20.0), thick=4.0, n_st=64, n_pts=64, hub_seg=96, scale=1.0,
                   sweep=0.0, gap=1.0):
    """Synthetic propeller about the x axis, origin at the hub centre (BASELINE c3/c5 recipe).

    Disjoint closed components (hub + blades separated by `gap` cells) so the union is a
    valid parity solid.  scale multiplies every length.  Faces ~ n_blades*2*n_st*n_pts.
    """
    parts_v, parts_t, off = [], [], 0
    hv, ht = cylinder_mesh(hub_r * scale, -0.5 * hub_len * scale, 0.5 * hub_len * scale,
                           hub_seg)
    ht = _orient_outward(hv, ht.astype(np.int64))
    parts_v.append(hv)
    parts_t.append(ht)
    off += len(hv)
    for k in range(n_blades):
        phi = 2 * np.pi * k / n_blades
        bv, bt = _blade((hub_r + gap) * scale, r_tip * scale, n_st, n_pts, chord[0] * scale,
                        chord[1] * scale, pitch[0], pitch[1], thick * scale, phi, sweep * scale)
        bt = _orient_outward(bv, bt)
        parts_v.append(bv)
        parts_t.append(bt + off)
        off += len(bv)
    return np.concatenate(parts_v), np.concatenate(parts_t).astype(np.int32)
