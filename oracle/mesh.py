"""ORACLE (test infrastructure only) -- triangle-mesh solid coupling, float64.

The reference ships no geometry module; this restates the SPEC/PAPER contract:
  * link-triangle intersection: barycentric (Moller-Trumbore) ray-triangle test with
    eps = 1e-9 inclusive edges, earliest t wins, ties broken by the lowest triangle index
    (SPEC.md:406-412, 431-433); a link parallel to the triangle plane never hits
    ("parallel link coplanar with triangle -> no hit").
  * the pull link of direction i at node x is the segment x -> x - c_i (the population
    streamed into x, Eq. 3); a hit at parameter t in (0, 1] gives the
    intersection point p = x - t c_i.
  * boundary moments at p (Eq. 8): rho_p = rho_x,
    u_p = v + omega x (p - center), S_p = u_p u_p + (S_x - u_x u_x), evaluated from the
    post-collision moments of x; f_i(x) <- h_i(rho_p, u_p, S_p) (Eq. 7) replaces the streamed
    population (Alg. 1; Alg. 3 correction Delta f_i = f_i(p) - f_i(x - c_i)).
  * force on the solid by momentum exchange of the corrections: Delta P = -Delta f_i c_i,
    torque = sum (p - center) x Delta P.

All arithmetic below is written out operation by operation (no np.cross / np.dot) so the
CUDA preprocessing, which uses the same order without FMA contraction, reproduces it bit for
bit.
"""

from __future__ import annotations

import numpy as np

from . import lattice as L
from .collision import collide_moments
from .moments import moments_from_distributions, reconstruct_distributions

EPS = 1e-9
DET_EPS = 1e-12


def cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def dot(a, b):
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def segment_triangle(o, d, v0, v1, v2):
    """Parameter t of the hit of o + t d (0 < t <= 1) with triangle (v0,v1,v2), or None.

    Vectorised over leading axes: every argument is a 3-tuple of arrays; returns (hit, t)."""
    e1 = sub(v1, v0)
    e2 = sub(v2, v0)
    pvec = cross(d, e2)
    det = dot(e1, pvec)
    ok = np.abs(det) >= DET_EPS
    inv = 1.0 / np.where(ok, det, 1.0)
    tvec = sub(o, v0)
    u = dot(tvec, pvec) * inv
    qvec = cross(tvec, e1)
    v = dot(d, qvec) * inv
    t = dot(e2, qvec) * inv
    hit = ok & (u >= -EPS) & (u <= 1.0 + EPS) & (v >= -EPS) & ((u + v) <= 1.0 + EPS) & (t > EPS) & (t <= 1.0 + EPS)
    return hit, t


def cut_links(vertices, faces, dims, lat=None):
    """Earliest hit per (node, direction) of every pull link x -> x - c_i (directions of ``lat``:
    D3Q27 by default, D3Q19 tests its 18 links only).

    Returns (cells int64 sorted, masks uint32, t float64 (n, 27) with NaN where uncut,
    tri int64 (n, 27) with -1 where uncut)."""
    lat = lat or L.D3Q27
    V = np.asarray(vertices, dtype=np.float64)
    F = np.asarray(faces, dtype=np.int64)
    nx, ny, nz = dims
    best_t = {}
    best_tri = {}
    for k, (a, b, c) in enumerate(F):
        p0, p1, p2 = V[a], V[b], V[c]
        lo = np.floor(np.minimum(np.minimum(p0, p1), p2)).astype(np.int64) - 1
        hi = np.ceil(np.maximum(np.maximum(p0, p1), p2)).astype(np.int64) + 1
        lo = np.maximum(lo, 0)
        hi = np.minimum(hi, np.array(dims) - 1)
        if np.any(hi < lo):
            continue
        xs = np.arange(lo[0], hi[0] + 1)
        ys = np.arange(lo[1], hi[1] + 1)
        zs = np.arange(lo[2], hi[2] + 1)
        X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
        X, Y, Z = X.ravel(), Y.ravel(), Z.ravel()
        o = (X.astype(np.float64), Y.astype(np.float64), Z.astype(np.float64))
        for i in range(1, lat.Q):
            cx, cy, cz = (float(-v) for v in lat.C[i])
            d = (np.full(X.shape, cx), np.full(X.shape, cy), np.full(X.shape, cz))
            hit, t = segment_triangle(o, d, tuple(p0), tuple(p1), tuple(p2))
            for j in np.nonzero(hit)[0]:
                cell = (int(X[j]) * ny + int(Y[j])) * nz + int(Z[j])
                key = (cell, i)
                tj = float(t[j])
                if key not in best_t or tj < best_t[key] or (tj == best_t[key] and k < best_tri[key]):
                    best_t[key] = tj
                    best_tri[key] = k
    cells = np.array(sorted({c for c, _ in best_t}), dtype=np.int64)
    index = {c: n for n, c in enumerate(cells.tolist())}
    masks = np.zeros(len(cells), dtype=np.uint32)
    tt = np.full((len(cells), 27), np.nan)
    tri = np.full((len(cells), 27), -1, dtype=np.int64)
    for (c, i), tv in best_t.items():
        n = index[c]
        masks[n] |= np.uint32(1 << i)
        tt[n, i] = tv
        tri[n, i] = best_tri[(c, i)]
    return cells, masks, tt, tri


def step_with_mesh(rho, mom, stress, tau, cells, t, solid=None, force=None, lat=None, bc=None):
    """One fluid step with the Eq.-8 boundary populations on cut links (``lat``: D3Q27 default, or
    D3Q19).  ``bc`` (oracle.step.BC, default periodic): domain faces; links into a wall face take
    the half-way bounce-back population, which wins over a mesh hit on the same link.

    ``solid`` = (v, omega, center) of the rigid body (zero by default).  Returns
    (rho, mom, stress, F_solid, T_solid)."""
    nx, ny, nz = rho.shape
    v, om, cen = (np.zeros(3), np.zeros(3), np.zeros(3)) if solid is None else (np.asarray(a, float) for a in solid)
    lat = lat or L.D3Q27
    wall = None
    if bc is None:
        r, m, s = collide_moments(rho, mom, stress, force, tau)                # collision.py:137
        f = reconstruct_distributions(r, m, s, lat)                              # moments.py:64
        fs = np.stack([np.roll(f[i], shift=tuple(lat.C[i]), axis=(0, 1, 2)) for i in range(lat.Q)])
    else:
        from . import step as OS
        padded = OS.pad_state(rho, mom, stress, bc)
        rp, mp, sp_ = collide_moments(padded[0], padded[1:4], padded[4:10], force, tau)
        fpad = reconstruct_distributions(rp, mp, sp_, lat)
        fs = np.stack([fpad[i, 1 - cx:1 - cx + nx, 1 - cy:1 - cy + ny, 1 - cz:1 - cz + nz]
                       for i, (cx, cy, cz) in enumerate(lat.C)])
        f = fpad[:, 1:-1, 1:-1, 1:-1]
        r, m, s = rp[1:-1, 1:-1, 1:-1], mp[:, 1:-1, 1:-1, 1:-1], sp_[:, 1:-1, 1:-1, 1:-1]
        wall = OS.link_masks_dense(np.zeros((nx, ny, nz), dtype=bool), bc, lat)
        for i in range(1, lat.Q):
            sel = ((wall >> np.uint32(i)) & np.uint32(1)).astype(bool)
            if sel.any():
                fs[i][sel] = f[lat.OPP[i]][sel]
    Fs = np.zeros(3)
    Ts = np.zeros(3)
    for n, cell in enumerate(cells.tolist()):
        x, rem = divmod(cell, ny * nz)
        y, z = divmod(rem, nz)
        rx = r[x, y, z]
        ux = m[:, x, y, z] / rx
        sx = s[:, x, y, z] / rx
        for i in range(1, lat.Q):
            if not np.isfinite(t[n, i]):
                continue
            if wall is not None and (int(wall[x, y, z]) >> i) & 1:
                continue                                   # the wall wins: bounce-back already set
            c = lat.C[i].astype(np.float64)
            p = np.array([x, y, z], dtype=np.float64) - t[n, i] * c
            up = v + np.cross(om, p - cen)
            # S_p = u_p u_p + (S_x - u_x u_x)   (Eq. 8), Voigt order xx xy xz yy yz zz
            pairs = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))
            sp = np.array([up[a] * up[b] + (sx[k] - ux[a] * ux[b]) for k, (a, b) in enumerate(pairs)])
            fp = reconstruct_distributions(np.array([rx]), (rx * up)[:, None], (rx * sp)[:, None], lat)[i, 0]
            df = fp - fs[i, x, y, z]
            fs[i, x, y, z] = fp
            dP = -df * c
            Fs += dP
            Ts += np.cross(p - cen, dP)
    r2, m2, s2 = moments_from_distributions(fs, lat)                            # moments.py:25
    return r2, m2, s2, Fs, Ts


def icosphere(center, radius, subdiv=1):
    """Closed triangle mesh of a sphere (test geometry)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
             (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [np.array(v, dtype=np.float64) / np.linalg.norm(v) for v in verts]
    for _ in range(subdiv):
        cache = {}
        new_faces = []

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            new_faces += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = new_faces
    V = np.array(verts) * radius + np.asarray(center, dtype=np.float64)
    return V, np.array(faces, dtype=np.int64)
