"""Voxel solid masks for the benchmark scenes (input construction, host side).

The split scheme's boundary handling works on a voxel solid mask (the north-star variant of
the paper's surface voxelization).  These builders make
the masks of SURVEY.md §8(d) configs 3-5; the boundary lists and link masks are built on
the GPU by ``Solver.set_mask`` (csrc/hlbm_cells.cu).
"""

from __future__ import annotations

import numpy as np


def sphere_mask(dims, center, radius) -> np.ndarray:
    """Cells whose centre lies inside the sphere (voxel test at cell centres)."""
    nx, ny, nz = dims
    x = np.arange(nx)[:, None, None] - center[0]
    y = np.arange(ny)[None, :, None] - center[1]
    z = np.arange(nz)[None, None, :] - center[2]
    return ((x * x + y * y + z * z) <= radius * radius).astype(np.uint8)


def _box(m, lo, hi):
    nx, ny, nz = m.shape
    a = [max(0, int(round(l))) for l in lo]
    b = [min(n, int(round(h))) for h, n in zip(hi, (nx, ny, nz))]
    if all(bb > aa for aa, bb in zip(a, b)):
        m[a[0]:b[0], a[1]:b[1], a[2]:b[2]] = 1


def _ellipsoid(m, c, r):
    nx, ny, nz = m.shape
    x0, x1 = max(0, int(c[0] - r[0]) - 1), min(nx, int(c[0] + r[0]) + 2)
    y0, y1 = max(0, int(c[1] - r[1]) - 1), min(ny, int(c[1] + r[1]) + 2)
    z0, z1 = max(0, int(c[2] - r[2]) - 1), min(nz, int(c[2] + r[2]) + 2)
    x = (np.arange(x0, x1)[:, None, None] - c[0]) / r[0]
    y = (np.arange(y0, y1)[None, :, None] - c[1]) / r[1]
    z = (np.arange(z0, z1)[None, None, :] - c[2]) / r[2]
    m[x0:x1, y0:y1, z0:z1] |= ((x * x + y * y + z * z) <= 1.0).astype(np.uint8)


def _cylinder_y(m, c, radius, y0, y1):
    """Cylinder with axis along y (a wheel), centre (cx, cz)."""
    nx, ny, nz = m.shape
    xa, xb = max(0, int(c[0] - radius) - 1), min(nx, int(c[0] + radius) + 2)
    za, zb = max(0, int(c[1] - radius) - 1), min(nz, int(c[1] + radius) + 2)
    x = np.arange(xa, xb)[:, None] - c[0]
    z = np.arange(za, zb)[None, :] - c[1]
    disk = (x * x + z * z) <= radius * radius
    ya, yb = max(0, int(y0)), min(ny, int(y1))
    if yb > ya:
        m[xa:xb, ya:yb, za:zb] |= disk[:, None, :].astype(np.uint8)


def vehicle_mask(dims, seed=0) -> np.ndarray:
    """Seeded procedural vehicle-like obstacle (body, cabin, 4 wheels, rear wing).

    Coordinates: x streamwise, y spanwise, z vertical; the car sits on z = 0 and occupies a
    few percent of the domain."""
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    m = np.zeros(dims, dtype=np.uint8)
    L = 0.40 * nx * (1 + 0.05 * rng.uniform(-1, 1))
    W = 0.36 * ny * (1 + 0.05 * rng.uniform(-1, 1))
    H = 0.16 * nz * (1 + 0.05 * rng.uniform(-1, 1))
    x0 = 0.22 * nx
    yc = ny / 2
    clearance = 0.04 * nz
    wheel_r = 0.07 * nz
    # body: box + rounded nose / tail
    _box(m, (x0, yc - W / 2, clearance + wheel_r * 0.6), (x0 + L, yc + W / 2, clearance + wheel_r * 0.6 + H))
    _ellipsoid(m, (x0, yc, clearance + wheel_r * 0.6 + H / 2), (0.10 * L, W / 2, H / 2))
    _ellipsoid(m, (x0 + L, yc, clearance + wheel_r * 0.6 + H / 2), (0.06 * L, W / 2, H / 2))
    # cabin
    _ellipsoid(m, (x0 + 0.55 * L, yc, clearance + wheel_r * 0.6 + H), (0.25 * L, 0.40 * W, 0.55 * H))
    # wheels
    for fx in (0.18, 0.80):
        for side in (-1, 1):
            ya = yc + side * (W / 2) - (0.12 * W if side > 0 else 0.0)
            _cylinder_y(m, (x0 + fx * L, wheel_r), wheel_r, ya, ya + 0.12 * W)
    # rear wing on two struts
    zw = clearance + wheel_r * 0.6 + 1.7 * H
    _box(m, (x0 + 0.92 * L, yc - 0.45 * W, zw), (x0 + 1.02 * L, yc + 0.45 * W, zw + 0.05 * nz))
    for s in (-0.25, 0.25):
        _box(m, (x0 + 0.95 * L, yc + s * W - 1, clearance + wheel_r * 0.6 + H), (x0 + 0.97 * L, yc + s * W + 1, zw))
    return m


def turbulence_modes(n, kmin=1.0, kmax=4.0, u_rms=0.05, seed=0, dims=None) -> np.ndarray:
    """Solenoidal random Fourier modes (kx,ky,kz, ax,ay,az, phase) with kmin <= |k| <= kmax,
    scaled so that the velocity field has the requested rms."""
    rng = np.random.default_rng(seed)
    kr = int(np.ceil(kmax))
    modes = []
    for kx in range(-kr, kr + 1):
        for ky in range(-kr, kr + 1):
            for kz in range(0, kr + 1):
                if kz == 0 and (ky < 0 or (ky == 0 and kx <= 0)):
                    continue   # one of each +-k pair
                k = np.array([kx, ky, kz], dtype=np.float64)
                kn = np.linalg.norm(k)
                if kn < kmin or kn > kmax:
                    continue
                a = rng.normal(size=3)
                a -= k * (a @ k) / (kn * kn)          # solenoidal: a . k = 0
                a *= kn ** (-5.0 / 6.0)               # mild spectral slope
                modes.append([kx, ky, kz, a[0], a[1], a[2], rng.uniform(0, 2 * np.pi)])
    modes = np.array(modes, dtype=np.float64)
    # each mode contributes <sin^2> = 1/2 of |a|^2 to <|u|^2>; rms over 3 components
    e = 0.5 * np.sum(modes[:, 3:6] ** 2)
    modes[:, 3:6] *= u_rms * np.sqrt(3.0 / (2.0 * e)) if e > 0 else 0.0
    return modes


def evaluate_modes(modes, shape, origin=(0, 0, 0), global_dims=None):
    """Host evaluation of the mode sum on a box (used by tests to build oracle inputs)."""
    gd = global_dims if global_dims is not None else shape
    x = (np.arange(shape[0]) + origin[0])[:, None, None] / gd[0]
    y = (np.arange(shape[1]) + origin[1])[None, :, None] / gd[1]
    z = (np.arange(shape[2]) + origin[2])[None, None, :] / gd[2]
    u = np.zeros((3,) + tuple(shape))
    for kx, ky, kz, ax, ay, az, ph in modes:
        s = np.sin(2 * np.pi * (kx * x + ky * y + kz * z) + ph)
        u[0] += ax * s
        u[1] += ay * s
        u[2] += az * s
    return u


def voxel_surface_mesh(mask):
    """Triangulated boundary of a voxel solid: every solid-voxel face that touches a fluid voxel
    becomes two triangles on the cube [x-1/2, x+1/2]^3 (cell centres at integer coordinates).
    Gives million-triangle test meshes comparable to the paper's scanned models."""
    m = np.asarray(mask, dtype=bool)
    nx, ny, nz = m.shape
    verts = []
    faces = []
    nv = 0
    for ax in range(3):
        for sgn in (-1, 1):
            nb = np.zeros_like(m)
            sl_src = [slice(None)] * 3
            sl_dst = [slice(None)] * 3
            if sgn > 0:
                sl_dst[ax] = slice(0, m.shape[ax] - 1)
                sl_src[ax] = slice(1, None)
            else:
                sl_dst[ax] = slice(1, None)
                sl_src[ax] = slice(0, m.shape[ax] - 1)
            nb[tuple(sl_dst)] = m[tuple(sl_src)]
            exposed = m & ~nb
            idx = np.argwhere(exposed).astype(np.float64)
            if not len(idx):
                continue
            c = idx.copy()
            c[:, ax] += 0.5 * sgn
            u = [a for a in range(3) if a != ax]
            corners = []
            for du, dv in ((-0.5, -0.5), (0.5, -0.5), (0.5, 0.5), (-0.5, 0.5)):
                p = c.copy()
                p[:, u[0]] += du
                p[:, u[1]] += dv
                corners.append(p)
            q = len(idx)
            verts.append(np.concatenate(corners))          # 4q vertices: corner k of quad j at k*q + j
            j = np.arange(q)
            base = nv
            faces.append(np.stack([base + j, base + q + j, base + 2 * q + j], axis=1))
            faces.append(np.stack([base + j, base + 2 * q + j, base + 3 * q + j], axis=1))
            nv += 4 * q
    if not verts:
        return np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int32)
    return np.concatenate(verts), np.concatenate(faces).astype(np.int32)


def load_obj(path, transform=None):
    """Wavefront OBJ -> (vertices (nv, 3) float64, faces (nf, 3) int32); SPEC.md:404-407 `load_mesh`.

    Reads `v` and `f` records only (`vt` / `vn` / `o` / `g` / `s` / comments are skipped); face
    entries may be `i`, `i/t`, `i//n` or `i/t/n`, 1-based or negative (relative); polygons are fan-
    triangulated.  ``transform`` is a 3x4 (or 4x4) affine matrix applied to the vertices (lattice
    coordinates).  Malformed records raise ValueError naming the line; degenerate faces (repeated
    vertices or zero area) raise ValueError naming the face index."""
    verts, faces = [], []
    with open(path, "r") as f:
        for ln, line in enumerate(f, 1):
            s = line.split("#", 1)[0].strip()
            if not s:
                continue
            tok = s.split()
            if tok[0] == "v":
                if len(tok) < 4:
                    raise ValueError(f"{path}:{ln}: vertex record needs 3 coordinates")
                try:
                    verts.append([float(t) for t in tok[1:4]])
                except ValueError:
                    raise ValueError(f"{path}:{ln}: malformed vertex record") from None
            elif tok[0] == "f":
                if len(tok) < 4:
                    raise ValueError(f"{path}:{ln}: face record needs at least 3 vertices")
                idx = []
                for t in tok[1:]:
                    try:
                        i = int(t.split("/")[0])
                    except ValueError:
                        raise ValueError(f"{path}:{ln}: malformed face entry {t!r}") from None
                    i = i - 1 if i > 0 else len(verts) + i
                    if i < 0 or i >= len(verts) or int(t.split("/")[0]) == 0:
                        raise ValueError(f"{path}:{ln}: face index {t!r} out of range")
                    idx.append(i)
                for k in range(1, len(idx) - 1):
                    faces.append((idx[0], idx[k], idx[k + 1]))
    V = np.array(verts, dtype=np.float64).reshape(-1, 3)
    F = np.array(faces, dtype=np.int32).reshape(-1, 3)
    if transform is not None:
        T = np.asarray(transform, dtype=np.float64)
        V = V @ T[:3, :3].T + T[:3, 3]
    for fi, (a, b, c) in enumerate(F):
        if a == b or b == c or a == c or np.linalg.norm(np.cross(V[b] - V[a], V[c] - V[a])) == 0.0:
            raise ValueError(f"{path}: degenerate face {fi} (vertices {a}, {b}, {c})")
    return V, F


def save_obj(path, vertices, faces):
    """Write (vertices, faces) as a Wavefront OBJ (1-based `v` / `f` records)."""
    with open(path, "w") as f:
        for v in np.asarray(vertices, dtype=np.float64):
            f.write(f"v {float(v[0])!r} {float(v[1])!r} {float(v[2])!r}\n")
        for a, b, c in np.asarray(faces, dtype=np.int64):
            f.write(f"f {a + 1} {b + 1} {c + 1}\n")


def icosphere(center, radius, subdiv=1):
    """Closed triangle mesh of a sphere: the icosahedron's 12 vertices / 20 faces, each face split
    into 4 `subdiv` times with the new vertices pushed onto the sphere (scene geometry for the
    triangle-mesh path; 20 * 4^subdiv faces)."""
    g = (1.0 + 5 ** 0.5) / 2.0
    V = [np.array(v, dtype=np.float64) for v in
         ((-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0), (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
          (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1))]
    V = [v / np.linalg.norm(v) for v in V]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
         (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        mids = {}

        def midpoint(a, b):
            e = (a, b) if a < b else (b, a)
            if e not in mids:
                m = V[a] + V[b]
                V.append(m / np.linalg.norm(m))
                mids[e] = len(V) - 1
            return mids[e]
        nf = []
        for a, b, c in F:
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = nf
    return np.array(V) * float(radius) + np.asarray(center, dtype=np.float64), np.array(F, dtype=np.int64)


def taylor_green_fields(n, u0=0.05):
    """Taylor-Green vortex on an n^3 periodic box: (rho, u) for
    ``Solver.set_equilibrium`` -- u = u0 (sin x cos y cos z, -cos x sin y cos z, 0), k = 2 pi / n,
    with the matching pressure field in rho."""
    k = 2 * np.pi / n
    x = np.arange(n)[:, None, None]
    y = np.arange(n)[None, :, None]
    z = np.arange(n)[None, None, :]
    u = np.zeros((3, n, n, n))
    u[0] = u0 * np.sin(k * x) * np.cos(k * y) * np.cos(k * z)
    u[1] = -u0 * np.cos(k * x) * np.sin(k * y) * np.cos(k * z)
    rho = 1.0 + 3.0 * (u0 ** 2 / 16.0) * (np.cos(2 * k * x) + np.cos(2 * k * y)) * (np.cos(2 * k * z) + 2.0)
    return np.broadcast_to(rho, (n, n, n)).copy(), u
