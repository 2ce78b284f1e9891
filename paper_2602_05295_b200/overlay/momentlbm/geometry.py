"""momentlbm.geometry -- obstacle geometry of the reference package's layout (pkg/src/momentlbm/
__init__.py:1-9), installed next to the reference modules by
``paper_2602_05295_b200.dropin.install()``.

  TriangleMesh / SolidState / SurfaceMask
  load_mesh(path, transform)                SPEC.md:404-407 (Wavefront OBJ, v / f records)
  link_intersect(x, c_i, tri)               SPEC.md:408-412 (earliest hit on [x, x - c_i])
  voxelize_surface(mesh, dims)              SPEC.md:413-416 (conservative AABB-triangle overlap + 1-cell dilation)

The step itself never calls these on the host: ``Solver.set_mesh`` finds every cut link once on
the GPU (hlbm_mesh.cu, the same Moller-Trumbore test and tie rules as ``link_intersect``), and the
candidate nodes it tests are the bounding boxes grown by one cell -- a superset of
``voxelize_surface``.  They are the SPEC's host-side API for inspecting a scene.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from paper_2602_05295_b200.geometry import load_obj

__all__ = ["TriangleMesh", "SolidState", "load_mesh", "link_intersect", "voxelize_surface"]

EPS = 1e-9        # inclusive barycentric edges and t > EPS (hlbm_mesh.cu kEps)
DET_EPS = 1e-12   # |det| below this: the link is parallel to the triangle -> no hit


@dataclass
class SolidState:
    """Rigid motion of an obstacle: linear velocity v (lattice units / step),
    angular velocity omega (rad / step) about `center`."""
    v: Sequence[float] = (0.0, 0.0, 0.0)
    omega: Sequence[float] = (0.0, 0.0, 0.0)
    center: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class TriangleMesh:
    """Vertices (nv, 3) float64 in lattice coordinates, faces (nf, 3) int."""
    vertices: np.ndarray
    faces: np.ndarray
    state: SolidState = field(default_factory=SolidState)

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        self.faces = np.ascontiguousarray(self.faces, dtype=np.int64).reshape(-1, 3)
        if self.faces.size and (self.faces.min() < 0 or self.faces.max() >= len(self.vertices)):
            raise ValueError("face index out of range")

    def __iter__(self):   # (vertices, faces, motion) -- the obstacle form momentlbm.solver accepts
        yield self.vertices
        yield self.faces
        yield {"velocity": tuple(self.state.v), "omega": tuple(self.state.omega),
               "center": tuple(self.state.center)}

    def __len__(self):
        return 3

    def __getitem__(self, k):
        return list(iter(self))[k]


def load_mesh(path, transform=None, state: Optional[SolidState] = None) -> TriangleMesh:
    """Wavefront OBJ (v / f records) with an optional 3x4 / 4x4 affine transform; malformed records
    raise ValueError naming the line, degenerate faces naming the face index."""
    V, F = load_obj(path, transform)
    return TriangleMesh(V, F, state or SolidState())


def link_intersect(x, c, tri):
    """Earliest hit of the pull link x -> x - c (parameter t in (0, 1]) with triangle `tri`
    ((3, 3) vertices): (t, p = x - t c) or None.  Parallel / coplanar links never hit."""
    o = np.asarray(x, dtype=np.float64)
    d = -np.asarray(c, dtype=np.float64)
    v0, v1, v2 = (np.asarray(v, dtype=np.float64) for v in tri)
    e1, e2 = v1 - v0, v2 - v0
    pvec = np.cross(d, e2)
    det = float(e1 @ pvec)
    if not abs(det) >= DET_EPS:
        return None
    inv = 1.0 / det
    tvec = o - v0
    u = float(tvec @ pvec) * inv
    qvec = np.cross(tvec, e1)
    v = float(d @ qvec) * inv
    t = float(e2 @ qvec) * inv
    if u >= -EPS and u <= 1.0 + EPS and v >= -EPS and u + v <= 1.0 + EPS and t > EPS and t <= 1.0 + EPS:
        return t, o + t * d
    return None


def _tri_box_overlap(center, h, v0, v1, v2):
    """Separating-axis test of triangles (arrays (n, 3)) against the cubes center +- h (n, 3)."""
    a, b, c = v0 - center, v1 - center, v2 - center
    ok = np.ones(len(center), dtype=bool)
    # the cube's face normals
    for k in range(3):
        lo = np.minimum(np.minimum(a[:, k], b[:, k]), c[:, k])
        hi = np.maximum(np.maximum(a[:, k], b[:, k]), c[:, k])
        ok &= (lo <= h) & (hi >= -h)
    # the triangle's normal
    nrm = np.cross(b - a, c - a)
    r = h * np.abs(nrm).sum(axis=1)
    s = (nrm * a).sum(axis=1)
    ok &= np.abs(s) <= r + 1e-12
    # the nine edge cross products
    for e in (b - a, c - b, a - c):
        for k in range(3):
            ax = np.zeros_like(e)
            ax[:, (k + 1) % 3] = -e[:, (k + 2) % 3]
            ax[:, (k + 2) % 3] = e[:, (k + 1) % 3]
            pa, pb, pc = (ax * a).sum(1), (ax * b).sum(1), (ax * c).sum(1)
            rr = h * np.abs(ax).sum(axis=1)
            ok &= ~((np.minimum(np.minimum(pa, pb), pc) > rr + 1e-12) | (np.maximum(np.maximum(pa, pb), pc) < -rr - 1e-12))
    return ok


def voxelize_surface(mesh: TriangleMesh, dims, dilate: int = 1) -> np.ndarray:
    """SurfaceMask: bool (nx, ny, nz), a node marked iff some triangle
    overlaps its unit cell [x - 1/2, x + 1/2]^3 (conservative separating-axis AABB-triangle test),
    then dilated by `dilate` cells -- a superset of every node whose links can hit the mesh."""
    nx, ny, nz = (int(d) for d in dims)
    mask = np.zeros((nx, ny, nz), dtype=bool)
    V, F = mesh.vertices, mesh.faces
    for a, b, c in F:
        p = V[[a, b, c]]
        lo = np.maximum(np.floor(p.min(axis=0) - 0.5).astype(int), 0)
        hi = np.minimum(np.ceil(p.max(axis=0) + 0.5).astype(int), np.array([nx, ny, nz]) - 1)
        if np.any(hi < lo):
            continue
        g = np.stack(np.meshgrid(*(np.arange(l, h + 1) for l, h in zip(lo, hi)), indexing="ij"), -1).reshape(-1, 3)
        n = len(g)
        hit = _tri_box_overlap(g.astype(np.float64), 0.5 + 1e-9, np.repeat(p[None, 0], n, 0),
                               np.repeat(p[None, 1], n, 0), np.repeat(p[None, 2], n, 0))
        sel = g[hit]
        mask[sel[:, 0], sel[:, 1], sel[:, 2]] = True
    for _ in range(dilate):   # separable 3x3x3 box dilation (diagonal links reach corner cells)
        for ax in range(3):
            m = mask.copy()
            for sh in (-1, 1):
                src = [slice(None)] * 3
                dst = [slice(None)] * 3
                src[ax] = slice(max(0, -sh), mask.shape[ax] - max(0, sh))
                dst[ax] = slice(max(0, sh), mask.shape[ax] - max(0, -sh))
                m[tuple(dst)] |= mask[tuple(src)]
            mask = m
    return mask
