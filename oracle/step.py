"""ORACLE (test infrastructure only) -- the HOME-LBM fluid step, float64.

Composes the restated reference functions into SPEC's ``fluid_update_step``
("collision -> reconstruct -> stream -> extract -> write", SPEC.md:473-477;
PAPER.md Alg. 2), plus the pieces the reference package does
not ship:

  * pull streaming f_i(x) <- f_i(x - c_i)   -- Eq. 3
  * domain BCs by ghost fill                -- SPEC.md:501-502
      periodic: wrap; inflow(u): equilibrium moments (rho=1, u, sneq=0);
      outflow: copy the nearest interior plane; wall: links that cross the
      face bounce back (the ghost layer counts as solid)
  * voxel solids: half-way bounce-back f_i(x) <- f+_opp(i)(x) for every link
    whose source x - c_i is solid ("reflect links via
    opposite-direction pairing"; ``opposite`` lattice.py:198-201); solid
    cells are reset to the rest state every step.
  * mask -> boundary lists (sorted linear indices + 27-bit link masks in the
    reference direction order, lattice.py:99-116).

State convention = the reference's array layout (moments.py:11-13):
``rho`` (nx,ny,nz), ``mom`` (3,nx,ny,nz), ``stress`` (6,nx,ny,nz) float64,
holding post-streaming (pre-collision) moments as in Alg. 2.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import codec
from . import lattice as L
from .collision import collide_moments, tau_from_viscosity
from .moments import (moments_from_distributions, neq_decompose, neq_recompose,
                      reconstruct_distributions)

FACES = ("x-", "x+", "y-", "y+", "z-", "z+")


@dataclass
class BC:
    """Per-face boundary condition.  x faces: periodic|inflow|outflow|wall;
    y/z faces: periodic|wall.  ``u_in`` is the inflow velocity."""
    x: tuple = ("periodic", "periodic")
    y: tuple = ("periodic", "periodic")
    z: tuple = ("periodic", "periodic")
    u_in: tuple = (0.0, 0.0, 0.0)

    def axis(self, a):
        return (self.x, self.y, self.z)[a]


# ---------------------------------------------------------------- padding

def _pad_axis(arr, axis, kinds, fill_lo=None, fill_hi=None):
    """Pad one grid axis (array axis ``axis``) by one ghost layer per side."""
    n = arr.shape[axis]
    idx_lo = [slice(None)] * arr.ndim
    idx_hi = [slice(None)] * arr.ndim
    lo_kind, hi_kind = kinds

    def take(i):
        s = [slice(None)] * arr.ndim
        s[axis] = slice(i, i + 1)
        return arr[tuple(s)]

    lo = take(n - 1) if lo_kind == "periodic" else take(0)
    hi = take(0) if hi_kind == "periodic" else take(n - 1)
    if lo_kind == "inflow":
        lo = np.broadcast_to(fill_lo, lo.shape).copy()
    if hi_kind == "inflow":
        hi = np.broadcast_to(fill_hi, hi.shape).copy()
    del idx_lo, idx_hi
    return np.concatenate([lo, arr, hi], axis=axis)


def pad_state(rho, mom, stress, bc: BC):
    """Stack the 10 components, add one ghost layer per face (x, then y, then z)."""
    st = np.concatenate([rho[None], mom, stress], axis=0)
    u = np.asarray(bc.u_in, dtype=np.float64)
    eq = np.concatenate([[1.0], u, [u[0] * u[0], u[0] * u[1], u[0] * u[2],
                                    u[1] * u[1], u[1] * u[2], u[2] * u[2]]])
    eq = eq.reshape(10, 1, 1, 1)
    st = _pad_axis(st, 1, bc.x, eq, eq)
    st = _pad_axis(st, 2, bc.y)
    st = _pad_axis(st, 3, bc.z)
    return st


def padded_solid(mask, bc: BC):
    """Solid flags on the ghost-padded grid (x padded first, then y, then z)."""
    m = np.asarray(mask, dtype=bool)
    if m.ndim != 3:
        raise ValueError("mask must be 3-D")

    def pad(arr, axis, kinds):
        n = arr.shape[axis]
        s_lo = [slice(None)] * 3
        s_hi = [slice(None)] * 3
        s_lo[axis] = slice(n - 1, n) if kinds[0] == "periodic" else slice(0, 1)
        s_hi[axis] = slice(0, 1) if kinds[1] == "periodic" else slice(n - 1, n)
        lo = arr[tuple(s_lo)].copy()
        hi = arr[tuple(s_hi)].copy()
        if kinds[0] != "periodic":
            lo[...] = kinds[0] == "wall"
        if kinds[1] != "periodic":
            hi[...] = kinds[1] == "wall"
        return np.concatenate([lo, arr, hi], axis=axis)

    m = pad(m, 0, bc.x)
    m = pad(m, 1, bc.y)
    m = pad(m, 2, bc.z)
    return m


def link_masks_dense(mask, bc: BC, lat=None):
    """(nx,ny,nz) uint32: bit i set iff fluid cell x has a solid source x - c_i."""
    lat = lat or L.D3Q27
    ps = padded_solid(mask, bc)
    nx, ny, nz = mask.shape
    out = np.zeros((nx, ny, nz), dtype=np.uint32)
    for i in range(1, lat.Q):
        cx, cy, cz = lat.C[i]
        src = ps[1 - cx:1 - cx + nx, 1 - cy:1 - cy + ny, 1 - cz:1 - cz + nz]
        out |= (src.astype(np.uint32) << np.uint32(i))
    out[np.asarray(mask, dtype=bool)] = 0
    return out


def boundary_lists(mask, bc: BC, lat=None):
    """(cells int64 sorted by linear index, link masks uint32) -- fluid cells
    with at least one solid pull source."""
    lm = link_masks_dense(mask, bc, lat)
    flat = lm.reshape(-1)
    cells = np.nonzero(flat)[0].astype(np.int64)
    return cells, flat[cells].astype(np.uint32)


def solid_cells(mask):
    return np.nonzero(np.asarray(mask, dtype=bool).reshape(-1))[0].astype(np.int64)


# ---------------------------------------------------------------- the step

def step_padded(padded, tau, force=None, link_solid=None, lat=None, collide=True):
    """One Alg.-2 update of a ghost-padded 10-component block.

    ``padded`` is (10, nx+2, ny+2, nz+2) in (rho, mom, stress) form; returns
    the (rho, mom, stress) of the nx*ny*nz interior.  ``link_solid`` is an
    optional (27, nx, ny, nz) bool array: True where the pull source of
    direction i is solid (half-way bounce-back replaces that population)."""
    lat = lat or L.D3Q27
    rho, mom, stress = padded[0], padded[1:4], padded[4:10]
    if collide:
        r, m, s = collide_moments(rho, mom, stress, force, tau)   # collision.py:137
    else:                                                         # streaming S alone (Alg.-1 cut)
        r, m, s = rho, mom, stress
    f = reconstruct_distributions(r, m, s, lat)                     # moments.py:64
    nx, ny, nz = (d - 2 for d in rho.shape)
    fs = np.empty((lat.Q, nx, ny, nz))
    for i in range(lat.Q):
        cx, cy, cz = lat.C[i]
        # pull: f_i(x) <- f_i(x - c_i)
        fs[i] = f[i, 1 - cx:1 - cx + nx, 1 - cy:1 - cy + ny, 1 - cz:1 - cz + nz]
    if link_solid is not None:
        inner = f[:, 1:-1, 1:-1, 1:-1]
        for i in range(1, lat.Q):
            sel = link_solid[i]
            if sel.any():
                fs[i][sel] = inner[lat.OPP[i]][sel]
    return moments_from_distributions(fs, lat)                      # moments.py:25


def fluid_step(rho, mom, stress, tau, bc: BC | None = None, force=None, mask=None, lat=None, collide=True):
    """One fluid update of the whole grid in the reference layout (``lat``: D3Q27 default);
    ``collide=False`` applies the streaming operator alone (``stream_step``)."""
    bc = bc or BC()
    lat = lat or L.D3Q27
    padded = pad_state(rho, mom, stress, bc)
    link_solid = None
    solid = None
    if mask is not None and np.any(mask) or _has_wall(bc):
        mask = np.zeros(rho.shape, dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
        lm = link_masks_dense(mask, bc, lat)
        link_solid = ((lm[None] >> np.arange(lat.Q, dtype=np.uint32)[:, None, None, None])
                      & np.uint32(1)).astype(bool)
        solid = mask
    r, m, s = step_padded(padded, tau, force, link_solid, lat, collide)
    if solid is not None and solid.any():
        r[solid] = 1.0
        m[:, solid] = 0.0
        s[:, solid] = 0.0
    return r, m, s


def stream_step(rho, mom, stress, bc: BC | None = None, mask=None, lat=None):
    """The streaming operator S alone: reconstruct the stored moments (moments.py:64-90), pull-stream
    with the same BC / bounce-back rules as ``fluid_step``, extract (moments.py:25-39); solid cells
    at rest.  A split step is S o C and an Alg.-1 step is C o S, so
    (S o C)^n o S = S o (C o S)^n relates the two storage cuts."""
    return fluid_step(rho, mom, stress, 1.0, bc, None, mask, lat, collide=False)


def alg1_step(rho, mom, stress, tau, bc: BC | None = None, force=None, mask=None, lat=None):
    """One original HOME-LBM step (Alg. 1) on post-collision moments: C o S."""
    r, m, s = stream_step(rho, mom, stress, bc, mask, lat)
    r2, m2, s2 = collide_moments(r, m, s, force, tau)
    if mask is not None and np.any(mask):
        sol = np.asarray(mask, dtype=bool)
        r2[sol] = 1.0
        m2[:, sol] = 0.0
        s2[:, sol] = 0.0
    return r2, m2, s2


def _has_wall(bc: BC):
    return any(k == "wall" for k in bc.x + bc.y + bc.z)


def run(rho, mom, stress, tau, steps, bc=None, force=None, mask=None, lat=None):
    for _ in range(steps):
        rho, mom, stress = fluid_step(rho, mom, stress, tau, bc, force, mask, lat)
    return rho, mom, stress


# ---------------------------------------------------------------- q16 path

def fluid_step_q16(words, tau, step_index, bc=None, force=None, mask=None,
                   mmin=codec.DEFAULT_MIN, mmax=codec.DEFAULT_MAX, bits=None,
                   dither=False, seed=0, x0=0, global_shape=None, lat=None):
    """Reference quantized path: decode -> float64 step -> encode.

    Dither noise is keyed by the global linear cell index; ``x0`` and
    ``global_shape`` locate a slab inside the global grid."""
    rho, mom, sneq = codec.decode_state(words, mmin, mmax, bits)
    stress = neq_recompose(rho, mom, sneq)
    r, m, s = fluid_step(rho, mom, stress, tau, bc, force, mask, lat)
    n = neq_decompose(r, m, s)
    noise = None
    if dither:
        noise = codec.dither_noise(global_cell_index(r.shape, x0, global_shape), step_index, seed)
    return codec.encode_state(r, m, n, mmin, mmax, bits, noise)


def global_cell_index(shape, x0=0, global_shape=None):
    nx, ny, nz = shape
    gy, gz = (ny, nz) if global_shape is None else global_shape[1:]
    x = np.arange(nx, dtype=np.int64)[:, None, None] + x0
    y = np.arange(ny, dtype=np.int64)[None, :, None]
    z = np.arange(nz, dtype=np.int64)[None, None, :]
    return (x * gy + y) * gz + z


# ---------------------------------------------------------------- scenes

def taylor_green(n, u0=0.05):
    """TGV initial state, sneq = 0."""
    k = 2 * np.pi / n
    x = np.arange(n)[:, None, None]
    y = np.arange(n)[None, :, None]
    z = np.arange(n)[None, None, :]
    ux = u0 * np.sin(k * x) * np.cos(k * y) * np.cos(k * z)
    uy = -u0 * np.cos(k * x) * np.sin(k * y) * np.cos(k * z)
    uz = np.zeros_like(ux + uy)
    rho = 1.0 + 3.0 * (u0 ** 2 / 16.0) * (np.cos(2 * k * x) + np.cos(2 * k * y)) * (np.cos(2 * k * z) + 2.0)
    rho = np.broadcast_to(rho, (n, n, n)).astype(np.float64)
    mom = np.stack([rho * ux, rho * uy, rho * uz])
    stress = neq_recompose(rho, mom, np.zeros((6, n, n, n)))
    return rho, mom, stress


def random_state(shape, seed=0, drho=0.1, umax=0.1, sneq=0.01):
    rng = np.random.default_rng(seed)
    rho = 1.0 + rng.uniform(-drho, drho, shape)
    mom = rho * rng.uniform(-umax, umax, (3,) + tuple(shape))
    n = rng.uniform(-sneq, sneq, (6,) + tuple(shape))
    return rho, mom, neq_recompose(rho, mom, n)
