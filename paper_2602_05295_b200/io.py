"""On-disk formats of the solver: checkpoint / resume and logs.

  packed-buffer dump  magic 'HLBMPK01', uint32 dims[3], uint32 C, uint32 bits[C],
                      float64 min[C], float64 max[C], int64 step, then node-major words
                      (5 little-endian u32 per node for the 16-bit state)     -- SPEC.md:381
  snapshot            magic 'HLBMSN01', int64 step, uint32 dims[3], uint32 C=10,
                      uint32 precision (0 fp32, 1 q16), then node-major float32
                      (rho, rho u_xyz, rho S xx,xy,xz,yy,yz,zz)                -- SPEC.md:510
  raw state           magic 'HLBMRS01', int64 step, uint32 dims[3], uint32 NC, uint32 precision,
                      then the solver's internal 32-bit state, component-major: an exact,
                      bit-for-bit resume point
  StepStats CSV       step, t_fluid_ms, t_copy_ms, t_solid_ms, mass, momentum_x/y/z, max_u,
                      saturation_0..9                                              -- SPEC.md:531
  vorticity PGM       binary P5 of omega_z = d u_y/dx - d u_x/dy (central differences) on one z
                      slice, linear map of [-range, range] onto 0..255          -- SPEC.md:510
"""

from __future__ import annotations

import csv
import struct

import numpy as np

PK_MAGIC = b"HLBMPK01"
SN_MAGIC = b"HLBMSN01"
RS_MAGIC = b"HLBMRS01"


def write_packed(path, words, bits, mmin, mmax, step=0):
    """words: (5, nx, ny, nz) uint32 component-major (Solver.codes)."""
    w = np.asarray(words, dtype="<u4")
    C = 10
    dims = w.shape[1:]
    with open(path, "wb") as f:
        f.write(PK_MAGIC)
        f.write(struct.pack("<3I", *dims))
        f.write(struct.pack("<I", C))
        f.write(struct.pack(f"<{C}I", *[int(b) for b in bits]))
        f.write(struct.pack(f"<{C}d", *[float(v) for v in mmin]))
        f.write(struct.pack(f"<{C}d", *[float(v) for v in mmax]))
        f.write(struct.pack("<q", int(step)))
        f.write(np.ascontiguousarray(np.moveaxis(w, 0, -1)).tobytes())   # node-major


def read_packed(path):
    with open(path, "rb") as f:
        if f.read(8) != PK_MAGIC:
            raise ValueError("not a packed-buffer dump")
        dims = struct.unpack("<3I", f.read(12))
        (C,) = struct.unpack("<I", f.read(4))
        bits = struct.unpack(f"<{C}I", f.read(4 * C))
        mmin = struct.unpack(f"<{C}d", f.read(8 * C))
        mmax = struct.unpack(f"<{C}d", f.read(8 * C))
        (step,) = struct.unpack("<q", f.read(8))
        nw = (C * 16 + 31) // 32
        data = np.frombuffer(f.read(), dtype="<u4").reshape(tuple(dims) + (nw,))
    return {"dims": dims, "bits": bits, "min": mmin, "max": mmax, "step": step,
            "words": np.ascontiguousarray(np.moveaxis(data, -1, 0)).astype(np.uint32)}


def write_snapshot(path, rho, mom, stress, step=0, precision=0):
    st = np.concatenate([np.asarray(rho)[None], np.asarray(mom), np.asarray(stress)]).astype("<f4")
    with open(path, "wb") as f:
        f.write(SN_MAGIC)
        f.write(struct.pack("<q3III", int(step), *st.shape[1:], 10, int(precision)))
        f.write(np.ascontiguousarray(np.moveaxis(st, 0, -1)).tobytes())


def read_snapshot(path):
    with open(path, "rb") as f:
        if f.read(8) != SN_MAGIC:
            raise ValueError("not a snapshot")
        step, nx, ny, nz, C, prec = struct.unpack("<q3III", f.read(28))
        data = np.frombuffer(f.read(), dtype="<f4").reshape(nx, ny, nz, C)
    st = np.moveaxis(data, -1, 0).astype(np.float64)
    return {"step": step, "precision": prec, "rho": st[0], "mom": st[1:4], "stress": st[4:10]}


def save_checkpoint(path, solver):
    """Exact resume point: the raw internal state and the step counter (dither key)."""
    w = solver.get_state()
    prec = 1 if solver.config.precision == "q16" else 0
    with open(path, "wb") as f:
        f.write(RS_MAGIC)
        f.write(struct.pack("<q3III", solver.steps, *w.shape[1:], w.shape[0], prec))
        f.write(np.ascontiguousarray(w).astype(w.dtype.newbyteorder("<")).tobytes())


def load_checkpoint(path, solver):
    with open(path, "rb") as f:
        if f.read(8) != RS_MAGIC:
            raise ValueError("not a raw-state checkpoint")
        step, nx, ny, nz, NC, prec = struct.unpack("<q3III", f.read(28))
        if (nx, ny, nz) != tuple(solver.grid.dims) or prec != (1 if solver.config.precision == "q16" else 0):
            raise ValueError("checkpoint does not match the solver's grid / precision")
        dt = "<u4" if prec else "<f4"
        w = np.frombuffer(f.read(), dtype=dt).reshape(NC, nx, ny, nz)
    solver.set_state(w, step=step)
    return step


class StatsCSV:
    """StepStats log."""

    FIELDS = (["step", "t_fluid_ms", "t_copy_ms", "t_solid_ms", "mass", "momentum_x", "momentum_y",
               "momentum_z", "max_u"] + [f"saturation_{k}" for k in range(10)])

    def __init__(self, path):
        self._f = open(path, "w", newline="")
        self._w = csv.writer(self._f)
        self._w.writerow(self.FIELDS)

    def write(self, st):
        self._w.writerow([st.step, st.t_fluid_ms, st.t_copy_ms, st.t_solid_ms, repr(st.mass),
                          *(repr(float(v)) for v in st.momentum), repr(st.max_u),
                          *(int(v) for v in st.saturation)])
        self._f.flush()

    def close(self):
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def vorticity_z(velocity, z=None):
    """omega_z = d u_y / dx - d u_x / dy by periodic central differences on one z slice (default: the
    middle) of a (3, nx, ny, nz) velocity field -> (nx, ny) float64 (SPEC.md:510, 2-D flows)."""
    u = np.asarray(velocity, dtype=np.float64)
    k = u.shape[3] // 2 if z is None else int(z)
    ux, uy = u[0, :, :, k], u[1, :, :, k]
    return 0.5 * (np.roll(uy, -1, axis=0) - np.roll(uy, 1, axis=0)) - 0.5 * (np.roll(ux, -1, axis=1) - np.roll(ux, 1, axis=1))


def write_vorticity_pgm(path, velocity, vrange, z=None):
    """Optional PGM vorticity image of a snapshot: omega_z of one z slice mapped linearly
    from [-vrange, vrange] onto grey levels 0..255 (clipped), binary P5, rows = y (top = ny - 1), columns = x."""
    w = vorticity_z(velocity, z)
    g = np.clip(np.rint((w / float(vrange) + 1.0) * 127.5), 0, 255).astype(np.uint8)
    img = np.ascontiguousarray(g.T[::-1])   # (ny, nx), y up
    with open(path, "wb") as f:
        f.write(f"P5\n{img.shape[1]} {img.shape[0]}\n255\n".encode("ascii"))
        f.write(img.tobytes())
    return w
