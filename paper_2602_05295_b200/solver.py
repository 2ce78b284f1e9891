"""Solver API of the B200 HOME-LBM fluid step -- drop-in for the reference's solver path.

The reference package (``momentlbm``, /root/reference/pkg) specifies but does not ship its
``solver`` module; this module implements that surface over the C-ABI
``libhlbm.so``:

  * ``SimGrid``        -- SPEC.md:451-456 (dims, solid mask)
  * ``SolverConfig``   -- SPEC.md:457-459 (lattice, nu -> tau, force, BCs, quantization)
  * ``StepStats``      -- SPEC.md:460-462 (phase times, mass, momentum, max|u|, saturation)
  * ``Solver``         -- state on the GPU; ``step()``; moment / velocity accessors in the
                          reference array layout (moments.py:11-13)
  * ``fluid_update_step`` / ``run`` -- SPEC.md:473-477, 486-490

Errors follow the reference: ``ValueError`` for bad shapes / tau <= 1/2 / rho <= 0
(moments.py:33-34,147-150; collision.py:102-103,203-204), ``FloatingPointError`` on
divergence (collision.py:207-208).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .moments import MomentSet
from .quantization import QuantSpec

CS2 = 1.0 / 3.0


def tau_from_viscosity(nu: float) -> float:
    """tau = 0.5 + nu / cs2 (collision.py:30-31)."""
    return 0.5 + nu / CS2


@dataclass
class SimGrid:
    """Grid dims (x, y, z) and an optional uint8/bool solid mask (nx, ny, nz), C order."""
    dims: Sequence[int]
    mask: Optional[np.ndarray] = None

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        if len(self.dims) != 3:
            raise ValueError("D3Q27 grids are 3-D")
        if any(d < 1 for d in self.dims):
            raise ValueError("grid dims must be positive")
        if self.dims[2] % 4:
            raise ValueError("nz must be a multiple of 4")
        if self.mask is not None:
            m = np.asarray(self.mask)
            if m.shape != self.dims:
                raise ValueError(f"mask shape {m.shape} != dims {self.dims}")
            self.mask = np.ascontiguousarray(m.astype(np.uint8))


@dataclass
class SolverConfig:
    """Solver configuration.  ``bc`` maps axis -> (lo, hi); x faces accept
    periodic | inflow | outflow | wall, y/z faces periodic | wall."""
    lattice: str = "D3Q27"
    nu: float = 0.01
    force: Sequence[float] = (0.0, 0.0, 0.0)
    bc: dict = field(default_factory=lambda: {"x": ("periodic", "periodic"),
                                              "y": ("periodic", "periodic"),
                                              "z": ("periodic", "periodic")})
    u_in: Sequence[float] = (0.0, 0.0, 0.0)
    precision: str = "fp32"
    quant: QuantSpec = field(default_factory=QuantSpec)
    seed: int = 0
    device: int = 0
    xseg: int = 0

    def __post_init__(self):
        if self.lattice.upper() not in ("D3Q27", "D3Q19"):
            raise ValueError("the B200 step implements the D3Q27 and D3Q19 lattices")
        if self.precision not in _lib.PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_lib.PRECISIONS)}")
        if not self.tau > 0.5:
            raise ValueError("tau must exceed 0.5 (non-negative viscosity)")
        for ax in ("x", "y", "z"):
            lo, hi = self.bc.get(ax, ("periodic", "periodic"))
            for k in (lo, hi):
                if k not in _lib.BC_CODES:
                    raise ValueError(f"unknown boundary condition {k!r}")
            if ax != "x" and (lo in ("inflow", "outflow") or hi in ("inflow", "outflow")):
                raise ValueError("y/z faces support periodic or wall only")

    @property
    def tau(self) -> float:
        return tau_from_viscosity(self.nu)

    def faces(self):
        out = []
        for ax in ("x", "y", "z"):
            out.extend(self.bc.get(ax, ("periodic", "periodic")))
        return out


@dataclass
class StepStats:
    step: int
    t_fluid_ms: float
    t_copy_ms: float
    t_solid_ms: float
    mass: float
    momentum: np.ndarray
    max_u: float
    saturation: np.ndarray
    n_fluid: int
    force: np.ndarray = None      # triangle mesh: momentum exchange on the solid
    torque: np.ndarray = None
    finite: bool = True

    @classmethod
    def _from_c(cls, s: "_lib.HlbmStats") -> "StepStats":
        return cls(step=int(s.step), t_fluid_ms=s.t_fluid_ms, t_copy_ms=s.t_copy_ms,
                   t_solid_ms=s.t_solid_ms, mass=s.mass, momentum=np.array(list(s.momentum)),
                   max_u=s.max_u, saturation=np.array(list(s.saturation), dtype=np.int64),
                   n_fluid=int(s.n_fluid), force=np.array(list(s.force)),
                   torque=np.array(list(s.torque)), finite=bool(s.finite))


@dataclass
class Slab:
    """Placement of this solver's grid inside an x-slab-decomposed global grid."""
    x0: int
    gnx: int
    lo_remote: bool
    hi_remote: bool


class Solver:
    """HOME-LBM D3Q27 state resident on one B200 plus the step kernels."""

    def __init__(self, grid: SimGrid, config: SolverConfig, slab: Optional[Slab] = None):
        self.grid = grid
        self.config = config
        self.slab = slab
        self.state_version = 0   # bumped by every host-side state change and step (halo sync)
        self._lib = _lib.load()
        nx, ny, nz = grid.dims
        c = _lib.HlbmConfig()
        self._lib.hlbm_config_init(C.byref(c))     # struct_size (ABI guard) + defaults
        c.nx, c.ny, c.nz = nx, ny, nz
        c.gnx = slab.gnx if slab else nx
        c.gny, c.gnz = ny, nz
        c.x0 = slab.x0 if slab else 0
        c.x_lo_remote = int(bool(slab and slab.lo_remote))
        c.x_hi_remote = int(bool(slab and slab.hi_remote))
        c.tau = config.tau
        for k in range(3):
            c.force[k] = float(config.force[k])
            c.u_in[k] = float(config.u_in[k])
        for k, f in enumerate(config.faces()):
            c.bc[k] = _lib.BC_CODES[f]
        c.precision = _lib.PRECISIONS[config.precision]
        q = config.quant
        for k in range(10):
            c.qmin[k] = float(q.mmin[k])
            c.qmax[k] = float(q.mmax[k])
            c.bits[k] = int(q.bits[k])
        c.dither = int(bool(q.dither))
        c.seed = int(config.seed) & 0xFFFFFFFF
        c.device = int(config.device)
        c.xseg = int(config.xseg)
        c.q = 19 if config.lattice.upper() == "D3Q19" else 27   # D3Q19: two-chain streaming
        ctx = C.c_void_p()
        rc = self._lib.hlbm_create(C.byref(c), C.byref(ctx))
        self._ctx = ctx
        if rc != _lib.HLBM_OK:
            try:
                _lib.check(rc, ctx if ctx.value else None)
            finally:
                if ctx.value:
                    self._lib.hlbm_destroy(ctx)
                self._ctx = None
        self._last = None
        if grid.mask is not None:
            self.set_mask(grid.mask)

    # ---------------------------------------------------------------- lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.hlbm_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _chk(self, rc):
        _lib.check(rc, self._ctx)

    # ---------------------------------------------------------------- setup
    def set_mask(self, mask, ghost_lo=None, ghost_hi=None):
        m = np.ascontiguousarray(np.asarray(mask).astype(np.uint8))
        if m.shape != self.grid.dims:
            raise ValueError("mask shape does not match the grid")
        gl = None if ghost_lo is None else np.ascontiguousarray(np.asarray(ghost_lo).astype(np.uint8))
        gh = None if ghost_hi is None else np.ascontiguousarray(np.asarray(ghost_hi).astype(np.uint8))
        self._chk(self._lib.hlbm_set_mask(self._ctx, m.ctypes.data,
                                          None if gl is None else gl.ctypes.data,
                                          None if gh is None else gh.ctypes.data))
        self.grid.mask = m

    def set_mesh(self, vertices, faces, velocity=(0.0, 0.0, 0.0), omega=(0.0, 0.0, 0.0),
                 center=(0.0, 0.0, 0.0)):
        """Static triangle mesh in lattice coordinates (global grid): the pull links it cuts take
        the Eq.-8 boundary populations; replaces any voxel mask."""
        V = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        F = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
        motion = np.ascontiguousarray(np.concatenate([velocity, omega, center]), dtype=np.float64)
        self._chk(self._lib.hlbm_set_mesh(self._ctx, _lib.dptr(V), len(V),
                                          F.ctypes.data_as(C.POINTER(C.c_int32)), len(F), _lib.dptr(motion)))

    def set_solid_motion(self, velocity=(0.0, 0.0, 0.0), omega=(0.0, 0.0, 0.0), center=(0.0, 0.0, 0.0)):
        motion = np.ascontiguousarray(np.concatenate([velocity, omega, center]), dtype=np.float64)
        self._chk(self._lib.hlbm_set_solid_motion(self._ctx, _lib.dptr(motion)))

    def cut_links(self):
        """(global cells int64, masks uint32, t (n,27) float64 NaN where uncut, tri (n,27) int32)."""
        n = C.c_int64(0)
        self._chk(self._lib.hlbm_get_cut_links(self._ctx, None, None, None, None, C.byref(n)))
        cells = np.empty(n.value, dtype=np.int64)
        masks = np.empty(n.value, dtype=np.uint32)
        t = np.empty((n.value, 27), dtype=np.float64)
        tri = np.empty((n.value, 27), dtype=np.int32)
        if n.value:
            self._chk(self._lib.hlbm_get_cut_links(
                self._ctx, cells.ctypes.data_as(C.POINTER(C.c_int64)),
                masks.ctypes.data_as(C.POINTER(C.c_uint32)), _lib.dptr(t),
                tri.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n)))
        return cells, masks, t, tri

    def set_moments(self, rho, mom, stress):
        self.state_version += 1
        nx, ny, nz = self.grid.dims
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        mom = np.ascontiguousarray(mom, dtype=np.float64)
        stress = np.ascontiguousarray(stress, dtype=np.float64)
        if rho.shape != (nx, ny, nz) or mom.shape != (3, nx, ny, nz) or stress.shape != (6, nx, ny, nz):
            raise ValueError("expected rho (nx,ny,nz), mom (3,...), stress (6,...)")
        self._chk(self._lib.hlbm_set_moments(self._ctx, _lib.dptr(rho), _lib.dptr(mom),
                                             _lib.dptr(stress)))

    def set_equilibrium(self, rho, u):
        """rho, u fields -> (rho, rho u, rho u u) with sneq = 0 (SPEC.md:503 initialisation)."""
        rho = np.asarray(rho, dtype=np.float64)
        u = np.asarray(u, dtype=np.float64)
        mom = rho * u
        st = np.stack([mom[a] * u[b] for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])
        self.set_moments(rho, mom, st)

    def init_modes(self, modes: np.ndarray, rho0: float = 1.0):
        self.state_version += 1
        modes = np.ascontiguousarray(modes, dtype=np.float64).reshape(-1, 7)
        self._chk(self._lib.hlbm_init_modes(self._ctx, float(rho0), _lib.dptr(modes), len(modes)))

    # ---------------------------------------------------------------- stepping
    def step(self, n: int = 1) -> StepStats:
        self.state_version += 1
        s = _lib.HlbmStats()
        self._chk(self._lib.hlbm_step(self._ctx, int(n), C.byref(s)))
        self._last = StepStats._from_c(s)
        return self._last

    def step_async(self, n: int = 1, with_stats: bool = False):
        self.state_version += 1
        self._chk(self._lib.hlbm_step_async(self._ctx, int(n), int(with_stats)))

    def read_stats(self, check: bool = True) -> StepStats:
        """StepStats of the last step run with statistics.  ``check=False`` returns them even when
        they report divergence (``finite`` False or max|u| >= 0.9) instead of raising, so that a
        multi-rank caller can reduce a divergence flag before raising on every rank."""
        s = _lib.HlbmStats()
        rc = self._lib.hlbm_read_stats(self._ctx, C.byref(s))
        if not (rc == _lib.HLBM_EDIVERGED and not check):
            self._chk(rc)
        return StepStats._from_c(s)

    def step_fused(self, n: int = 1) -> StepStats:
        """The original HOME-LBM step (Alg. 1, SPEC.md `fused_step`): the stored state is
        read as POST-collision moments (Alg. 1's storage cut); per node reconstruct own f, stream
        through shared memory (8^3 tiles), solid links inline, extract, collide, write back.  n steps
        of it from m0 followed by one streaming S equal n split steps from S(m0).
        The in-repo baseline of the split scheme (voxel solids or a triangle mesh: cut links take the
        Eq.-8 population from the node's own stored post-collision moments; single domain)."""
        self.state_version += 1
        s = _lib.HlbmStats()
        self._chk(self._lib.hlbm_step_fused(self._ctx, int(n), C.byref(s)))
        self._last = StepStats._from_c(s)
        return self._last

    def fluid_update(self, with_stats: bool = True):
        """SPEC `fluid_update_step` (Alg. 2): the interior kernel over every
        cell, no obstacle logic.  With obstacles the step is committed by ``solid_correction``."""
        self.state_version += 1
        self._chk(self._lib.hlbm_fluid_update(self._ctx, int(with_stats)))

    def solid_correction(self) -> StepStats:
        """SPEC `solid_correction_step`: the compacted boundary / solid / cut-link
        kernels on the pending fluid update's output (identity when none is pending); returns the
        step's StepStats (phase times t_fluid_ms / t_solid_ms)."""
        self.state_version += 1
        s = _lib.HlbmStats()
        self._chk(self._lib.hlbm_solid_correction(self._ctx, C.byref(s)))
        self._last = StepStats._from_c(s)
        return self._last

    def stream(self):
        """The streaming operator S alone (no collision, not a time step): turns an Alg.-1
        (post-collision) state into the split scheme's storage cut."""
        self.state_version += 1
        self._chk(self._lib.hlbm_stream(self._ctx))

    def step_percell(self, n: int = 1) -> StepStats:
        """Per-cell gather step with the same storage cut as ``step`` (one thread per cell pulls its
        sources, each re-evaluating the source's collision): the GPU cross-check of the split kernels."""
        self.state_version += 1
        s = _lib.HlbmStats()
        self._chk(self._lib.hlbm_step_percell(self._ctx, int(n), C.byref(s)))
        self._last = StepStats._from_c(s)
        return self._last

    def step_reference(self, n: int = 1):
        """Full-grid update with the per-cell pull kernel (GPU cross-check of the fast kernel)."""
        self.state_version += 1
        self._chk(self._lib.hlbm_step_reference(self._ctx, int(n)))

    def set_stream(self, stream_ptr: int):
        self._chk(self._lib.hlbm_set_stream(self._ctx, C.c_void_p(stream_ptr)))

    @property
    def steps(self) -> int:
        return int(self._lib.hlbm_step_count(self._ctx))

    @property
    def launches(self) -> int:
        return int(self._lib.hlbm_launch_count(self._ctx))

    # ---------------------------------------------------------------- accessors
    def moments(self):
        """(rho, mom, stress) float64 in the reference layout."""
        nx, ny, nz = self.grid.dims
        rho = np.empty((nx, ny, nz))
        mom = np.empty((3, nx, ny, nz))
        st = np.empty((6, nx, ny, nz))
        self._chk(self._lib.hlbm_get_moments(self._ctx, _lib.dptr(rho), _lib.dptr(mom), _lib.dptr(st)))
        return rho, mom, st

    def moments_box(self, x0, cx, y0, cy, z0, cz):
        rho = np.empty((cx, cy, cz))
        mom = np.empty((3, cx, cy, cz))
        st = np.empty((6, cx, cy, cz))
        self._chk(self._lib.hlbm_get_moments_box(self._ctx, x0, cx, y0, cy, z0, cz, _lib.dptr(rho),
                                                 _lib.dptr(mom), _lib.dptr(st)))
        return rho, mom, st

    @property
    def rho(self):
        return self.moments()[0]

    @property
    def mom(self):
        return self.moments()[1]

    @property
    def stress(self):
        return self.moments()[2]

    @property
    def velocity(self):
        r, m, _ = self.moments()
        return m / r

    @property
    def sneq(self):
        """sneq = stress - mom mom / rho (moments.py:93-96)."""
        r, m, s = self.moments()
        outer = np.stack([m[a] * m[b] for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])
        return s - outer / r

    def moment_set(self, x, y, z) -> MomentSet:
        r, m, s = self.moments_box(x, 1, y, 1, z, 1)
        return MomentSet(rho=float(r[0, 0, 0]), mom=m[:, 0, 0, 0], stress=s[:, 0, 0, 0])

    def boundary(self):
        """(global linear cell indices int64 sorted, uint32 link masks)."""
        n = C.c_int64(0)
        self._chk(self._lib.hlbm_get_boundary(self._ctx, None, None, C.byref(n)))
        cells = np.empty(n.value, dtype=np.int64)
        masks = np.empty(n.value, dtype=np.uint32)
        if n.value:
            self._chk(self._lib.hlbm_get_boundary(
                self._ctx, cells.ctypes.data_as(C.POINTER(C.c_int64)),
                masks.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(n)))
        return cells, masks

    @property
    def boundary_cells(self):
        return self.boundary()[0]

    @property
    def link_masks(self):
        return self.boundary()[1]

    def get_codes(self, out=None):
        """Raw packed q16 words (5, nx, ny, nz) uint32, optionally into a caller buffer."""
        nx, ny, nz = self.grid.dims
        w = np.empty((5, nx, ny, nz), dtype=np.uint32) if out is None else out
        if w.shape != (5, nx, ny, nz) or w.dtype != np.uint32 or not w.flags.c_contiguous:
            raise ValueError("codes buffer must be a contiguous (5, nx, ny, nz) uint32 array")
        self._chk(self._lib.hlbm_get_codes(self._ctx, _lib.u32ptr(w)))
        return w

    @property
    def codes(self):
        """Raw packed q16 words (5, nx, ny, nz) uint32."""
        return self.get_codes()

    @codes.setter
    def codes(self, words):
        self.state_version += 1
        w = np.ascontiguousarray(words, dtype=np.uint32)
        if w.shape != (5,) + self.grid.dims:
            raise ValueError("codes must be (5, nx, ny, nz) uint32")
        self._chk(self._lib.hlbm_set_codes(self._ctx, _lib.u32ptr(w)))

    def get_state(self):
        """Raw internal state (NC, nx, ny, nz): float32 (rho-1, rho u, sneq) or uint32 q16 words."""
        nx, ny, nz = self.grid.dims
        q16 = self.config.precision == "q16"
        w = np.empty((5 if q16 else 10, nx, ny, nz), dtype=np.uint32 if q16 else np.float32)
        self._chk(self._lib.hlbm_get_state(self._ctx, w.ctypes.data))
        return w

    def set_state(self, words, step=None):
        self.state_version += 1
        nx, ny, nz = self.grid.dims
        q16 = self.config.precision == "q16"
        w = np.ascontiguousarray(words, dtype=np.uint32 if q16 else np.float32)
        if w.shape != ((5 if q16 else 10), nx, ny, nz):
            raise ValueError("state shape does not match the grid / precision")
        self._chk(self._lib.hlbm_set_state(self._ctx, w.ctypes.data))
        if step is not None:
            self._chk(self._lib.hlbm_set_step_count(self._ctx, int(step)))

    def halo_planes(self, next_buffer: bool = False):
        """Device pointers (send_lo, send_hi, recv_lo, recv_hi) and bytes per plane of the current
        state buffer, or of the buffer the step in progress writes (``next_buffer``)."""
        p = [C.c_void_p() for _ in range(4)]
        nb = C.c_int64()
        fn = self._lib.hlbm_next_halo_planes if next_buffer else self._lib.hlbm_halo_planes
        self._chk(fn(self._ctx, *(C.byref(x) for x in p), C.byref(nb)))
        return [x.value for x in p], nb.value

    # peer-store halo through CUDA IPC (include/hlbm.h hlbm_ipc_*; DistributedSolver transport="ipc")
    def ipc_export(self):
        """(handles: 128 bytes, current buffer index) for the neighbours' ``ipc_open``."""
        buf = C.create_string_buffer(128)
        cur = C.c_int32()
        self._chk(self._lib.hlbm_ipc_export(self._ctx, buf, C.byref(cur)))
        return buf.raw, cur.value

    def ipc_open(self, side: int, handles: bytes, peer_nx: int, peer_cur: int):
        if len(handles) != 128:
            raise ValueError("expected the 128 bytes of ipc_export")
        buf = C.create_string_buffer(handles, 128)
        self._chk(self._lib.hlbm_ipc_open(self._ctx, int(side), buf, int(peer_nx), int(peer_cur)))

    def ipc_sync(self, side: int, peer_cur: int):
        self._chk(self._lib.hlbm_ipc_sync(self._ctx, int(side), int(peer_cur)))

    def current_buffer(self) -> int:
        return self.ipc_export()[1]

    def halo_push(self, next_buffer: bool, stream_ptr: Optional[int] = None):
        self._chk(self._lib.hlbm_halo_push(self._ctx, int(bool(next_buffer)),
                                           C.c_void_p(int(stream_ptr)) if stream_ptr else None))

    def ipc_close(self):
        self._chk(self._lib.hlbm_ipc_close(self._ctx))

    # one step split into x-ranges of destination planes (overlapped multi-GPU schedule)
    def step_begin(self, with_stats: bool = False):
        self._chk(self._lib.hlbm_step_begin(self._ctx, int(with_stats)))

    def step_range(self, x_begin: int, x_end: int, stream_ptr: Optional[int] = None):
        """Destination planes [x_begin, x_end) of the step in progress, on the solver's stream or
        on `stream_ptr` (a CUDA stream handle; the caller orders it against the solver's stream)."""
        if stream_ptr is None:
            self._chk(self._lib.hlbm_step_range(self._ctx, int(x_begin), int(x_end)))
        else:
            self._chk(self._lib.hlbm_step_range_on(self._ctx, int(x_begin), int(x_end), C.c_void_p(int(stream_ptr))))

    def step_end(self):
        self.state_version += 1
        self._chk(self._lib.hlbm_step_end(self._ctx))

    def state_buffer(self):
        p = C.c_void_p()
        nb = C.c_int64()
        self._chk(self._lib.hlbm_state_buffer(self._ctx, C.byref(p), C.byref(nb)))
        return p.value, nb.value


# ---------------------------------------------------------------- functional wrappers

def fluid_update_step(solver: Solver) -> StepStats:
    """One split-scheme fluid update (Alg. 2)."""
    return solver.step(1)


def run(solver: Solver, steps: int, stats_every: int = 0, callback=None):
    """Advance ``steps`` steps, collecting StepStats every ``stats_every`` steps.

    Divergence raises FloatingPointError from the step that detected it."""
    out = []
    if steps <= 0:
        return out
    every = stats_every if stats_every > 0 else steps
    done = 0
    while done < steps:
        n = min(every, steps - done)
        st = solver.step(n)
        done += n
        out.append(st)
        if callback is not None:
            callback(solver, st)
    return out
