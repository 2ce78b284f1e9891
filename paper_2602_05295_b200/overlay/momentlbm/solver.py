"""momentlbm.solver -- the reference package's time-integration module, backed by the B200 kernels.

The reference package names ``momentlbm.solver`` in its layout (pkg/src/momentlbm/__init__.py:1-9)
and specifies it in SPEC.md:446-516, but does not ship it.  This file is that module: installed
into the reference package's namespace by ``paper_2602_05295_b200.dropin.install()`` (which adds
this directory to ``momentlbm.__path__``), so that

    import momentlbm.solver as S
    grid = S.SimGrid((64, 64, 64))
    cfg = S.SolverConfig(nu=0.01)
    S.fluid_update_step(grid, cfg)

runs the hand-written sm_100a kernels of ``libhlbm.so``.  The reference's own types are reused:
``MomentSet`` (moments.py:136-172) for per-node access, ``make_lattice`` for the lattice kind.
There is no CPU fallback: without a CUDA device the first step raises RuntimeError.

Operations:
  fused_step(grid, config)            Alg. 1 (:465-472) -- the original HOME-LBM kernel
  fluid_update_step(grid, config)     Alg. 2 (:473-477) -- interior kernel, no obstacle logic
  solid_correction_step(grid, config) Alg. 3 role (:478-485) -- compacted boundary kernels
  run(config, steps)                  (:486-490) -- StepStats, snapshots; divergence aborts with
                                      the last-good snapshot (the grid is restored to it)
Storage cuts: a grid advanced by ``fused_step`` holds post-collision moments (Alg. 1), one advanced
by ``fluid_update_step`` post-streaming moments (Alg. 2); ``align_to_split(grid)`` applies the
streaming operator S once, (S o C)^n o S = S o (C o S)^n.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from momentlbm.lattice import make_lattice
from momentlbm.moments import MomentSet

from paper_2602_05295_b200 import QuantSpec
from paper_2602_05295_b200 import io as _io
from paper_2602_05295_b200.geometry import load_obj
from paper_2602_05295_b200 import solver as _b200
from paper_2602_05295_b200.solver import StepStats

__all__ = ["SimGrid", "SolverConfig", "StepStats", "Snapshot", "RunResult", "SolverDiverged",
           "fused_step", "fluid_update_step", "solid_correction_step", "run", "align_to_split"]

TILE = 8                      # SPEC.md:452 "tile size 8 per axis"
FACES = ("x-", "x+", "y-", "y+", "z-", "z+")


def _face_spec(spec):
    """'periodic' | 'outflow' | 'wall' | ('inflow', (ux, uy, uz)) | 'inflow' -> (kind, u or None)."""
    if isinstance(spec, str):
        if spec not in ("periodic", "inflow", "outflow", "wall"):
            raise ValueError(f"unknown boundary condition {spec!r}")
        return spec, None
    kind, u = spec
    if kind != "inflow":
        raise ValueError(f"only inflow takes a velocity, got {spec!r}")
    return "inflow", tuple(float(v) for v in u)


@dataclass
class SolverConfig:
    """lattice kind, nu (tau = 0.5 + 3 nu, collision.py:30-31), body force F,
    boundary condition per face (periodic | inflow(velocity) | outflow | wall), quantization preset
    ("16/16" ... "12/11", a QuantSpec) or None, obstacle list (voxel masks, triangle meshes
    (vertices, faces[, motion]) in lattice coordinates, or Wavefront OBJ paths).  ``dims`` / ``initial`` let ``run(config, steps)``
    build its own grid (``initial``: None = rest, or a (rho, mom, stress) triple)."""
    lattice: str = "D3Q27"
    nu: float = 0.01
    force: Sequence[float] = (0.0, 0.0, 0.0)
    bc: dict = field(default_factory=dict)
    quantization: object = None
    dither: bool = False
    obstacles: list = field(default_factory=list)
    seed: int = 0
    device: int = 0
    dims: Optional[Sequence[int]] = None
    initial: object = None

    def __post_init__(self):
        make_lattice(self.lattice)                       # the reference validates the kind
        if not self.nu > 0:
            raise ValueError("tau must exceed 0.5 (non-negative viscosity)")   # collision.py:102-103
        for f in self.bc:
            if f not in FACES:
                raise ValueError(f"unknown face {f!r} (expected one of {FACES})")
            _face_spec(self.bc[f])

    @property
    def tau(self) -> float:
        return 0.5 + 3.0 * self.nu

    def quant_spec(self) -> Optional[QuantSpec]:
        q = self.quantization
        if q is None or q is False:
            return None
        if isinstance(q, QuantSpec):
            spec = q
        elif isinstance(q, str):
            spec = QuantSpec.preset(q)
        else:
            raise ValueError(f"quantization must be None, a preset name or a QuantSpec, got {q!r}")
        if self.dither and not spec.dither:
            spec = QuantSpec(mmin=spec.mmin, mmax=spec.mmax, bits=spec.bits, dither=True)
        return spec

    def _b200(self) -> "_b200.SolverConfig":
        faces = {f: _face_spec(self.bc.get(f, "periodic")) for f in FACES}
        u_in = [u for k, u in faces.values() if k == "inflow"]
        if len({tuple(u) for u in u_in}) > 1:
            raise ValueError("inflow faces must share one velocity")
        bc = {ax: (faces[ax + "-"][0], faces[ax + "+"][0]) for ax in "xyz"}
        q = self.quant_spec()
        return _b200.SolverConfig(lattice=self.lattice, nu=self.nu, force=tuple(self.force), bc=bc,
                                  u_in=u_in[0] if u_in else (0.0, 0.0, 0.0),
                                  precision="q16" if q is not None else "fp32",
                                  quant=q if q is not None else QuantSpec(), seed=self.seed, device=self.device)


class SimGrid:
    """dims, per-node moment storage (on the GPU, structure of arrays), the solid
    mask and the step counter.  The device state is created on the first operation with a config
    and rebuilt (state carried over in float64) if a later call passes a different config."""

    def __init__(self, dims: Sequence[int], mask: Optional[np.ndarray] = None):
        self.dims = tuple(int(d) for d in dims)
        if len(self.dims) != 3:
            raise ValueError("the B200 solver runs 3-D grids (D3Q27 / D3Q19)")
        self.mask = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
        if self.mask is not None and self.mask.shape != self.dims:
            raise ValueError(f"mask shape {self.mask.shape} != dims {self.dims}")
        self._solver: Optional[_b200.Solver] = None
        self._key = None
        self._pending = None     # moments set before the device state exists

    # ------------------------------------------------------------------ device binding
    def bind(self, config: SolverConfig) -> _b200.Solver:
        cfg = config._b200()
        key = repr(cfg) + repr([(id(o)) for o in config.obstacles])
        if self._solver is not None and key == self._key:
            return self._solver
        carried = None
        step = 0
        if self._solver is not None:
            carried = self._solver.moments()
            step = self._solver.steps
            self._solver.close()
        mask = self.mask
        meshes = []
        for ob in config.obstacles:
            if isinstance(ob, (str, os.PathLike)):      # Wavefront OBJ (SPEC.md:404-407 load_mesh)
                ob = load_obj(ob)
            if isinstance(ob, np.ndarray):
                m = np.asarray(ob, dtype=np.uint8)
                mask = m if mask is None else (mask | m)
            else:
                meshes.append(ob)
        if meshes and mask is not None:
            raise ValueError("voxel masks and triangle meshes cannot be combined in one grid")
        if len(meshes) > 1:
            raise ValueError("one triangle mesh per grid (concatenate the obstacles' meshes)")
        s = _b200.Solver(_b200.SimGrid(self.dims, mask), cfg)
        if meshes:
            V, F = meshes[0][:2]
            motion = meshes[0][2] if len(meshes[0]) > 2 else {}
            s.set_mesh(V, F, **motion)     # motion: {velocity, omega, center} (SPEC SolidState)
        init = carried if carried is not None else self._pending
        if init is not None:
            s.set_moments(*init)
            self._pending = None
        if step:
            s._chk(s._lib.hlbm_set_step_count(s._ctx, int(step)))
        self._solver, self._key = s, key
        return s

    @property
    def solver(self) -> _b200.Solver:
        if self._solver is None:
            raise RuntimeError("the grid has no device state yet: pass it to an operation with a config")
        return self._solver

    def close(self):
        if self._solver is not None:
            self._solver.close()
            self._solver = None

    # ------------------------------------------------------------------ state
    def set_moments(self, rho, mom, stress):
        if self._solver is None:
            self._pending = (np.asarray(rho, np.float64), np.asarray(mom, np.float64),
                             np.asarray(stress, np.float64))
        else:
            self._solver.set_moments(rho, mom, stress)

    def moments(self):
        if self._solver is None:
            if self._pending is not None:
                return self._pending
            n = self.dims
            return np.ones(n), np.zeros((3,) + n), np.zeros((6,) + n)
        return self._solver.moments()

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
    def step_count(self) -> int:
        return 0 if self._solver is None else self._solver.steps

    def moment_set(self, x: int, y: int, z: int) -> MomentSet:
        """The reference's per-node value type (moments.py:136-172)."""
        if self._solver is None:
            r, m, s = self.moments()
            return MomentSet(rho=float(r[x, y, z]), mom=m[:, x, y, z], stress=s[:, x, y, z])
        r, m, s = self._solver.moments_box(x, 1, y, 1, z, 1)
        return MomentSet(rho=float(r[0, 0, 0]), mom=m[:, 0, 0, 0], stress=s[:, 0, 0, 0])


# ---------------------------------------------------------------------- operations
def fused_step(grid: SimGrid, config: SolverConfig) -> SimGrid:
    """SPEC.md:465-472 / PAPER.md Alg. 1: one original HOME-LBM step on post-collision moments."""
    grid.bind(config).step_fused(1)
    return grid


def fluid_update_step(grid: SimGrid, config: SolverConfig) -> SimGrid:
    """SPEC.md:473-477 / PAPER.md Alg. 2: collision -> reconstruct -> stream -> extract -> write over
    every node, no obstacle logic.  With obstacles the step is finished by solid_correction_step
    (or implicitly by the next state access)."""
    grid.bind(config).fluid_update(with_stats=True)
    return grid


def solid_correction_step(grid: SimGrid, config: SolverConfig) -> SimGrid:
    """the boundary correction of the pending fluid update -- half-way bounce-back on
    voxel cut links, the Eq.-8 boundary populations on triangle-mesh cut links,
    solid nodes at rest.  Identity when no obstacle is present.  The step's StepStats are kept in
    ``grid.last_stats``."""
    grid.last_stats = grid.bind(config).solid_correction()
    return grid


def align_to_split(grid: SimGrid, config: SolverConfig) -> SimGrid:
    """Apply the streaming operator S once: an Alg.-1 (fused) state -> the split scheme's cut."""
    grid.bind(config).stream()
    return grid


@dataclass
class Snapshot:
    step: int
    rho: np.ndarray
    mom: np.ndarray
    stress: np.ndarray

    def write(self, path, precision: int = 0):
        """SPEC.md:510 snapshot format (paper_2602_05295_b200.io)."""
        _io.write_snapshot(path, self.rho, self.mom, self.stress, self.step, precision)


@dataclass
class RunResult:
    stats: list
    snapshots: list
    grid: SimGrid


class SolverDiverged(FloatingPointError):
    """Divergence (|u| >= 0.9 or a non-finite moment) during ``run``: carries the step
    that diverged, the last-good snapshot (the grid has been restored to it) and the stats so far."""

    def __init__(self, msg, step, last_good: Snapshot, stats):
        super().__init__(msg)
        self.step = step
        self.last_good = last_good
        self.stats = stats


def _snapshot(s: _b200.Solver) -> Snapshot:
    r, m, st = s.moments()
    return Snapshot(s.steps, r, m, st)


def run(config: SolverConfig, steps: int, grid: Optional[SimGrid] = None, *, snapshot_every: int = 0,
        stats_every: int = 1, checkpoint_every: int = 100,
        on_snapshot: Optional[Callable[[Snapshot], None]] = None) -> RunResult:
    """advance ``steps`` split steps (BCs applied every step), recording StepStats
    every ``stats_every`` steps and snapshots every ``snapshot_every`` steps (the initial snapshot is
    always recorded: 0 steps -> initial snapshot only).  The raw state is checkpointed every
    ``checkpoint_every`` steps (and at every snapshot); on divergence the grid is restored to the
    last checkpoint and SolverDiverged (a FloatingPointError) carries it as the last-good snapshot."""
    if steps < 0:
        raise ValueError("steps must be >= 0")
    if grid is None:
        if config.dims is None:
            raise ValueError("run(config, steps) needs config.dims (or a grid)")
        grid = SimGrid(config.dims)
        if config.initial is not None:
            grid.set_moments(*config.initial)
    s = grid.bind(config)
    snaps = [_snapshot(s)]
    if on_snapshot:
        on_snapshot(snaps[0])
    stats = []
    good = (s.get_state(), s.steps)
    marks = [m for m in (stats_every, snapshot_every, checkpoint_every) if m and m > 0]
    done = 0
    while done < steps:
        n = steps - done
        for m in marks:                    # stop at the next multiple of every cadence
            n = min(n, m - (done % m))
        try:
            st = s.step(n)
        except FloatingPointError as e:
            words, step = good
            s.set_state(words, step=step)
            raise SolverDiverged(f"divergence within steps {s.steps - n + 1}..{done + n} of the run: {e}",
                                 done + n, _snapshot(s), stats) from e
        done += n
        if stats_every and done % stats_every == 0:
            stats.append(st)
        if snapshot_every and done % snapshot_every == 0:
            snaps.append(_snapshot(s))
            if on_snapshot:
                on_snapshot(snaps[-1])
        if (checkpoint_every and done % checkpoint_every == 0) or (snapshot_every and done % snapshot_every == 0):
            good = (s.get_state(), s.steps)
    grid.last_stats = stats[-1] if stats else None
    return RunResult(stats=stats, snapshots=snaps, grid=grid)
