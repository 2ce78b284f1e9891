"""Per-node moment value type returned by ``Solver.moment_set`` (host-side accessor).

The reference's own ``MomentSet`` (momentlbm/moments.py:136-172) when the reference package is
importable; otherwise a stand-in with the same fields, validation (ValueError for rho <= 0 or
|u_a| >= 1), ``velocity`` and ``decompose`` (moments.py:93-96).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_VOIGT_PAIRS = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


@dataclass
class _MomentSet:
    rho: float
    mom: np.ndarray
    stress: np.ndarray

    def __post_init__(self):
        self.mom = np.asarray(self.mom, dtype=np.float64)
        self.stress = np.asarray(self.stress, dtype=np.float64)
        if self.rho <= 0:
            raise ValueError("density must be positive")
        if np.any(np.abs(self.mom / self.rho) >= 1.0):
            raise ValueError("velocity components must stay below 1")

    @property
    def velocity(self) -> np.ndarray:
        return self.mom / self.rho

    def decompose(self) -> np.ndarray:
        outer = np.array([self.mom[a] * self.mom[b] for a, b in _VOIGT_PAIRS])
        return self.stress - outer / self.rho


try:   # the reference class itself when the reference package is on the path
    from momentlbm.moments import MomentSet  # noqa: F401
except ImportError:
    MomentSet = _MomentSet
