"""paper_2602_05295_b200 -- B200-native HOME-LBM D3Q27 fluid step (arXiv 2602.05295).

Drop-in for the reference package's solver path (momentlbm): the Python
API in :mod:`.solver` drives hand-written sm_100a kernels through the C-ABI libhlbm.so
(include/hlbm.h).  There is no CPU fallback.
"""

from .quantization import QuantSpec
from .solver import (SimGrid, Slab, Solver, SolverConfig, StepStats, fluid_update_step, run,
                     tau_from_viscosity)

__all__ = ["QuantSpec", "SimGrid", "Slab", "Solver", "SolverConfig", "StepStats",
           "fluid_update_step", "run", "tau_from_viscosity"]
__version__ = "0.1.0"
