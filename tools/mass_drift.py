"""Relative mass drift over 1000 periodic steps (< 1e-10 for the float64 reference)
for fp32 and q16 (with / without dither) state.  usage: python tools/mass_drift.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2602_05295_b200 import Solver, SimGrid, SolverConfig, QuantSpec
for shape in [(32,32,32),(128,128,128)]:
    rng = np.random.default_rng(3)
    rho = 1.0 + rng.uniform(-0.02, 0.02, shape)
    u = rng.uniform(-0.03, 0.03, (3,) + shape)
    for prec, q in [("fp32", QuantSpec()), ("q16", QuantSpec(dither=True)), ("q16", QuantSpec(dither=False))]:
        with Solver(SimGrid(shape), SolverConfig(nu=0.02, precision=prec, quant=q, seed=1)) as s:
            s.set_equilibrium(rho, u)
            m0 = s.step(1); m1 = s.step(999)
            print(shape, prec, q.dither, "rel mass drift %.3e" % ((m1.mass - m0.mass) / m0.mass), "mom", m1.momentum - m0.momentum, flush=True)
