"""The bench workload (512^3 turbulence box, xseg 128) for a few steps, for ncu captures."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes

prec = sys.argv[1] if len(sys.argv) > 1 else "q16"
xseg = int(sys.argv[2]) if len(sys.argv) > 2 else 128
n = 512
with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec, xseg=xseg)) as s:
    s.init_modes(turbulence_modes(n))
    st = s.step(3)
    print(f"{prec}: t_fluid {st.t_fluid_ms:.3f} ms")
