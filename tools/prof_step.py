"""Small fixed workload for ncu captures: N^3 turbulence box, a few steps."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec)) as s:
    s.init_modes(turbulence_modes(n))
    st = s.step(steps)
    print(f"{n}^3 {prec}: t_fluid {st.t_fluid_ms:.3f} ms, max_u {st.max_u:.4f}")
