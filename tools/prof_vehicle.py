import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig, QuantSpec
from paper_2602_05295_b200.geometry import vehicle_mask
dims = (1000, 400, 400)
cfg = SolverConfig(nu=1e-5, precision="q16", quant=QuantSpec(dither=True), seed=1,
                   bc={"x": ("inflow", "outflow")}, u_in=(0.1, 0, 0))
with Solver(SimGrid(dims, vehicle_mask(dims, seed=0)), cfg) as s:
    s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
    st = s.step(4)
    print("t_fluid", st.t_fluid_ms, "t_solid", st.t_solid_ms)
