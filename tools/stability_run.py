"""Long-run stability of the 16-bit path at full scene size: StepStats every `every` steps (mass
drift, momentum, max|u|, saturation counts, finiteness).  usage:
    python tools/stability_run.py box|vehicle steps every"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes, vehicle_mask

scene = sys.argv[1] if len(sys.argv) > 1 else "box"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
if scene == "box":
    dims, mask = (512, 512, 512), None
    cfg = SolverConfig(nu=1e-4, precision="q16", quant=QuantSpec(dither=True), seed=1)
    init = lambda s: s.init_modes(turbulence_modes(512))
else:
    dims = (1000, 400, 400)
    mask = vehicle_mask(dims, seed=0)
    cfg = SolverConfig(nu=1e-5, precision="q16", quant=QuantSpec(dither=True), seed=1,
                       bc={"x": ("inflow", "outflow")}, u_in=(0.1, 0, 0))
    init = lambda s: s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
with Solver(SimGrid(dims, mask), cfg) as s:
    init(s)
    st0 = s.step(1)
    print(f"{scene} {dims} q16+dither: step 1 mass {st0.mass:.6e} max|u| {st0.max_u:.4f}", flush=True)
    done = 1
    sat = np.zeros(10, dtype=np.int64)
    while done < steps:
        n = min(every, steps - done)
        st = s.step(n)
        done += n
        sat += st.saturation
        print(f"step {done:6d}: mass drift {(st.mass - st0.mass) / st0.mass:+.3e}  momentum "
              f"{np.array2string(st.momentum, precision=4)}  max|u| {st.max_u:.4f}  "
              f"rho saturations (sampled steps) {int(st.saturation[0])}  finite {st.finite}", flush=True)
    print(f"done: {done} steps, saturation counts summed over the sampled steps {sat.tolist()}")
