"""Solid-correction phase time (StepStats.t_solid_ms, averaged over steps) on the config-3 / config-4
voxel scenes, and a checksum of the state after the run (A/B of library variants via HLBM_LIB).
usage: python tools/time_solid.py [steps] [--save PREFIX]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask, vehicle_mask

steps = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 10
save = sys.argv[sys.argv.index("--save") + 1] if "--save" in sys.argv else None
scenes = {
    "vehicle": ((1000, 400, 400), lambda d: vehicle_mask(d, seed=0)),
    "sphere": ((512, 256, 256), lambda d: sphere_mask(d, (128.3, 127.7, 128.1), 32.0)),
}
for name, (dims, mk) in scenes.items():
    for prec in ("q16", "fp32"):
        cfg = SolverConfig(nu=1e-5, precision=prec, quant=QuantSpec(dither=prec == "q16"), seed=1,
                           bc={"x": ("inflow", "outflow")}, u_in=(0.1, 0, 0))
        with Solver(SimGrid(dims, mk(dims)), cfg) as s:
            s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
            s.step(3)
            ts, tf = [], []
            for _ in range(steps):
                st = s.step(1)
                ts.append(st.t_solid_ms)
                tf.append(st.t_fluid_ms)
            w = s.get_state()
            print(f"{name} {prec}: t_solid {np.mean(ts):.4f} ms  t_fluid {np.mean(tf):.4f} ms  "
                  f"checksum {int(w.view(np.uint32).astype(np.uint64).sum())}", flush=True)
            if save:
                np.save(f"{save}_{name}_{prec}.npy", w)
