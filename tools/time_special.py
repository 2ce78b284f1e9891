"""Interior-kernel time with statistics, with and without special (boundary / solid) cells, at the
paper's sphere scene size: the STATS+SPECIAL kernel variant vs the STATS one.
usage: python tools/time_special.py [n_sub]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
dims = (512, 256, 256)
cfg = SolverConfig(nu=1e-3, precision="q16", bc={"x": ("inflow", "outflow")}, u_in=(0.05, 0, 0))
from paper_2602_05295_b200.geometry import icosphere, sphere_mask
one = np.zeros(dims, np.uint8)
one[400, 10, 10] = 1
for sub in (None, 3, "voxel", "one"):
    with Solver(SimGrid(dims), cfg) as s:
        if sub == "voxel":
            s.set_mask(sphere_mask(dims, (128.3, 127.7, 128.1), 32.0))
        elif sub == "one":
            s.set_mask(one)
        elif sub is not None:
            V, F = icosphere((128.3, 127.7, 128.1), 32.0, sub)
            s.set_mesh(V, F)
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.init_modes(np.array([[0, 0, 0, 0.05, 0, 0, np.pi / 2]]))
        s.step_async(3)
        for stats in (False, True):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20):
                s.step_async(1, with_stats=stats)
            e1.record(); torch.cuda.synchronize()
            print(f"mesh={sub} stats={stats}: {e0.elapsed_time(e1) / 20:.4f} ms/step", flush=True)
        st = s.step(1)
        print(f"   t_fluid {st.t_fluid_ms:.4f} t_solid {st.t_solid_ms:.4f} sat {st.saturation.tolist()}", flush=True)
