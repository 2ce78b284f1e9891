"""Phase breakdown of an obstacle scene on one B200: interior (fluid update) vs compacted boundary
kernels, with and without dither.  usage: python tools/scene_breakdown.py [nx ny nz]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import vehicle_mask

dims = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 512, 512)
mask = vehicle_mask(dims, seed=0)
bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
for prec, dither, m in (("q16", True, mask), ("q16", False, mask), ("q16", False, None), ("fp32", False, mask)):
    cfg = SolverConfig(nu=1e-5, precision=prec, quant=QuantSpec(dither=dither), bc=bc, u_in=(0.1, 0, 0))
    with Solver(SimGrid(dims, m), cfg) as s:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
        s.step_async(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.step_async(10); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl, so = [], []
        for _ in range(5):
            st = s.fluid_update(with_stats=False) or s.solid_correction()
            fl.append(st.t_fluid_ms); so.append(st.t_solid_ms)
        nb = len(s.boundary_cells) if m is not None else 0
    print(f"{dims} {prec} dither={dither} mask={m is not None}: {ms:.4f} ms/step ({np.prod(dims)/ms/1e3:.0f} MLUPS); "
          f"fluid update {np.median(fl):.4f} ms, solid correction {np.median(so):.4f} ms, boundary cells {nb}", flush=True)
