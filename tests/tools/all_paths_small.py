"""Small end-to-end run of every kernel family (CUDA_LAUNCH_BLOCKING=1 catches launch errors at the call) on
tiny grids -- interior (fp32, q16 + dither + stats + solids), compacted lists (voxel, mesh), Alg. 1,
the stream operator, per-cell step, import / export, D3Q19."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
from oracle import mesh as M
from oracle import step as OS
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask

shape = (20, 33, 68)
mask = sphere_mask(shape, (9, 16.5, 33.5), 5)
state = OS.random_state(shape, seed=1, drho=0.03, umax=0.04, sneq=0.003)
bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
for lat in ("D3Q27", "D3Q19"):
    for prec, q in (("fp32", QuantSpec()), ("q16", QuantSpec(dither=True)), ("q16", QuantSpec.preset("14/13"))):
        cfg = SolverConfig(nu=0.02, precision=prec, quant=q, bc=bc, u_in=(0.05, 0, 0), lattice=lat, force=(1e-5, 0, 0))
        with Solver(SimGrid(shape, mask), cfg) as s:
            s.set_moments(*state)
            s.step(2)
            s.step_async(2, with_stats=False)
            s.step_fused(1)
            s.stream()
            s.step_percell(1)
            s.fluid_update(True)
            s.solid_correction()
            s.moments()
        print(lat, prec, "ok", flush=True)
V, F = M.icosphere((9.3, 16.7, 33.1), 5.2, 2)
with Solver(SimGrid(shape), SolverConfig(nu=0.02, precision="q16")) as s:
    s.set_mesh(V, F)
    s.set_moments(*state)
    s.step(2)
    s.cut_links()
    s.step_fused(2)      # Alg. 1 with the mesh's cut links
    s.stream()
    s.moments()
print("mesh ok")
