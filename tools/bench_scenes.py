"""Throughput of the BASELINE.json scene configs on one B200 (supplementary to bench.py).

config 1: TGV 64^3 fp32 periodic (parity config; L2-resident, not a roofline number)
config 2: turbulence box 512^3, fp32 and q16 (bench.py's headline)
config 3: channel past a sphere 512x256x256 (inflow/outflow, periodic y/z), fp32 and q16
config 4: procedural vehicle 1000x400x400, q16 + dither, inflow/outflow, periodic y/z
Prints one JSON object per line: MLUPS (all cells), fluid-cell MLUPS, the split phase times
(fluid_interior vs compacted boundary kernel), boundary-list sizes and, for voxel scenes, the
time of the original HOME-LBM kernel (Alg. 1: own-population reconstruction into
shared memory, 8^3 tiles, solid links inline, post-collision storage) -- the in-repo version of the
paper's split / quantization attribution: fp32 Alg. 1 -> fp32 split -> q16 split.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask, turbulence_modes, vehicle_mask, voxel_surface_mesh


def timed(s, steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step_async(steps)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run(name, dims, cfg, init, mask=None, steps=50, mesh=None):
    t0 = time.perf_counter()
    s = Solver(SimGrid(dims, mask), cfg)
    if mesh is not None:
        s.set_mesh(*mesh)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    setup = time.perf_counter() - t0
    init(s)
    s.step_async(5)
    ms = timed(s, steps)
    st = s.step(3)              # phase split (events around each kernel) + stats
    fused_ms = None
    if True:                    # the fused Alg.-1 baseline (one kernel, solid / cut links inline)
        s.step_fused(1)
        fused_ms = s.step_fused(max(2, steps // 10)).t_fluid_ms
    cells = int(np.prod(dims))
    nb = len(s.boundary_cells) if mask is not None else (len(s.cut_links()[0]) if mesh is not None else 0)
    out = {"config": name, "dims": list(dims), "precision": cfg.precision, "ms_per_step": round(ms, 4),
           "mlups": round(cells / ms / 1e3, 1), "fluid_mlups": round(st.n_fluid / ms / 1e3, 1),
           "t_fluid_ms": round(st.t_fluid_ms, 4), "t_solid_ms": round(st.t_solid_ms, 4),
           "boundary_cells": nb, "solid_cells": cells - st.n_fluid, "setup_s": round(setup, 2),
           "triangles": 0 if mesh is None else int(len(mesh[1])),
           "max_u": round(st.max_u, 4), "saturation_rho": int(st.saturation[0])}
    if fused_ms is not None:
        out["fused_alg1_ms_per_step"] = round(fused_ms, 4)
        out["split_speedup_vs_fused"] = round(fused_ms / ms, 2)
    s.close()
    print(json.dumps(out), flush=True)


def main():
    from paper_2602_05295_b200.geometry import taylor_green_fields
    tgv = taylor_green_fields(64)
    run("1 TGV 64^3", (64, 64, 64), SolverConfig(nu=0.01), lambda s: s.set_equilibrium(*tgv), steps=200)
    for prec in ("fp32", "q16"):
        run("2 turbulence box", (512, 512, 512), SolverConfig(nu=1e-4, precision=prec),
            lambda s: s.init_modes(turbulence_modes(512)))
    uniform = lambda u: (lambda s: s.init_modes(np.array([[0, 0, 0, u, 0, 0, np.pi / 2]])))
    # D3Q27 vs D3Q19 at the paper's 720x360x360 comparison size; D3Q19 runs the
    # two-chain interior kernel (216 w = prod(4,1,1) + prod(2,-1,-1))
    for lat in ("D3Q27", "D3Q19"):
        run(f"lattice {lat} 720x360x360 box", (720, 360, 360), SolverConfig(nu=1e-4, precision="q16", lattice=lat),
            lambda s: s.init_modes(turbulence_modes(360, dims=(720, 360, 360))), steps=20)
    dims = (512, 256, 256)
    m = sphere_mask(dims, (128, 128, 128), 32)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")}
    for prec in ("fp32", "q16"):
        run("3 sphere channel", dims, SolverConfig(nu=1e-4, bc=bc, u_in=(0.1, 0, 0), precision=prec),
            uniform(0.1), mask=m)
    from paper_2602_05295_b200.geometry import icosphere
    sph = icosphere((128, 128, 128), 32.0, 5)
    run("3b sphere channel, triangle mesh", dims, SolverConfig(nu=1e-4, bc=bc, u_in=(0.1, 0, 0), precision="q16"),
        uniform(0.1), mesh=sph)
    dims = (1000, 400, 400)
    m = vehicle_mask(dims, seed=0)
    run("4 vehicle", dims, SolverConfig(nu=1e-5, bc=bc, u_in=(0.1, 0, 0), precision="q16",
                                        quant=QuantSpec(dither=True)), uniform(0.1), mask=m)
    run("4 vehicle", dims, SolverConfig(nu=1e-5, bc=bc, u_in=(0.1, 0, 0), precision="fp32"), uniform(0.1), mask=m)
    mesh = voxel_surface_mesh(m)
    run("4b vehicle, triangle mesh", dims, SolverConfig(nu=1e-5, bc=bc, u_in=(0.1, 0, 0), precision="q16",
                                                        quant=QuantSpec(dither=True)), uniform(0.1), mesh=mesh)


if __name__ == "__main__":
    main()
