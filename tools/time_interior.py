"""ms/step of the interior kernel at the bench workload (CUDA events), q16 and fp32.
usage: python tools/time_interior.py [q16|fp32 ...] [--xseg N] [--n N]"""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes
ap = argparse.ArgumentParser()
ap.add_argument("prec", nargs="*", default=["q16", "fp32"])
ap.add_argument("--xseg", type=int, default=0)
ap.add_argument("--n", type=int, default=512)
a = ap.parse_args()
n = a.n
for prec in a.prec:
    with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec, xseg=a.xseg)) as s:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.init_modes(turbulence_modes(n))
        s.step_async(5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.step_async(100); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 100
        e0.record()
        for _ in range(20): s.step_async(1, with_stats=True)
        e1.record(); torch.cuda.synchronize()
        ms_st = e0.elapsed_time(e1) / 20
        print(f"{prec} xseg={a.xseg}: {ms:.4f} ms/step  {n**3/ms/1e3:.0f} MLUPS   (stats every step: {ms_st:.4f} ms)", flush=True)
