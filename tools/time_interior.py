"""ms/step of the interior kernel at the bench workload (CUDA events), q16 and fp32."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes
n = 512
for prec in sys.argv[1:] or ["q16", "fp32"]:
    with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec, xseg=128)) as s:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.init_modes(turbulence_modes(n))
        s.step_async(5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.step_async(100); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 100
        print(f"{prec}: {ms:.4f} ms/step  {n**3/ms/1e3:.0f} MLUPS", flush=True)
