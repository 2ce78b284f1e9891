"""Where the e2e time goes: set_codes / K x step(1) / get_codes at the bench workload."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes
n = 512
with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision="q16")) as s:
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.init_modes(turbulence_modes(n))
    host = torch.empty((5, n, n, n), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    s.get_codes(host)
    for rep in range(2):
        t0 = time.perf_counter(); s.codes = host; t1 = time.perf_counter()
        for _ in range(50): s.step(1)
        t2 = time.perf_counter(); s.get_codes(host); t3 = time.perf_counter()
        print(f"set_codes {1e3*(t1-t0):.1f} ms, step(1) {1e3*(t2-t1)/50:.3f} ms/step, get_codes {1e3*(t3-t2):.1f} ms")
    t0 = time.perf_counter()
    for _ in range(50): s.step_async(1, with_stats=True); s.read_stats()
    t1 = time.perf_counter()
    print(f"step_async(1,stats)+read_stats {1e3*(t1-t0)/50:.3f} ms/step")
