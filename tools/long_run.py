"""Sustained ms/step over many steps (power-cap regime) with nvidia-smi clock samples."""
import sys, subprocess, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes
prec = sys.argv[1] if len(sys.argv) > 1 else "q16"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n = 512
samples = []
stop = threading.Event()
def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.1)
with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec)) as s:
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.init_modes(turbulence_modes(n))
    s.step_async(10); torch.cuda.synchronize()
    t = threading.Thread(target=sampler, daemon=True); t.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s.step_async(steps); e1.record(); torch.cuda.synchronize()
    stop.set(); t.join()
    ms = e0.elapsed_time(e1) / steps
    clk = sorted(float(x.split(",")[0]) for x in samples if x)
    pw = sorted(float(x.split(",")[1]) for x in samples if x)
    print(f"{prec} {steps} steps: {ms:.4f} ms/step {n**3/ms/1e3:.0f} MLUPS  sm clk median {clk[len(clk)//2]:.0f}  power median {pw[len(pw)//2]:.0f} W")
