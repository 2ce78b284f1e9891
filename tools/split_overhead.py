"""Single-GPU cost of the overlapped multi-GPU step schedule: the per-rank kernels of
a slab step -- edge planes (0, 1) and (nx-1, nx), then the bulk (1, nx-1) -- against one full-slab
launch, 512^3 per GPU (the weak-scaling slab).  The halo exchange itself runs on a side stream
during the bulk and is not included (one GPU).  usage: python tools/split_overhead.py [q16|fp32 ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2602_05295_b200 import SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import turbulence_modes

n, reps = 512, 50
for prec in (sys.argv[1:] or ["q16", "fp32"]):
    with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4, precision=prec)) as s:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.init_modes(turbulence_modes(n))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        side = torch.cuda.Stream()
        res = {}
        for split in (False, True, "side", False, True, "side"):
            s.step_async(3)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                if split == "side":   # DistributedSolver's schedule: edges on a side stream
                    s.step_begin(False)
                    ev = torch.cuda.Event()
                    ev.record()
                    side.wait_event(ev)
                    s.step_range(0, 1, side.cuda_stream)
                    s.step_range(n - 1, n, side.cuda_stream)
                    done = torch.cuda.Event()
                    done.record(side)
                    s.step_range(1, n - 1)
                    torch.cuda.current_stream().wait_event(done)
                    s.step_end()
                elif split:
                    s.step_begin(False)
                    for a, b in ((0, 1), (n - 1, n), (1, n - 1)):
                        s.step_range(a, b)
                    s.step_end()
                else:
                    s.step_async(1)
            e1.record()
            torch.cuda.synchronize()
            res[split] = e0.elapsed_time(e1) / reps
        print(f"{prec}: full step {res[False]:.4f} ms, split schedule in order {res[True]:.4f} ms "
              f"(+{100 * (res[True] / res[False] - 1):.1f}%), edges on a side stream {res['side']:.4f} ms "
              f"(+{100 * (res['side'] / res[False] - 1):.1f}%, weak-scaling bound {res[False] / res['side']:.3f})", flush=True)
