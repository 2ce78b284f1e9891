"""Benchmark of the HOME-LBM D3Q27 fluid step on B200 (BASELINE.json metric: MLUPS and % of
the HBM roofline, fp32 vs 16-bit moments).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): periodic fluid-only turbulence box, 512^3 cells per GPU
(weak scaling: the global grid is (512 N) x 512 x 512, x-slab decomposed, one process per
GPU, NCCL halo exchange).  Synthetic initial state: solenoidal random Fourier modes,
1 <= |k| <= 4, u_rms = 0.05, seed 0; nu = 1e-4.  The headline `value` is the 16-bit path;
the fp32 path is measured in the same run and reported beside it.

``--strong`` runs SURVEY.md §8d config 5 instead: a 2048 x 512 x 512 global grid split into N
x-slabs (strong scaling).

Emits ONE JSON line on rank 0.  `--impl reference` times the reference's own CPU
implementation of the step (momentlbm from baseline/_ref, else the oracle port) on the
host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MLUPS (1/2/4/8 B200) and % of HBM roofline, fp32 vs 16-bit moments"
BYTES_PER_CELL = {"q16": 40, "fp32": 80}     # algorithmic HBM bytes per cell update
N_PER_GPU = 512
STRONG_NX = 2048      # SURVEY.md §8d config 5 global x extent (bench.py --strong)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def ncu_traffic(precision):
    """dram__bytes_read.sum + dram__bytes_write.sum per fluid_interior launch, from the committed
    ncu --set full capture of this workload (profiles/*_traffic.json)."""
    best = None
    for f in sorted((ROOT / "profiles").glob("*_traffic.json")):
        try:
            d = json.loads(f.read_text())
            if precision in d:
                best = d[precision]
        except Exception:
            pass
    return best


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------ reference arm (CPU)

def _ref_modules():
    """The reference's own functions (baseline/_ref install) or, if absent, the oracle port."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "momentlbm").exists():
        sys.path.insert(0, str(ref))
        import momentlbm.collision as RC
        import momentlbm.lattice as RL
        import momentlbm.moments as RM
        lat = RL.make_lattice("D3Q27")

        def step(rho, mom, stress, tau):
            r, m, s = RC.collide_moments(rho, mom, stress, None, tau, 3)
            f = RM.reconstruct_distributions(r, m, s, lat)
            fs = np.stack([np.roll(f[i], shift=tuple(lat.velocities[i]), axis=(0, 1, 2)) for i in range(27)])
            return RM.moments_from_distributions(fs, lat)
        return "reference", step
    from oracle import step as OS  # the CPU oracle port (only the bench's reference leg uses it)

    return "port", lambda rho, mom, stress, tau: OS.fluid_step(rho, mom, stress, tau)


def _cpu_worker(args):
    n, warmup, steps, seed = args
    kind, step = _ref_modules()
    from paper_2602_05295_b200.geometry import evaluate_modes, turbulence_modes
    u = evaluate_modes(turbulence_modes(N_PER_GPU, seed=0), (n, n, n), origin=(seed * n, 0, 0),
                       global_dims=(N_PER_GPU,) * 3)
    rho = np.ones((n, n, n))
    mom = rho * u
    stress = np.stack([mom[a] * u[b] for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])
    tau = 0.5 + 3e-4
    for _ in range(warmup):
        rho, mom, stress = step(rho, mom, stress, tau)
    t0 = time.perf_counter()
    for _ in range(steps):
        rho, mom, stress = step(rho, mom, stress, tau)
    return time.perf_counter() - t0, n ** 3 * steps, kind


def _cpu_procs(n):
    """All host cores, bounded by memory (~2 KB per cell in flight for the NumPy reference)."""
    procs = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
        procs = max(1, min(procs, int(0.5 * avail / (2500 * n ** 3))))
    except Exception:
        pass
    return procs


def cpu_reference(steps, warmup=1, n=48, procs=None):
    """Reference CPU path on the host cores: `procs` processes, each stepping an independent n^3
    periodic block of the same synthetic workload (warmup untimed steps, then `steps` timed)."""
    import multiprocessing as mp
    procs = procs or _cpu_procs(n)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"          # inherited by the spawned workers before numpy loads
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(n, warmup, steps, i) for i in range(procs)])
    cells = sum(r[1] for r in res)
    per_proc = max(r[0] for r in res)
    return {"mlups": cells / per_proc / 1e6, "kind": res[0][2], "cores": procs, "timed_s": per_proc,
            "sample": f"{procs} processes x {steps} timed steps (after {warmup} warm-up) of an independent "
                      f"{n}^3 periodic block each, OPENBLAS_NUM_THREADS=1"}


# ------------------------------------------------------------------------ GPU arm

def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _make(precision, world, rank, local, gnx=None):
    """Weak scaling (default): (512 N) x 512 x 512, the same field on every slab.  Strong scaling
    (gnx given): gnx x 512 x 512 split into N x-slabs."""
    from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
    from paper_2602_05295_b200.geometry import turbulence_modes
    cfg = SolverConfig(nu=1e-4, precision=precision, quant=QuantSpec(), device=local)
    gnx = N_PER_GPU * world if gnx is None else gnx
    gdims = (gnx, N_PER_GPU, N_PER_GPU)
    modes = turbulence_modes(N_PER_GPU, seed=0)
    modes = modes.copy()
    modes[:, 0] *= gnx // N_PER_GPU   # wave numbers along x scale with the global nx
    if world > 1:
        from paper_2602_05295_b200.distributed import DistributedSolver
        ds = DistributedSolver(gdims, cfg)
        ds.solver.init_modes(modes)
        return ds, ds.solver
    import torch
    s = Solver(SimGrid(gdims), cfg)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.init_modes(modes)
    return None, s


def _timed(ds, s, steps, warmup, world):
    """Device time of `steps` steps (CUDA events on the launching stream), max over ranks."""
    import torch
    import torch.distributed as dist

    def run(n):
        if ds is not None:
            ds.step(n, stats=False)
        else:
            s.step_async(n, with_stats=False)

    run(warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = s.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(steps)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = s.launches - l0
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, launches


def _kernel_time(s, reps=10):
    """Average fluid_interior launch duration on this rank (one launch per fluid-only step)."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.step_async(2, with_stats=False)
    torch.cuda.synchronize()
    e0.record()
    s.step_async(reps, with_stats=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _e2e(ds, s, world, steps):
    """End to end through the public API with HOST buffers: upload the packed initial state
    from pinned host memory (set_codes), `steps` x step(1) -- each reads StepStats back to the
    host (all-reduced over ranks when N > 1) -- and download the final packed state, all inside
    the timed region.  Runs on the q16 headline path."""
    import torch
    import torch.distributed as dist
    nx, ny, nz = s.grid.dims
    host = torch.empty((5, nx, ny, nz), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    out = torch.empty((5, nx, ny, nz), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    s.get_codes(host)                              # the initial condition, staged on the host
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    s.codes = host                                 # H2D: packed state from pinned host memory
    for _ in range(steps):
        st = ds.step(1) if ds is not None else s.step(1)    # C-ABI step + D2H StepStats
    s.get_codes(out)                               # D2H: packed state into pinned host memory
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    state_bytes = 5 * 4 * nx * ny * nz
    return {"value": round(nx * ny * nz * world * steps / dt / 1e6, 1), "unit": "MLUPS",
            "h2d_bytes_per_step": int(state_bytes / steps),
            "d2h_bytes_per_step": int(state_bytes / steps + C_STATS_BYTES),
            "steps": steps,
            "note": "pinned host codes -> set_codes -> steps x step(1) with StepStats to the host each step "
                    "-> get_codes to pinned host memory; wall clock, max over ranks",
            "final_mass": st.mass}


C_STATS_BYTES = 8 + 3 * 8 + 8 + 3 * 8 + 8 + 10 * 8 + 8 + 8   # hlbm_stats read back per step


def run_ours(args):
    import torch
    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, peak_kind = peaks()
    strong = args.strong
    gnx = STRONG_NX if strong else N_PER_GPU * world
    if gnx % world:
        raise SystemExit(f"strong scaling needs {STRONG_NX} planes divisible by the GPU count")
    results = {}
    for precision in ("q16", "fp32"):
        ds, s = _make(precision, world, rank, local, gnx if strong else None)
        with ClockSampler(local) as clk:
            ms, launches = _timed(ds, s, args.steps, args.warmup, world)
        kt = _kernel_time(s)
        cells = (gnx // world) * N_PER_GPU * N_PER_GPU      # this rank's slab
        achieved = cells * BYTES_PER_CELL[precision] / (kt * 1e-3) / 1e9
        tr = ncu_traffic(precision)
        results[precision] = {
            "value": cells * world * args.steps / (ms * 1e-3) / 1e6,
            "ms_per_step": ms / args.steps,
            "launches": launches,
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": tr, "peak_kind": peak_kind,
                         "kernel": "fluid_interior", "kernel_ms": round(kt, 4),
                         "algorithmic_bytes_per_launch": cells * BYTES_PER_CELL[precision]},
        }
        if precision == "q16":
            e2e = _e2e(ds, s, world, max(args.steps, 50))
        if ds is not None:
            ds.solver.close()
        else:
            s.close()
    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_reference(steps=3)
    head = results["q16"]
    line = {
        "metric": METRIC, "value": round(head["value"], 1), "unit": "MLUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["ms_per_step"], 4),
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: solenoidal random Fourier modes 1<=|k|<=4, u_rms=0.05, seed 0",
        "config": {"workload": ("SURVEY config 5 (strong scaling): periodic fluid-only turbulence box "
                                f"{STRONG_NX}x512x512 in x-slabs, 16-bit moments (fp32 measured beside)") if strong else
                               ("BASELINE configs[1]: periodic fluid-only turbulence box, 16-bit moments "
                                "(fp32 measured beside)"),
                   "grid_per_gpu": [gnx // world, N_PER_GPU, N_PER_GPU], "global_grid": [gnx, N_PER_GPU, N_PER_GPU],
                   "nu": 1e-4, "precision": "q16", "parallelism": f"x-slab dp{world}",
                   "l2": "inputs larger than L2: 2.7 GB (q16) / 5.4 GB (fp32) state per GPU vs 126 MB L2"},
        "roofline": head["roofline"],
        "clocks": head["clocks"],
        "gpu_launches": head["launches"],
        "fp32": {"value": round(results["fp32"]["value"], 1), "unit": "MLUPS",
                 "ms_per_step": round(results["fp32"]["ms_per_step"], 4), "roofline": results["fp32"]["roofline"],
                 "clocks": results["fp32"]["clocks"], "gpu_launches": results["fp32"]["launches"]},
        "paper_ref": {"value": 7097, "unit": "MLUPS", "what": "paper fluid-only 1024^3 16-bit on a 6912-core 80 GB GPU (PAPER.md:855)"},
    }
    if e2e is not None:
        line["e2e"] = e2e
    if cpu is not None:
        line["cpu_baseline"] = {"value": round(cpu["mlups"], 3), "unit": "MLUPS", "cores": cpu["cores"],
                                "kind": cpu["kind"], "sample": cpu["sample"]}
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's own CPU implementation on all host cores (rank 0 only)."""
    world, rank, local = _dist_env()
    if rank != 0:
        return
    n = 48
    steps = max(1, min(args.steps, 20))      # bounded: the whole run stays within a few minutes
    res = cpu_reference(steps=steps, warmup=min(max(args.warmup, 1), 3), n=n)
    v = res["mlups"]
    line = {"metric": METRIC, "value": round(v, 3), "unit": "MLUPS", "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * res["timed_s"] / steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "impl": "reference",
            "data": "synthetic: solenoidal random Fourier modes 1<=|k|<=4, u_rms=0.05, seed 0",
            "config": {"workload": "BASELINE configs[1] sample: periodic fluid-only turbulence box blocks "
                                   f"({n}^3 per host core)", "precision": "float64 (reference NumPy)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "MLUPS", "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"]},
            "e2e": {"value": round(v, 3), "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: 2048x512x512 global grid split over the GPUs (default: weak, 512^3 per GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
