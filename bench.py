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
        # NVML (the library nvidia-smi reads), opened here -- outside the timed region -- and polled
        # every 10 ms, so a 35 ms timed region still gets several samples; else nvidia-smi / 100 ms
        self._nvml = None
        try:
            import pynvml as nvml
            nvml.nvmlInit()
            vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
            phys = int(vis[index]) if len(vis) > index and vis[index].strip().isdigit() else index
            self._h = nvml.nvmlDeviceGetHandleByIndex(phys)   # NVML counts physical devices
            self._mx = nvml.nvmlDeviceGetMaxClockInfo(self._h, nvml.NVML_CLOCK_SM)
            self._bits = [nvml.nvmlClocksThrottleReasonHwSlowdown, nvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                          nvml.nvmlClocksThrottleReasonSwThermalSlowdown, nvml.nvmlClocksThrottleReasonSwPowerCap]
            self._nvml = nvml
        except Exception:
            self._nvml = None

    def _run(self):
        nvml = self._nvml
        if nvml is not None:
            h, mx, bits = self._h, self._mx, self._bits
        while not self._stop.is_set():
            try:
                if nvml is not None:
                    sm = nvml.nvmlDeviceGetClockInfo(h, nvml.NVML_CLOCK_SM)
                    r = nvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.01 if nvml is not None else 0.1)
        if nvml is not None:
            try:
                nvml.nvmlShutdown()
            except Exception:
                pass

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
    """The reference's own functions (baseline/_ref install) or, if absent, the oracle port:
    (kind, step over a periodic grid, step of a ghost-padded block -> its interior)."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "momentlbm").exists():
        sys.path.insert(0, str(ref))
        import momentlbm.collision as RC
        import momentlbm.lattice as RL
        import momentlbm.moments as RM
        lat = RL.make_lattice("D3Q27")
        vel = [tuple(int(c) for c in v) for v in lat.velocities]

        def step(rho, mom, stress, tau):
            r, m, s = RC.collide_moments(rho, mom, stress, None, tau, 3)
            f = RM.reconstruct_distributions(r, m, s, lat)
            fs = np.stack([np.roll(f[i], shift=vel[i], axis=(0, 1, 2)) for i in range(27)])
            return RM.moments_from_distributions(fs, lat)

        def step_padded(rho, mom, stress, tau):
            r, m, s = RC.collide_moments(rho, mom, stress, None, tau, 3)
            f = RM.reconstruct_distributions(r, m, s, lat)
            nx, ny, nz = (d - 2 for d in rho.shape)
            fs = np.stack([f[i, 1 - cx:1 - cx + nx, 1 - cy:1 - cy + ny, 1 - cz:1 - cz + nz]
                           for i, (cx, cy, cz) in enumerate(vel)])
            return RM.moments_from_distributions(fs, lat)
        return "reference", step, step_padded
    from oracle import step as OS  # the CPU oracle port (only the bench's reference leg uses it)

    return ("port", lambda rho, mom, stress, tau: OS.fluid_step(rho, mom, stress, tau),
            lambda rho, mom, stress, tau: OS.step_padded(np.concatenate([rho[None], mom, stress]), tau))


def _initial_state(n, x0=0, nx=None):
    from paper_2602_05295_b200.geometry import evaluate_modes, turbulence_modes
    nx = n if nx is None else nx
    u = evaluate_modes(turbulence_modes(N_PER_GPU, seed=0), (nx, n, n), origin=(x0, 0, 0), global_dims=(n, n, n))
    rho = np.ones((nx, n, n))
    mom = rho * u
    stress = np.stack([mom[a] * u[b] for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))])
    return np.concatenate([rho[None], mom, stress])


TAU = 0.5 + 3e-4


def _single_core(n, warmup, steps):
    """One process, one BLAS thread: the reference step of an n^3 periodic box."""
    kind, step, _ = _ref_modules()
    st = _initial_state(n)
    rho, mom, stress = st[0], st[1:4], st[4:10]
    for _ in range(warmup):
        rho, mom, stress = step(rho, mom, stress, TAU)
    t0 = time.perf_counter()
    for _ in range(steps):
        rho, mom, stress = step(rho, mom, stress, TAU)
    return time.perf_counter() - t0, kind


# x-slab workers: the state lives in two file-backed float64 arrays (10, n, n, n) shared by all
# processes; each step every worker reads its planes x0-1 .. x1 (periodic halos, one plane per side)
# from the current array and writes its planes x0 .. x1-1 of the other one
_SLAB = {}


def _slab_init(paths, n):
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    _SLAB["bufs"] = [np.memmap(p, dtype=np.float64, mode="r+", shape=(10, n, n, n)) for p in paths]
    _SLAB["n"] = n
    _SLAB["step"] = _ref_modules()[2]


def _slab_step(args):
    x0, x1, src = args
    n = _SLAB["n"]
    a, b = _SLAB["bufs"][src], _SLAB["bufs"][1 - src]
    xs = [(x0 - 1) % n] + list(range(x0, x1)) + [x1 % n]
    blk = np.asarray(a[:, xs])
    blk = np.concatenate([blk[:, :, -1:], blk, blk[:, :, :1]], axis=2)       # periodic y ghosts
    blk = np.concatenate([blk[:, :, :, -1:], blk, blk[:, :, :, :1]], axis=3)  # periodic z ghosts
    r, m, s = _SLAB["step"](blk[0], blk[1:4], blk[4:10], TAU)
    b[0, x0:x1] = r
    b[1:4, x0:x1] = m
    b[4:10, x0:x1] = s
    return x1 - x0


def cpu_reference(steps, warmup=1, n=128, procs=None, single_n=64, single_steps=2):
    """Reference CPU path on the host cores: an n^3 periodic box split into
    `procs` x-slabs with one-plane halos, one process per core (steps timed after `warmup`), plus
    the single-core figure of a single_n^3 box (one process, OPENBLAS_NUM_THREADS=1)."""
    import multiprocessing as mp
    import tempfile
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"          # inherited by the spawned workers before numpy loads
    procs = procs or _cpu_procs(max(1, n // (os.cpu_count() or 1)) * n * n)
    procs = max(1, min(procs, n))
    ctx = mp.get_context("spawn")
    with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
        paths = [os.path.join(tmp, f"state{b}.f64") for b in range(2)]
        for p in paths:
            np.memmap(p, dtype=np.float64, mode="w+", shape=(10, n, n, n)).flush()
        init = np.memmap(paths[0], dtype=np.float64, mode="r+", shape=(10, n, n, n))
        init[:] = _initial_state(n)
        init.flush()
        del init
        bounds = np.linspace(0, n, procs + 1).astype(int)
        with ctx.Pool(procs, initializer=_slab_init, initargs=(paths, n)) as pool:
            src = 0
            for _ in range(warmup):
                pool.map(_slab_step, [(bounds[i], bounds[i + 1], src) for i in range(procs)])
                src = 1 - src
            t0 = time.perf_counter()
            for _ in range(steps):
                pool.map(_slab_step, [(bounds[i], bounds[i + 1], src) for i in range(procs)])
                src = 1 - src
            dt = time.perf_counter() - t0
    with ctx.Pool(1) as pool:
        t1, kind = pool.apply(_single_core, (single_n, 1, single_steps))
    return {"mlups": n ** 3 * steps / dt / 1e6, "kind": kind, "cores": procs, "timed_s": dt,
            "sample": f"{n}^3 periodic turbulence box in {procs} x-slabs with one-plane halos (one process per "
                      f"core, OPENBLAS_NUM_THREADS=1, shared file-backed state), {steps} timed steps after {warmup} warm-up",
            "single_core": {"value": round(single_n ** 3 * single_steps / t1 / 1e6, 3), "unit": "MLUPS", "cores": 1,
                            "sample": f"{single_n}^3 periodic box, {single_steps} timed steps, one process, "
                                      "OPENBLAS_NUM_THREADS=1"}}


def _cpu_procs(cells_per_proc):
    """All host cores, bounded by memory (~2.5 KB per cell in flight for the NumPy reference)."""
    procs = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
        procs = max(1, min(procs, int(0.5 * avail / (2500 * cells_per_proc))))
    except Exception:
        pass
    return procs


# ------------------------------------------------------------------------ GPU arm

def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _make(precision, world, rank, local, gnx=None, scene="box", halo="p2p"):
    """Weak scaling (default): (512 N) x 512 x 512, the same field on every slab.  Strong scaling
    (gnx given): gnx x 512 x 512 split into N x-slabs.  scene "vehicle"
    (SURVEY §8d configs 4/5): the procedural vehicle scaled to the global grid, inflow / outflow in
    x, periodic y / z, u_in = 0.1, nu = 1e-5, 16-bit with dither (fp32 beside)."""
    from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
    from paper_2602_05295_b200.geometry import turbulence_modes, vehicle_mask
    gnx = N_PER_GPU * world if gnx is None else gnx
    gdims = (gnx, N_PER_GPU, N_PER_GPU)
    mask = None
    if scene == "vehicle":
        cfg = SolverConfig(nu=1e-5, precision=precision, quant=QuantSpec(dither=precision == "q16"), device=local,
                           bc={"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")},
                           u_in=(0.1, 0.0, 0.0))
        modes = np.array([[0, 0, 0, 0.1, 0.0, 0.0, np.pi / 2]])   # uniform u_in
        mask = vehicle_mask(gdims, seed=0)
    else:
        cfg = SolverConfig(nu=1e-4, precision=precision, quant=QuantSpec(), device=local)
        modes = turbulence_modes(N_PER_GPU, seed=0)
        modes = modes.copy()
        modes[:, 0] *= gnx // N_PER_GPU   # wave numbers along x scale with the global nx
    if world > 1:
        from paper_2602_05295_b200.distributed import DistributedSolver
        ds = DistributedSolver(gdims, cfg, mask=mask, transport=halo)
        ds.solver.init_modes(modes)
        return ds, ds.solver
    import torch
    s = Solver(SimGrid(gdims, mask), cfg)
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


def _sustained(ds, s, world, local, seconds=2.0):
    """Steady-state throughput: about `seconds` of back-to-back steps after the burst-timed region
    (the chip settles at its power cap in long runs), with the clocks sampled during it."""
    import torch
    import torch.distributed as dist
    probe, _ = _timed(ds, s, 20, 0, world)
    n = max(50, int(seconds * 1e3 / (probe / 20)))
    if world > 1:   # every rank must run the same count
        t = torch.tensor([n], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n = int(t.item())
    with ClockSampler(local) as clk:
        ms, _ = _timed(ds, s, n, 0, world)
    return ms, n, clk.summary()


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
    e2e = None
    for precision in ("q16", "fp32"):
        ds, s = _make(precision, world, rank, local, gnx if strong else None, args.scene, args.halo)
        with ClockSampler(local) as clk:
            ms, launches = _timed(ds, s, args.steps, args.warmup, world)
        cells = (gnx // world) * N_PER_GPU * N_PER_GPU      # this rank's slab
        # roofline of the timed region itself: at N = 1 a fluid-only step is exactly one
        # fluid_interior launch (gpu_launches == steps), so the per-launch time is ms / steps;
        # at N > 1 a step is the edge + bulk launches of the slab and the figure covers both
        kt = ms / args.steps
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
                         "kernel_ms_from": "timed region (CUDA events on the launching stream) / steps",
                         "algorithmic_bytes_per_launch": cells * BYTES_PER_CELL[precision]},
        }
        sms, sn, sclk = _sustained(ds, s, world, local)
        results[precision]["sustained"] = {"value": round(cells * world * sn / (sms * 1e-3) / 1e6, 1),
                                           "unit": "MLUPS", "steps": sn, "seconds": round(sms * 1e-3, 2),
                                           "ms_per_step": round(sms / sn, 4), "clocks": sclk}
        if precision == "q16":
            e2e = _e2e(ds, s, world, max(args.steps, 200))
        if ds is not None:
            ds.close()
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
        "data": ("synthetic: procedural vehicle mask (geometry.vehicle_mask, seed 0), uniform inflow u = 0.1"
                 if args.scene == "vehicle" else "synthetic: solenoidal random Fourier modes 1<=|k|<=4, u_rms=0.05, seed 0"),
        "config": {"workload": (("SURVEY config 5 (strong scaling): " + (
                                   "procedural vehicle, inflow/outflow, 16-bit + dither" if args.scene == "vehicle"
                                   else "periodic fluid-only turbulence box") +
                                f" {STRONG_NX}x512x512 in x-slabs (fp32 measured beside)") if strong else
                               ("BASELINE configs[4]-style weak scaling: procedural vehicle over (512 N)x512x512, "
                                "16-bit + dither (fp32 beside)" if args.scene == "vehicle" else
                                "BASELINE configs[1]: periodic fluid-only turbulence box, 16-bit moments "
                                "(fp32 measured beside)")),
                   "grid_per_gpu": [gnx // world, N_PER_GPU, N_PER_GPU], "global_grid": [gnx, N_PER_GPU, N_PER_GPU],
                   "nu": 1e-4, "precision": "q16", "parallelism": f"x-slab dp{world}",
                   "halo": ("none" if world == 1 else
                            "CUDA IPC peer store" if args.halo == "ipc" else "torch.distributed P2P (NCCL)"),
                   "l2": f"inputs larger than L2: {2 * 20 * (gnx // world) * N_PER_GPU ** 2 / 1e9:.1f} GB (q16) / "
                         f"{2 * 40 * (gnx // world) * N_PER_GPU ** 2 / 1e9:.1f} GB (fp32) of double-buffered state "
                         "per GPU vs 126 MB L2"},
        "roofline": head["roofline"],
        "clocks": head["clocks"],
        "sustained": head["sustained"],
        "gpu_launches": head["launches"],
        "fp32": {"value": round(results["fp32"]["value"], 1), "unit": "MLUPS",
                 "ms_per_step": round(results["fp32"]["ms_per_step"], 4), "roofline": results["fp32"]["roofline"],
                 "clocks": results["fp32"]["clocks"], "gpu_launches": results["fp32"]["launches"],
                 "sustained": results["fp32"]["sustained"]},
        "paper_ref": {"value": 7097, "unit": "MLUPS", "what": "paper fluid-only 1024^3 16-bit on a 6912-core 80 GB GPU (PAPER.md:855)"},
    }
    if e2e is not None:
        line["e2e"] = e2e
    if cpu is not None:
        line["cpu_baseline"] = {"value": round(cpu["mlups"], 3), "unit": "MLUPS", "cores": cpu["cores"],
                                "kind": cpu["kind"], "sample": cpu["sample"], "single_core": cpu["single_core"]}
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's own CPU implementation on all host cores (rank 0 only): the 128^3 sample of
    the turbulence-box workload in x-slabs with one-plane halos, one process per core."""
    world, rank, local = _dist_env()
    if rank != 0:
        return
    n = int(os.environ.get("BENCH_REF_N", "128"))   # (the CPU tests shrink the sample)
    steps = max(1, min(args.steps, 10))      # bounded: the whole run stays within a few minutes
    res = cpu_reference(steps=steps, warmup=min(max(args.warmup, 1), 2), n=n, single_n=min(64, n))
    v = res["mlups"]
    line = {"metric": METRIC, "value": round(v, 3), "unit": "MLUPS", "n_gpus": args.gpus, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * res["timed_s"] / steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "impl": "reference",
            "data": "synthetic: solenoidal random Fourier modes 1<=|k|<=4, u_rms=0.05, seed 0",
            "config": {"workload": "BASELINE configs[1] sample: periodic fluid-only turbulence box "
                                   f"{n}^3 in x-slabs over the host cores", "precision": "float64 (reference NumPy)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "MLUPS", "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"], "single_core": res["single_core"]},
            "e2e": {"value": round(v, 3), "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch_cmd(argv, gpus, port=None):
    """`bench.py --gpus N` started without a launcher re-executes itself under torchrun with N
    ranks on this node (rendezvous on 127.0.0.1), so `--gpus N` always means N ranks."""
    if port is None:
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + list(argv)


def check_world(gpus, world, visible):
    """Fail loudly unless the launched world is exactly --gpus ranks with a GPU each."""
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}: the launched world must equal --gpus")
    if visible is not None and visible < gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but only {visible} CUDA device(s) are visible")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scene", default="box", choices=["box", "vehicle"],
                    help="box: periodic turbulence box (BASELINE configs[1]); vehicle: obstacle scene (configs 4/5)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: 2048x512x512 global grid split over the GPUs (default: weak, 512^3 per GPU)")
    ap.add_argument("--halo", default="p2p", choices=["p2p", "ipc"],
                    help="N > 1: halo planes as NCCL send/recv (p2p) or stored into the neighbours' ghost "
                         "planes through CUDA IPC mappings (ipc, DESIGN.md §7)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(subprocess.call(self_launch_cmd(sys.argv[1:], args.gpus)))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        check_world(args.gpus, world, None)     # CPU arm: rank 0 runs, the others exit 0
    else:
        import torch
        check_world(args.gpus, world, torch.cuda.device_count())
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
