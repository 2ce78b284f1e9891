"""Ad-hoc GPU bring-up checks (development tool; the pytest suite holds the real tests)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np
from oracle import codec, step as ostep
from oracle.moments import neq_decompose
from paper_2602_05295_b200 import QuantSpec, SimGrid, Solver, SolverConfig
from paper_2602_05295_b200.geometry import sphere_mask


def rel(got, ref):
    return [float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300)) for g, r in zip(got, ref)]


def per_comp(got, ref):
    g = np.concatenate([got[0][None], got[1], got[2]])
    r = np.concatenate([ref[0][None], ref[1], ref[2]])
    return [float(np.linalg.norm(g[k] - r[k]) / max(np.linalg.norm(r[k]), 1e-300)) for k in range(10)]


def check_random(shape, steps=1, ref_kernel=False):
    rho, mom, st = ostep.random_state(shape, seed=1, drho=0.05, umax=0.05, sneq=0.005)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid(shape), cfg) as s:
        s.set_moments(rho, mom, st)
        if ref_kernel:
            s.step_reference(steps)
        else:
            s.step(steps)
        got = s.moments()
    ref = (rho, mom, st)
    for _ in range(steps):
        ref = ostep.fluid_step(*ref, cfg.tau)
    print(f"random {shape} steps={steps} refkernel={ref_kernel}: max per-comp rel {max(per_comp(got, ref)):.3e}", flush=True)


def check_tgv(n=64, steps=20):
    rho, mom, st = ostep.taylor_green(n)
    cfg = SolverConfig(nu=0.01)
    with Solver(SimGrid((n, n, n)), cfg) as s:
        s.set_moments(rho, mom, st)
        s.step(steps)
        got = s.moments()
    ref = ostep.run(rho, mom, st, cfg.tau, steps)
    pc = per_comp(got, ref)
    print(f"TGV {n}^3 {steps} steps: per-comp rel {['%.2e' % v for v in pc]}", flush=True)


def check_q16(shape=(16, 16, 16), steps=1, dither=False):
    rho, mom, st = ostep.random_state(shape, seed=2, drho=0.05, umax=0.05, sneq=0.005)
    q = QuantSpec(dither=dither)
    cfg = SolverConfig(nu=0.02, precision="q16", quant=q, seed=7)
    w, _ = codec.encode_state(rho, mom, neq_decompose(rho, mom, st))
    with Solver(SimGrid(shape), cfg) as s:
        s.codes = w
        for _ in range(steps):
            s.step(1)
        got = s.codes
    ref = w
    for k in range(steps):
        ref, _ = ostep.fluid_step_q16(ref, cfg.tau, k, dither=dither, seed=7)
    d = np.abs(codec.unpack(got).astype(np.int64) - codec.unpack(ref).astype(np.int64))
    print(f"q16 {shape} steps={steps} dither={dither}: max LSB diff {d.max()}, frac nonzero {np.mean(d > 0):.4f}", flush=True)


def check_sphere(shape=(48, 32, 32), steps=3):
    mask = sphere_mask(shape, (16, 16, 16), 6)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0))
    obc = ostep.BC(x=bc["x"], y=bc["y"], z=bc["z"], u_in=(0.05, 0, 0))
    cells, masks = ostep.boundary_lists(mask, obc)
    rho = np.ones(shape)
    u = np.zeros((3,) + shape); u[0] = 0.05
    u[:, mask.astype(bool)] = 0
    mom = rho * u
    st = np.stack([mom[a] * u[b] for a, b in ((0,0),(0,1),(0,2),(1,1),(1,2),(2,2))])
    with Solver(SimGrid(shape, mask), cfg) as s:
        gc, gm = s.boundary()
        print(f"sphere lists: n={len(cells)} gpu n={len(gc)} cells equal={np.array_equal(gc, cells)} masks equal={np.array_equal(gm, masks)}", flush=True)
        s.set_moments(rho, mom, st)
        stt = s.step(steps)
        got = s.moments()
    ref = (rho, mom, st)
    for _ in range(steps):
        ref = ostep.fluid_step(*ref, cfg.tau, obc, None, mask)
    fl = ~mask.astype(bool)
    g = [got[0][fl], got[1][:, fl], got[2][:, fl]]
    r = [ref[0][fl], ref[1][:, fl], ref[2][:, fl]]
    print(f"sphere {steps} steps: rel {['%.2e' % v for v in rel(g, r)]}; mass gpu {stt.mass:.6f} oracle {ref[0][fl].sum():.6f}", flush=True)


def bench(n, precision, steps=10):
    cfg = SolverConfig(nu=1e-4, precision=precision)
    from paper_2602_05295_b200.geometry import turbulence_modes
    with Solver(SimGrid((n, n, n)), cfg) as s:
        s.init_modes(turbulence_modes(n))
        s.step(2)
        t = time.perf_counter()
        s.step_async(steps)
        s.read_stats()
        dt = (time.perf_counter() - t) / steps
        print(f"bench {n}^3 {precision}: {dt*1e3:.3f} ms/step, {n**3/dt/1e6:.0f} MLUPS", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["all"]
    if "all" in what or "small" in what:
        check_random((16, 16, 16))
        check_random((16, 16, 16), ref_kernel=True)
        check_random((20, 30, 68), steps=3)
        check_random((20, 30, 68), steps=3, ref_kernel=True)
        check_q16()
        check_q16(dither=True)
        check_q16((12, 20, 64), steps=5)
        check_sphere()
    if "all" in what or "tgv" in what:
        check_tgv(64, 20)
    if "all" in what or "bench" in what:
        for n in (256, 512):
            for p in ("fp32", "q16"):
                bench(n, p)
