"""Full-size properties on the GPU (BASELINE.json configs 2-5 sizes), where the float64 oracle
cannot run the whole grid: crop parity, shift equivariance, conservation, uniform-flow
invariance, and the x-slab decomposition emulated on one GPU (bitwise vs one domain)."""

import numpy as np
import pytest

from oracle import codec
from oracle import step as OS
from oracle.moments import neq_decompose, neq_recompose
from paper_2602_05295_b200 import QuantSpec, SimGrid, Slab, Solver, SolverConfig
from paper_2602_05295_b200.distributed import device_view, partition
from paper_2602_05295_b200.geometry import sphere_mask, turbulence_modes, vehicle_mask

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_512_crop_parity(precision):
    """Config 2 (512^3 turbulence box): 2 GPU steps vs the oracle on a 20^3 crop."""
    n, steps, h = 512, 2, 2
    cfg = SolverConfig(nu=1e-4, precision=precision)
    with Solver(SimGrid((n, n, n)), cfg) as s:
        s.init_modes(turbulence_modes(n))
        x0, y0, z0, c = 300, 17, 499, 20     # the z box wraps across the periodic face
        init = s.moments_box(x0 - h, c + 2 * h, y0 - h, c + 2 * h, z0 - h, c + 2 * h)
        s.step(steps)
        got = s.moments_box(x0, c, y0, c, z0, c)
    if precision == "fp32":
        ref = init
        for _ in range(steps):
            padded = np.concatenate([ref[0][None], ref[1], ref[2]])
            r, m, st = OS.step_padded(padded, cfg.tau)
            ref = (r, m, st)
        for g, r in zip(got, ref):
            assert np.linalg.norm(g - r) / np.linalg.norm(r) <= 1e-5
    else:
        words = codec.encode_state(init[0], init[1], neq_decompose(*init))[0]
        for k in range(steps):
            rho, mom, sn = codec.decode_state(words)
            padded = np.concatenate([rho[None], mom, neq_recompose(rho, mom, sn)])
            r, m, st = OS.step_padded(padded, cfg.tau)
            words = codec.encode_state(r, m, neq_decompose(r, m, st))[0]
        ref_codes = codec.unpack(words)
        got_codes = codec.unpack(codec.encode_state(got[0], got[1], neq_decompose(*got))[0])
        assert np.abs(got_codes.astype(np.int64) - ref_codes.astype(np.int64)).max() <= 2


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_shift_equivariance_bitwise(precision):
    """Every cell runs the same arithmetic wherever its tile falls: shifting the input by a
    lattice vector shifts the output bit-for-bit (size-independent parity property)."""
    shape = (96, 80, 124)
    state = OS.random_state(shape, seed=11, drho=0.05, umax=0.05, sneq=0.005)
    sh = (17, 29, 61)
    cfg = SolverConfig(nu=0.01, precision=precision)
    outs = []
    for shift in ((0, 0, 0), sh):
        st = tuple(np.roll(a, shift, axis=(-3, -2, -1)) for a in state)
        with Solver(SimGrid(shape), cfg) as s:
            s.set_moments(*st)
            s.step(3)
            outs.append(s.codes if precision == "q16" else np.concatenate([x.reshape(-1, *shape) for x in s.moments()]))
    assert np.array_equal(np.roll(outs[0], sh, axis=(-3, -2, -1)), outs[1])


def test_512_periodic_conservation_and_stats():
    n = 512
    with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-4)) as s:
        s.init_modes(turbulence_modes(n))
        st0 = s.step(1)
        st1 = s.step(20)
    assert abs(st1.mass - st0.mass) / st0.mass < 1e-7
    np.testing.assert_allclose(st1.momentum, st0.momentum, atol=1e-6 * n ** 3 * 0.05)
    assert 0.05 < st1.max_u < 0.5


def test_uniform_flow_invariant_full_size():
    n = 256
    modes = np.array([[0, 0, 0, 0.05, -0.02, 0.03, np.pi / 2]])   # sin(pi/2) = 1: uniform u
    with Solver(SimGrid((n, n, n)), SolverConfig(nu=1e-3)) as s:
        s.init_modes(modes)
        a = s.moments_box(0, 8, 100, 8, 60, 8)
        s.step(5)
        b = s.moments_box(0, 8, 100, 8, 60, 8)
    for x, y in zip(a, b):
        np.testing.assert_allclose(y, x, atol=2e-7)


def _emulate_slabs(gshape, cfg, world, init, mask=None, steps=3, x_periodic=True):
    """Run `world` slab contexts on one GPU with device-to-device halo copies between steps."""
    import torch
    plans = partition(gshape[0], world, x_periodic)
    solvers = []
    for p in plans:
        sl = slice(p.x0, p.x0 + p.nx)
        s = Solver(SimGrid((p.nx,) + gshape[1:]), cfg,
                   slab=Slab(p.x0, gshape[0], p.lo is not None, p.hi is not None))
        if mask is not None:
            lo = mask[(p.x0 - 1) % gshape[0]] if p.lo is not None else None
            hi = mask[(p.x0 + p.nx) % gshape[0]] if p.hi is not None else None
            s.set_mask(mask[sl], lo, hi)
        s.set_moments(init[0][sl], init[1][:, sl], init[2][:, sl])
        solvers.append(s)
    for _ in range(steps):
        views = []
        for s in solvers:
            (sl_, sh_, rl, rh), nb = s.halo_planes()
            views.append([device_view(p, nb) for p in (sl_, sh_, rl, rh)])
        for p, v in zip(plans, views):
            if p.lo is not None:
                v[2].copy_(views[p.lo][1])     # my recv_lo <- lower neighbour's last plane
            if p.hi is not None:
                v[3].copy_(views[p.hi][0])     # my recv_hi <- upper neighbour's first plane
        torch.cuda.synchronize()
        for s in solvers:
            s.step(1)
    out = [s.moments() for s in solvers]
    for s in solvers:
        s.close()
    return tuple(np.concatenate([o[k] for o in out], axis=-3) for k in range(3))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_slab_decomposition_bitwise_periodic(world):
    gshape = (40, 24, 32)
    state = OS.random_state(gshape, seed=12, drho=0.05, umax=0.05, sneq=0.005)
    cfg = SolverConfig(nu=0.02)
    with Solver(SimGrid(gshape), cfg) as s:
        s.set_moments(*state)
        s.step(3)
        ref = s.moments()
    got = _emulate_slabs(gshape, cfg, world, state)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_slab_decomposition_bitwise_solids(precision):
    gshape = (48, 24, 32)
    mask = sphere_mask(gshape, (20, 11.5, 15.5), 6)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0), precision=precision,
                       quant=QuantSpec(dither=True), seed=3)
    rho = np.ones(gshape)
    mom = np.zeros((3,) + gshape)
    mom[0] = 0.05
    mom[:, mask.astype(bool)] = 0
    state = (rho, mom, neq_recompose(rho, mom, np.zeros((6,) + gshape)))
    with Solver(SimGrid(gshape, mask), cfg) as s:
        s.set_moments(*state)
        s.step(3)
        ref = s.moments()
    got = _emulate_slabs(gshape, cfg, 3, state, mask=mask, x_periodic=False)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


@pytest.mark.parametrize("precision", ["fp32", "q16"])
def test_slab_decomposition_bitwise_d3q19(precision):
    """D3Q19 (two-chain interior kernel + 19-link compacted kernels): 3 slabs equal one domain
    bitwise, with a solid sphere, inflow/outflow and walls."""
    gshape = (48, 24, 32)
    mask = sphere_mask(gshape, (20, 11.5, 15.5), 6)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0), precision=precision, lattice="D3Q19",
                       quant=QuantSpec(dither=True), seed=5)
    rho = np.ones(gshape)
    mom = np.zeros((3,) + gshape)
    mom[0] = 0.05
    mom[:, mask.astype(bool)] = 0
    state = (rho, mom, neq_recompose(rho, mom, np.zeros((6,) + gshape)))
    with Solver(SimGrid(gshape, mask), cfg) as s:
        s.set_moments(*state)
        s.step(3)
        ref = s.moments()
    got = _emulate_slabs(gshape, cfg, 3, state, mask=mask, x_periodic=False)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


def test_vehicle_scene_lists_and_step():
    """Config 4 shape, scaled: procedural vehicle mask, q16 + dither, inflow/outflow."""
    gshape = (250, 100, 100)
    mask = vehicle_mask(gshape, seed=0)
    frac = mask.mean()
    assert 0.005 < frac < 0.06
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("periodic", "periodic")}
    obc = OS.BC(x=bc["x"], y=bc["y"], z=bc["z"], u_in=(0.1, 0, 0))
    cfg = SolverConfig(nu=1e-5, bc=bc, u_in=(0.1, 0, 0), precision="q16", quant=QuantSpec(dither=True))
    cells, masks = OS.boundary_lists(mask, obc)
    with Solver(SimGrid(gshape, mask), cfg) as s:
        gc, gm = s.boundary()
        assert np.array_equal(gc, cells) and np.array_equal(gm, masks)
        s.init_modes(np.array([[0, 0, 0, 0.1, 0, 0, np.pi / 2]]))
        st = s.step(20)
    assert np.isfinite(st.mass) and st.max_u < 0.5
    assert st.saturation[0] < 1e-3 * st.n_fluid


def _sphere_state(gshape, mask):
    rho = np.ones(gshape)
    mom = np.zeros((3,) + gshape)
    mom[0] = 0.05
    mom[:, mask.astype(bool)] = 0
    return rho, mom, neq_recompose(rho, mom, np.zeros((6,) + gshape))


@pytest.mark.parametrize("precision,mesh", [("fp32", False), ("q16", False), ("q16", True)])
def test_range_split_step_bitwise(precision, mesh):
    """The overlapped multi-GPU schedule's split step -- edge planes (0, 1), (nx-1, nx), then the
    bulk (1, nx-1) -- equals one full step bitwise (solids / triangle mesh, inflow/outflow,
    walls, dither); statistics agree to summation order."""
    from oracle.mesh import icosphere
    gshape = (40, 24, 32)
    mask = sphere_mask(gshape, (20, 11.5, 15.5), 6)
    bc = {"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")}
    cfg = SolverConfig(nu=0.02, bc=bc, u_in=(0.05, 0, 0), precision=precision,
                       quant=QuantSpec(dither=True), seed=3)
    state = _sphere_state(gshape, mask)
    nx = gshape[0]
    res = []
    for split in (False, True):
        with Solver(SimGrid(gshape, None if mesh else mask), cfg) as s:
            if mesh:
                v, f = icosphere((20, 11.5, 15.5), 6.3, 2)
                s.set_mesh(v, f)
            s.set_moments(*state)
            for k in range(3):
                if split:
                    s.step_begin(with_stats=k == 2)
                    for a, b in ((0, 1), (nx - 1, nx), (1, nx - 1)):
                        s.step_range(a, b)
                    s.step_end()
                else:
                    s.step_async(1, with_stats=k == 2)
            st = s.read_stats()
            res.append((s.get_state(), st))
    assert np.array_equal(res[0][0], res[1][0])
    a, b = res[0][1], res[1][1]
    assert a.mass == pytest.approx(b.mass, rel=1e-9) and a.max_u == b.max_u   # fp32 partial sums
    assert np.array_equal(a.saturation, b.saturation)
    np.testing.assert_allclose(a.momentum, b.momentum, rtol=1e-9, atol=1e-6)


def test_distributed_solver_single_rank_overlap_path():
    """DistributedSolver with one rank (no neighbours): the overlapped split step through the
    real C-ABI equals Solver.step_async bitwise."""
    from paper_2602_05295_b200.distributed import DistributedSolver
    gshape = (32, 16, 32)
    cfg = SolverConfig(nu=0.01, precision="q16")
    modes = turbulence_modes(32, seed=1)
    with Solver(SimGrid(gshape), cfg) as s:
        s.init_modes(modes)
        s.step_async(4)
        ref = s.get_state()
    ds = DistributedSolver(gshape, cfg, rank=0, world=1)
    try:
        ds.solver.init_modes(modes)
        ds.step(4, stats=False)
        got = ds.solver.get_state()
    finally:
        ds.solver.close()
    assert np.array_equal(got, ref)
