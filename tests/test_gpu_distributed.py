"""DistributedSolver driving the real Solver (libhlbm.so) on more than one rank: two or three gloo
processes share the one B200 of the test box, the halo planes are staged through host memory
(the same overlapped schedule as the NCCL path: edge planes on a side stream, exchange of the
written edge planes, bulk), and the gathered state must equal a single-domain run bitwise.
Divergence on one rank must raise FloatingPointError on every rank (no deadlock in the
statistics reduction)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GDIMS = (40, 24, 32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _config(kind):
    from paper_2602_05295_b200 import QuantSpec, SolverConfig
    if kind == "periodic_q16":
        return SolverConfig(nu=0.02, precision="q16", quant=QuantSpec(dither=True), seed=3)
    if kind == "periodic_d3q19":
        return SolverConfig(nu=0.02, precision="q16", quant=QuantSpec(dither=True), seed=3, lattice="D3Q19")
    if kind == "channel_fp32":
        return SolverConfig(nu=0.02, bc={"x": ("inflow", "outflow"), "y": ("periodic", "periodic"),
                                         "z": ("wall", "wall")}, u_in=(0.05, 0, 0))
    return SolverConfig(nu=0.02, precision="q16", quant=QuantSpec(dither=True), seed=3,
                        bc={"x": ("inflow", "outflow"), "y": ("periodic", "periodic"), "z": ("wall", "wall")},
                        u_in=(0.05, 0, 0))


def _inputs(kind):
    from oracle import step as OS
    from paper_2602_05295_b200.geometry import sphere_mask
    state = OS.random_state(GDIMS, seed=21, drho=0.04, umax=0.05, sneq=0.004)
    mask = None if kind.startswith("periodic") else sphere_mask(GDIMS, (19, 11.5, 15.5), 5)
    return state, mask


def _worker(rank, world, port, kind, steps, out, transport="p2p"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05295_b200.distributed import DistributedSolver
        torch.cuda.set_device(0)
        cfg = _config(kind)
        state, mask = _inputs(kind)
        ds = DistributedSolver(GDIMS, cfg, mask=mask, transport=transport)
        p = ds.plan
        sl = slice(p.x0, p.x0 + p.nx)
        ds.solver.set_moments(state[0][sl], state[1][:, sl], state[2][:, sl])
        if transport == "ipc" and rank == 0:
            # set_moments swaps the rank's buffers: rank 0's current index now differs from the
            # one its neighbours mapped at construction -- the prime must re-align them
            ds.solver.set_moments(state[0][sl], state[1][:, sl], state[2][:, sl])
        if transport == "ipc":
            # a host-side state change mid-run (set_moments swaps the rank's buffers) re-primes
            ds.step(steps // 2, stats=False)
            ds.solver.set_state(ds.solver.get_state())
            st = ds.step(steps - steps // 2)
        else:
            st = ds.step(steps)
        res = ds.solver.get_state()
        out[rank] = (p.x0, res, st.mass, int(st.n_fluid))
        ds.close()
        ds.solver.close()
    finally:
        dist.destroy_process_group()


def _single(kind, steps):
    from paper_2602_05295_b200 import SimGrid, Solver
    state, mask = _inputs(kind)
    with Solver(SimGrid(GDIMS, mask), _config(kind)) as s:
        s.set_moments(*state)
        st = s.step(steps)
        return s.get_state(), st


@pytest.mark.parametrize("world,kind", [(2, "periodic_q16"), (2, "channel_fp32"), (3, "channel_q16")])
def test_distributed_solver_real_slabs_bitwise(world, kind):
    steps = 4
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, kind, steps, out), nprocs=world, join=True)
    ref, st = _single(kind, steps)
    got = np.zeros_like(ref)
    mass = 0.0
    for r in range(world):
        x0, res, m, nf = out[r]
        got[:, x0:x0 + res.shape[1]] = res
        mass = m
        assert nf == st.n_fluid
    assert np.array_equal(got, ref)
    assert mass == pytest.approx(st.mass, rel=1e-9)


def _jitter_worker(rank, world, port, steps, out):
    """transport="ipc" with per-rank host delays between steps: ranks issue their steps out of
    phase, so a rank's stream waits on neighbour events recorded at different host times."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import time
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05295_b200.distributed import DistributedSolver
        torch.cuda.set_device(0)
        state, _ = _inputs("periodic_q16")
        ds = DistributedSolver(GDIMS, _config("periodic_q16"), transport="ipc")
        p = ds.plan
        sl = slice(p.x0, p.x0 + p.nx)
        ds.solver.set_moments(state[0][sl], state[1][:, sl], state[2][:, sl])
        rng = np.random.default_rng(rank)
        for _ in range(steps):
            time.sleep(float(rng.uniform(0, 0.004)))
            ds.step(1, stats=False)
        out[rank] = (p.x0, ds.solver.get_state())
        ds.close()
        ds.solver.close()
    finally:
        dist.destroy_process_group()


def test_ipc_peer_store_with_host_jitter():
    steps = 24
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_jitter_worker, args=(3, port, steps, out), nprocs=3, join=True)
    ref, _ = _single("periodic_q16", steps)
    got = np.zeros_like(ref)
    for r in range(3):
        x0, res = out[r]
        got[:, x0:x0 + res.shape[1]] = res
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("world,kind", [(2, "periodic_q16"), (3, "periodic_q16"), (3, "channel_q16"),
                                        (2, "channel_fp32"), (2, "periodic_d3q19")])
def test_distributed_solver_ipc_peer_store_bitwise(world, kind):
    """transport="ipc": CUDA IPC mappings of the neighbours' buffers, edge planes pushed straight
    into their ghost planes, interprocess events between the ranks' streams."""
    steps = 7
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, kind, steps, out, "ipc"), nprocs=world, join=True)
    ref, st = _single(kind, steps)
    got = np.zeros_like(ref)
    for r in range(world):
        x0, res, m, nf = out[r]
        got[:, x0:x0 + res.shape[1]] = res
        assert nf == st.n_fluid
    assert np.array_equal(got, ref)
    assert m == pytest.approx(st.mass, rel=1e-9)


def _diverge_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05295_b200 import SolverConfig
        from paper_2602_05295_b200.distributed import DistributedSolver
        from oracle.moments import neq_recompose
        torch.cuda.set_device(0)
        ds = DistributedSolver((16, 8, 8), SolverConfig(nu=0.02))
        nx = ds.plan.nx
        rho = np.ones((nx, 8, 8))
        mom = np.zeros((3, nx, 8, 8))
        if rank == 1:
            mom[0] = 0.95                   # |u| >= 0.9 on rank 1's slab only
        ds.solver.set_moments(rho, mom, neq_recompose(rho, mom, np.zeros((6, nx, 8, 8))))
        try:
            ds.step(1)
            out[rank] = "no error"
        except FloatingPointError:
            out[rank] = "FloatingPointError"
        ds.solver.close()
    finally:
        dist.destroy_process_group()


def test_divergence_raises_on_every_rank():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_diverge_worker, args=(2, port, out), nprocs=2, join=True)
    assert dict(out) == {0: "FloatingPointError", 1: "FloatingPointError"}
