"""x-slab decomposition + halo exchange (paper_2602_05295_b200.distributed) on CPU with gloo,
world size 2 and 3, using the oracle as each rank's slab stepper: the gathered result must
equal the single-domain oracle step."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import step as OS
from paper_2602_05295_b200.distributed import exchange_halos, partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, bc_x, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gdims = (13, 6, 8)
        bc = OS.BC(x=bc_x, u_in=(0.04, 0.0, 0.0))
        r, m, s = OS.random_state(gdims, seed=9, drho=0.05, umax=0.05, sneq=0.005)
        plan = partition(gdims[0], world, bc_x == ("periodic", "periodic"))[rank]
        sl = slice(plan.x0, plan.x0 + plan.nx)
        st = np.concatenate([r[None, sl], m[:, sl], s[:, sl]]).copy()       # (10, nx, ny, nz)
        for _ in range(steps):
            send_lo = torch.from_numpy(st[:, 0].copy())
            send_hi = torch.from_numpy(st[:, -1].copy())
            recv_lo = torch.zeros_like(send_lo)
            recv_hi = torch.zeros_like(send_hi)
            exchange_halos(send_lo, send_hi, recv_lo, recv_hi, plan)
            # x ghosts: neighbour planes, or the BC at a domain face (oracle/step.py:_pad_axis)
            full = OS.pad_state(st[0], st[1:4], st[4:10], bc)                  # BC-padded
            if plan.lo is not None:
                full[:, 0] = _pad_yz(recv_lo.numpy(), bc)
            if plan.hi is not None:
                full[:, -1] = _pad_yz(recv_hi.numpy(), bc)
            rr, mm, ss = OS.step_padded(full, 0.56)
            st = np.concatenate([rr[None], mm, ss])
        out[rank] = (plan.x0, st)
    finally:
        dist.destroy_process_group()


def _pad_yz(plane, bc):
    p = OS._pad_axis(plane, 1, bc.y)
    return OS._pad_axis(p, 2, bc.z)


def _run(world, bc_x, steps):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, bc_x, steps, out), nprocs=world, join=True)
    gdims = (13, 6, 8)
    bc = OS.BC(x=bc_x, u_in=(0.04, 0.0, 0.0))
    r, m, s = OS.random_state(gdims, seed=9, drho=0.05, umax=0.05, sneq=0.005)
    for _ in range(steps):
        r, m, s = OS.fluid_step(r, m, s, 0.56, bc)
    ref = np.concatenate([r[None], m, s])
    got = np.zeros_like(ref)
    for rank in range(world):
        x0, st = out[rank]
        got[:, x0:x0 + st.shape[1]] = st
    return got, ref


@pytest.mark.parametrize("world,bc_x", [(2, ("periodic", "periodic")), (3, ("periodic", "periodic")),
                                        (2, ("inflow", "outflow"))])
def test_slab_exchange_reproduces_single_domain(world, bc_x):
    got, ref = _run(world, bc_x, 3)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)


def test_partition_covers_domain():
    for gnx, world in ((2048, 8), (13, 3), (7, 7)):
        plans = partition(gnx, world, True)
        assert sum(p.nx for p in plans) == gnx
        assert plans[0].x0 == 0 and all(plans[i].x0 + plans[i].nx == plans[i + 1].x0 for i in range(world - 1))
        assert all(p.lo == (p.rank - 1) % world and p.hi == (p.rank + 1) % world for p in plans) or world == 1
    plans = partition(16, 4, False)
    assert plans[0].lo is None and plans[-1].hi is None


# ----------------------------------------------------------------------------- overlapped schedule
class OracleSlab:
    """CPU stand-in for one rank's Solver with the stepping/halo interface DistributedSolver
    drives (step_begin / step_range / step_end / halo_tensors / state_version).  Two buffers of
    (nx+2, 10, ny, nz) x-planes -- planes contiguous like the device layout -- each step of a
    destination range [a, b) is the oracle update of the padded source block (planes a-1 .. b)."""

    def __init__(self, st, plan, bc, tau):
        nx = st.shape[1]
        self.buf = [np.zeros((nx + 2,) + (10,) + st.shape[2:]) for _ in range(2)]
        self.buf[0][1:nx + 1] = np.moveaxis(st, 1, 0)
        self.cur, self.nx, self.plan, self.bc, self.tau = 0, nx, plan, bc, tau
        self.state_version = 1
        self.ranges = []

    def _face_ghosts(self, b):
        # ghost planes of domain faces (no neighbour): the BC, as the kernels resolve x = -1 / nx
        st = np.moveaxis(b[1:-1], 0, 1)                                   # (10, nx, ny, nz)
        pad = OS.pad_state(st[0], st[1:4], st[4:10], self.bc)[:, :, 1:-1, 1:-1]
        if self.plan.lo is None:
            b[0] = pad[:, 0]
        if self.plan.hi is None:
            b[-1] = pad[:, -1]

    def halo_tensors(self, next_buffer):
        b = self.buf[1 - self.cur if next_buffer else self.cur]
        return [torch.from_numpy(b[1]), torch.from_numpy(b[self.nx]), torch.from_numpy(b[0]),
                torch.from_numpy(b[self.nx + 1])]

    def step_begin(self, with_stats):
        self._face_ghosts(self.buf[self.cur])

    def step_range(self, a, b):
        self.ranges.append((a, b))
        src = np.moveaxis(self.buf[self.cur][a:b + 2], 0, 1)             # planes a-1 .. b
        full = OS._pad_axis(OS._pad_axis(src, 2, self.bc.y), 3, self.bc.z)
        r, m, s = OS.step_padded(full, self.tau)
        self.buf[1 - self.cur][a + 1:b + 1] = np.moveaxis(np.concatenate([r[None], m, s]), 1, 0)

    def step_end(self):
        self.cur = 1 - self.cur
        self.state_version += 1

    def state(self):
        return np.moveaxis(self.buf[self.cur][1:self.nx + 1], 0, 1)


def _overlap_worker(rank, world, port, bc_x, steps, overlap, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05295_b200 import SolverConfig
        from paper_2602_05295_b200.distributed import DistributedSolver
        gdims = (13, 6, 8)
        bc = OS.BC(x=bc_x, u_in=(0.04, 0.0, 0.0))
        r, m, s = OS.random_state(gdims, seed=9, drho=0.05, umax=0.05, sneq=0.005)
        cfg = SolverConfig(nu=(0.56 - 0.5) / 3, bc={"x": bc_x}, u_in=(0.04, 0.0, 0.0))
        plan = partition(gdims[0], world, bc_x == ("periodic", "periodic"))[rank]
        sl = slice(plan.x0, plan.x0 + plan.nx)
        slab = OracleSlab(np.concatenate([r[None, sl], m[:, sl], s[:, sl]]), plan, bc, 0.56)
        ds = DistributedSolver(gdims, cfg, solver=slab, overlap=overlap)
        assert ds.plan == plan
        ds.step(steps, stats=False)
        out[rank] = (plan.x0, slab.state(), slab.ranges[:3])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bc_x,overlap", [(2, ("periodic", "periodic"), True),
                                                (3, ("periodic", "periodic"), True),
                                                (3, ("inflow", "outflow"), True),
                                                (2, ("periodic", "periodic"), False)])
def test_overlapped_schedule_reproduces_single_domain(world, bc_x, overlap):
    """Edge planes -> exchange of the written edge planes -> bulk -> commit, driven by
    DistributedSolver over gloo, equals the single-domain oracle (3 steps)."""
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    steps = 3
    mp.spawn(_overlap_worker, args=(world, port, bc_x, steps, overlap, out), nprocs=world, join=True)
    gdims = (13, 6, 8)
    bc = OS.BC(x=bc_x, u_in=(0.04, 0.0, 0.0))
    r, m, s = OS.random_state(gdims, seed=9, drho=0.05, umax=0.05, sneq=0.005)
    for _ in range(steps):
        r, m, s = OS.fluid_step(r, m, s, 0.56, bc)
    ref = np.concatenate([r[None], m, s])
    got = np.zeros_like(ref)
    for rank in range(world):
        x0, st, ranges = out[rank]
        got[:, x0:x0 + st.shape[1]] = st
        nx = st.shape[1]
        assert ranges == ([(0, 1), (nx - 1, nx), (1, nx - 1)] if overlap else [(0, nx)] * 3)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)


def test_transport_validation():
    """transport="ipc" needs the CUDA Solver (it maps the neighbours' device buffers); unknown
    transports are rejected."""
    from paper_2602_05295_b200 import SolverConfig
    from paper_2602_05295_b200.distributed import DistributedSolver
    cfg = SolverConfig(nu=0.02)
    with pytest.raises(ValueError, match="ipc"):
        DistributedSolver((8, 4, 4), cfg, rank=0, world=1, solver=object(), transport="ipc")
    with pytest.raises(ValueError, match="transport"):
        DistributedSolver((8, 4, 4), cfg, rank=0, world=1, solver=object(), transport="tcp")


def test_ipc_slab_size_check_is_the_same_on_every_rank():
    """The > 2 planes rule is decided from the whole partition (before any collective), so a rank
    with enough planes refuses exactly when another rank would (no rank left waiting in a
    collective).  gnx = 7 over 3 ranks: slabs 3, 2, 2 -> every rank refuses, rank 0 included."""
    from paper_2602_05295_b200.distributed import partition
    assert [p.nx for p in partition(7, 3, True)] == [3, 2, 2]
    assert min(p.nx for p in partition(7, 3, False)) <= 2
