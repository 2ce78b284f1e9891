"""x-slab domain decomposition of the HOME-LBM step over one process per GPU.

The reference is single-GPU (SPEC.md:8 lists multi-GPU as out of scope); the B200 build
partitions the global grid into contiguous x-slabs, one per rank.  Every
cell update reads only its 26 neighbours, so each step needs exactly one exchange: each
rank sends its first and last interior x-planes (all components, including the y/z ghost
layers -- planes are contiguous in the state layout) into the neighbours' ghost planes.

The exchange runs over ``torch.distributed`` point-to-point (NCCL over NVLink on the GPU
box, gloo in the CPU tests).  With a gloo group and GPU slabs (several ranks sharing one GPU in
the tests) the planes are staged through host memory: device -> host, gloo send/recv, host ->
device, in stream order on the compute stream.  Ranks at a non-periodic x face have no neighbour there; their
ghost plane is resolved by the BC inside the kernels (inflow constants / outflow clamp /
wall bounce-back).

Transports: ``transport="p2p"`` (default) posts the planes as ``torch.distributed`` send/recv
pairs; ``transport="ipc"`` is the peer-store halo of SURVEY.md §8e (K6): every rank maps its
neighbours' state buffers once through CUDA IPC (``Solver.ipc_export`` / ``ipc_open``;
NVLink peer memory when the neighbours sit on other GPUs) and copies its freshly written edge
planes straight into their ghost planes (``Solver.halo_push``, a device-to-device copy on the
comm stream).  Ordering across processes uses interprocess CUDA events, two per kind
alternating by step parity: before writing into a neighbour's ghost plane a rank's comm stream
waits for that neighbour's edge kernels of the previous step (the last readers of that plane),
and a rank's edge kernels wait for the neighbours' pushes of the previous step.  A stream can
only wait for an event record that the other process has already issued, so each step starts
with a host barrier on a gloo group (no device synchronisation; the host runs ahead of the GPU).

Overlap: a step computes its two edge destination planes
(``step_range(0, 1)``, ``step_range(nx-1, nx)``) on a side stream while the bulk
``step_range(1, nx-1)`` runs on the compute stream; the exchange of the edge planes into the
neighbours' ghost planes of the buffer being written runs on a third stream that waits only
for the edge kernels.  The next step's kernels wait for the edges and the exchange with stream
events, never on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np


@dataclass(frozen=True)
class SlabPlan:
    rank: int
    world: int
    x0: int          # first global x plane owned by this rank
    nx: int          # planes owned
    gnx: int
    lo: Optional[int]   # rank owning plane x0-1 (None: domain face, BC applies)
    hi: Optional[int]   # rank owning plane x0+nx


def partition(gnx: int, world: int, x_periodic: bool) -> list[SlabPlan]:
    """Contiguous, as-even-as-possible x-slabs (first gnx % world ranks get one more plane)."""
    if world < 1 or gnx < world:
        raise ValueError("need at least one x plane per rank")
    base, extra = divmod(gnx, world)
    plans, x0 = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        lo = r - 1 if r > 0 else (world - 1 if x_periodic else None)
        hi = r + 1 if r < world - 1 else (0 if x_periodic else None)
        if world == 1:
            lo = hi = None   # a single periodic rank wraps inside the kernel
        plans.append(SlabPlan(r, world, x0, n, gnx, lo, hi))
        x0 += n
    return plans


def exchange_halos(send_lo, send_hi, recv_lo, recv_hi, plan: SlabPlan, group=None):
    """Post the per-step halo exchange (torch tensors, any backend supporting P2P).

    send_lo (first interior plane) goes to ``plan.lo``'s recv_hi; send_hi (last interior
    plane) goes to ``plan.hi``'s recv_lo."""
    import torch.distributed as dist

    # NCCL matches point-to-point messages between a pair of ranks in issue order (tags are
    # ignored).  Every rank posts: send up, send down, recv from below, recv from above --
    # so even with two ranks on a periodic axis (lo == hi) the k-th send of one rank meets
    # the k-th receive of the other: "up" lands in recv_lo, "down" in recv_hi.
    ops = []
    if plan.hi is not None:
        ops.append(dist.P2POp(dist.isend, send_hi, plan.hi, group))
    if plan.lo is not None:
        ops.append(dist.P2POp(dist.isend, send_lo, plan.lo, group))
    if plan.lo is not None:
        ops.append(dist.P2POp(dist.irecv, recv_lo, plan.lo, group))
    if plan.hi is not None:
        ops.append(dist.P2POp(dist.irecv, recv_hi, plan.hi, group))
    if not ops:
        return
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (u8, `nbytes`)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


def device_view(ptr: int, nbytes: int):
    import torch
    return torch.as_tensor(_CudaArray(ptr, nbytes), device="cuda")


def mask_ghost_planes(global_mask: np.ndarray, plan: SlabPlan):
    """Neighbouring slabs' mask planes for the boundary-list builder of this slab."""
    gnx = global_mask.shape[0]
    lo = global_mask[(plan.x0 - 1) % gnx] if plan.lo is not None else None
    hi = global_mask[(plan.x0 + plan.nx) % gnx] if plan.hi is not None else None
    return lo, hi


class DistributedSolver:
    """One rank's slab of a global grid: a ``Solver`` plus the per-step halo exchange.

    ``step(n)`` = n x (edge planes; post the exchange of the written edge planes; bulk
    planes).  All ranks must call it together.  Statistics are reduced over ranks with an
    all-reduce.  ``solver`` may be injected (any object with the Solver stepping/halo
    interface: step_begin / step_range / step_end / halo_tensors or halo_planes, state_version);
    the CPU tests drive this schedule with an oracle-backed slab over gloo."""

    def __init__(self, global_dims: Sequence[int], config, mask: Optional[np.ndarray] = None,
                 rank: Optional[int] = None, world: Optional[int] = None, group=None, solver=None,
                 overlap: bool = True, transport: str = "p2p"):
        import torch
        import torch.distributed as dist

        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        self.group = group
        self.overlap = overlap
        gnx, ny, nz = (int(d) for d in global_dims)
        x_periodic = tuple(config.bc.get("x", ("periodic", "periodic"))) == ("periodic", "periodic")
        self.plan = partition(gnx, self.world, x_periodic)[self.rank]
        p = self.plan
        self._torch = torch
        self._cuda = solver is None and torch.cuda.is_available()
        if solver is None:
            from .solver import SimGrid, Slab, Solver

            slab = Slab(x0=p.x0, gnx=gnx, lo_remote=p.lo is not None, hi_remote=p.hi is not None)
            solver = Solver(SimGrid((p.nx, ny, nz)), config, slab=slab)
            if mask is not None:
                gl, gh = mask_ghost_planes(np.asarray(mask), p)
                solver.set_mask(np.asarray(mask)[p.x0:p.x0 + p.nx], gl, gh)
        self.solver = solver
        self._comm_stream = None
        self._edge_stream = None
        self._comm_done = None
        # gloo cannot move device tensors: stage the planes through host memory
        self._staged = self._cuda and dist.is_initialized() and dist.get_backend(group) == "gloo"
        if self._cuda:
            # kernels run on torch's current stream; the halo exchange on its own stream
            self.solver.set_stream(torch.cuda.current_stream().cuda_stream)
            self._comm_stream = torch.cuda.Stream()
            self._edge_stream = torch.cuda.Stream()   # edge planes, concurrent with the bulk
        self._synced_version = None   # solver state version whose ghost planes are exchanged
        if transport not in ("p2p", "ipc"):
            raise ValueError("transport must be 'p2p' or 'ipc'")
        self.transport = transport
        if transport == "ipc":
            self._setup_ipc()

    # ------------------------------------------------------------------ exchange
    def _halo_tensors(self, next_buffer: bool):
        if hasattr(self.solver, "halo_tensors"):
            return self.solver.halo_tensors(next_buffer)
        (send_lo, send_hi, recv_lo, recv_hi), nbytes = self.solver.halo_planes(next_buffer)
        return [device_view(ptr, nbytes) for ptr in (send_lo, send_hi, recv_lo, recv_hi)]

    def exchange(self, next_buffer: bool = False):
        """Blocking (stream-ordered on CUDA) exchange of the current -- or next -- buffer's
        edge planes into the neighbours' ghost planes."""
        t = self._halo_tensors(next_buffer)
        if self._staged:
            host = [x.cpu() for x in t[:2]] + [self._torch.empty_like(x, device="cpu") for x in t[2:]]
            exchange_halos(host[0], host[1], host[2], host[3], self.plan, self.group)
            if self.plan.lo is not None:
                t[2].copy_(host[2])
            if self.plan.hi is not None:
                t[3].copy_(host[3])
            return
        exchange_halos(t[0], t[1], t[2], t[3], self.plan, self.group)

    def _post_exchange_next(self, edges_done=None):
        """Exchange the edge planes just written to the next buffer, overlapped with the bulk
        (`edges_done`: the event after the edge kernels; default: now on the compute stream)."""
        torch = self._torch
        if not self._cuda:
            self.exchange(next_buffer=True)
            return
        if self._staged:   # host-staged planes: in order on the compute stream
            if edges_done is not None:
                torch.cuda.current_stream().wait_event(edges_done)
            self.exchange(next_buffer=True)
            return
        if edges_done is None:
            edges_done = torch.cuda.Event()
            edges_done.record(torch.cuda.current_stream())
        with torch.cuda.stream(self._comm_stream):
            self._comm_stream.wait_event(edges_done)
            self.exchange(next_buffer=True)          # NCCL work ordered on the comm stream
            self._comm_done = torch.cuda.Event()
            self._comm_done.record(self._comm_stream)

    def _wait_halos(self):
        if self._cuda and self._comm_done is not None:
            self._torch.cuda.current_stream().wait_event(self._comm_done)
            self._comm_done = None

    # ------------------------------------------------------------------ peer-store halo (ipc)
    def _neighbours(self):
        return sorted({r for r in (self.plan.lo, self.plan.hi) if r is not None})

    def _setup_ipc(self):
        import torch
        import torch.distributed as dist
        if not self._cuda or not hasattr(self.solver, "ipc_export"):
            raise ValueError("transport='ipc' needs the CUDA Solver")
        # decided from the full partition, identically on every rank, before any collective
        if not self.overlap or min(p.nx for p in partition(self.plan.gnx, self.world, False)) <= 2:
            raise ValueError("transport='ipc' needs the overlapped schedule and > 2 planes per rank")
        # host ordering of the interprocess event records (see the module docstring)
        self._hostpg = self.group if dist.get_backend(self.group) == "gloo" else dist.new_group(backend="gloo")
        self._ev_edge = [torch.cuda.Event(interprocess=True) for _ in range(2)]
        self._ev_push = [torch.cuda.Event(interprocess=True) for _ in range(2)]
        handles, cur = self.solver.ipc_export()
        info = {"nx": self.plan.nx, "handles": handles, "cur": cur,
                "edge": [e.ipc_handle() for e in self._ev_edge], "push": [e.ipc_handle() for e in self._ev_push]}
        allinfo = [None] * self.world
        dist.all_gather_object(allinfo, info, group=self._hostpg)
        dev = torch.cuda.current_device()
        self._peer_ev = {}
        for r in self._neighbours():
            self._peer_ev[r] = ([torch.cuda.Event.from_ipc_handle(dev, h) for h in allinfo[r]["edge"]],
                                [torch.cuda.Event.from_ipc_handle(dev, h) for h in allinfo[r]["push"]])
        for side, r in ((0, self.plan.lo), (1, self.plan.hi)):
            if r is not None:
                self.solver.ipc_open(side, allinfo[r]["handles"], allinfo[r]["nx"], allinfo[r]["cur"])
        self._k = 0   # steps since the last prime (event parity)

    def _prime_ipc(self):
        """Collective: re-align the neighbours' buffer indices and push the current edge planes."""
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        _, cur = self.solver.ipc_export()
        curs = [None] * self.world
        dist.all_gather_object(curs, cur, group=self._hostpg)   # also the barrier before the push
        for side, r in ((0, self.plan.lo), (1, self.plan.hi)):
            if r is not None:
                self.solver.ipc_sync(side, curs[r])
        self.solver.halo_push(False, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        dist.barrier(group=self._hostpg)
        self._k = 0
        self._synced_version = self._state_version()

    def _one_step_ipc(self, with_stats: bool):
        import torch
        import torch.distributed as dist
        s, nx = self.solver, self.plan.nx
        # the step-start barrier also decides collectively whether a prime is due
        flag = torch.tensor([1.0 if self._synced_version != self._state_version() else 0.0])
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self._hostpg)
        if flag.item() > 0:
            self._prime_ipc()
        p = self._k & 1
        compute = torch.cuda.current_stream()
        compute.wait_event(self._ev_push[p])     # our push of step k-2 read the planes step k writes
        s.step_begin(with_stats)
        start = torch.cuda.Event()
        start.record(compute)
        es, cs = self._edge_stream, self._comm_stream
        es.wait_event(start)
        if self._k > 0:
            for r in self._neighbours():        # their step k-1 planes are in our ghost planes
                es.wait_event(self._peer_ev[r][1][p ^ 1])
        s.step_range(0, 1, es.cuda_stream)
        s.step_range(nx - 1, nx, es.cuda_stream)
        self._ev_edge[p].record(es)
        cs.wait_event(self._ev_edge[p])
        if self._k > 0:
            for r in self._neighbours():        # their step k-1 edges were the last readers of the
                cs.wait_event(self._peer_ev[r][0][p ^ 1])   # ghost planes we overwrite
        s.halo_push(True, cs.cuda_stream)
        self._ev_push[p].record(cs)
        s.step_range(1, nx - 1)
        compute.wait_event(self._ev_edge[p])
        s.step_end()
        self._k += 1
        self._synced_version = self._state_version()

    def close(self):
        """Unmap the neighbours (ipc) after every rank's work is done (collective)."""
        if self.transport == "ipc" and self._cuda:
            import torch
            import torch.distributed as dist
            torch.cuda.synchronize()
            dist.barrier(group=self._hostpg)      # no rank still pushes into our buffers
            self.solver.ipc_close()
            dist.barrier(group=self._hostpg)      # every mapping closed before any buffer is freed
            self.transport = "closed"

    # ------------------------------------------------------------------ stepping
    def _state_version(self):
        return getattr(self.solver, "state_version", 0)

    def _one_step(self, with_stats: bool):
        if self.transport == "ipc":
            return self._one_step_ipc(with_stats)
        if self.transport == "closed":
            raise RuntimeError("DistributedSolver.step after close() (the neighbours are unmapped)")
        s = self.solver
        nx = self.plan.nx
        if self._synced_version != self._state_version():
            self._wait_halos()
            self.exchange()                             # the state was set on the host: prime
        else:
            self._wait_halos()                          # ghosts posted during the last step
        s.step_begin(with_stats)
        if not self.overlap or nx <= 2:
            s.step_range(0, nx)
            s.step_end()
            self._synced_version = None                 # exchange at the next step's start
            return
        if self._cuda:
            # edge planes on a side stream, concurrently with the bulk on the compute stream (the
            # bulk's launch does not queue behind the small, latency-bound edge launches); the
            # exchange waits for the edges only; the next step waits for both streams
            torch = self._torch
            compute = torch.cuda.current_stream()
            start = torch.cuda.Event()
            start.record(compute)
            self._edge_stream.wait_event(start)
            es = self._edge_stream.cuda_stream
            s.step_range(0, 1, es)
            s.step_range(nx - 1, nx, es)
            edges_done = torch.cuda.Event()
            edges_done.record(self._edge_stream)
            self._post_exchange_next(edges_done)
            s.step_range(1, nx - 1)
            compute.wait_event(edges_done)
        else:
            s.step_range(0, 1)
            s.step_range(nx - 1, nx)
            self._post_exchange_next()
            s.step_range(1, nx - 1)
        s.step_end()
        self._synced_version = self._state_version()

    def step(self, n: int = 1, stats: bool = True):
        """n steps on every rank; with ``stats`` the StepStats of the last step reduced over the
        ranks.  Divergence on any rank raises FloatingPointError on every rank, after the
        reduction (a local raise before it would leave the other ranks blocked in it)."""
        for k in range(n):
            self._one_step(stats and k == n - 1)
        if stats:
            try:
                st = self.solver.read_stats(check=False)
            except TypeError:          # injected slabs without the check flag
                st = self.solver.read_stats()
            return self.reduce_stats(st)
        return None

    def reduce_stats(self, st):
        """Sum mass / momentum / n_fluid / saturation / force / torque, max of max|u| and of a
        diverged flag (non-finite or |u| >= 0.9) over the ranks; raises
        FloatingPointError on every rank when any rank diverged."""
        import torch
        import torch.distributed as dist
        dev = "cuda" if (self._cuda and not self._staged) else "cpu"
        force = np.zeros(3) if st.force is None else np.asarray(st.force, dtype=np.float64)
        torque = np.zeros(3) if st.torque is None else np.asarray(st.torque, dtype=np.float64)
        finite = bool(getattr(st, "finite", True)) and np.isfinite(st.max_u) and np.isfinite(st.mass)
        diverged = 0.0 if (finite and st.max_u < 0.9) else 1.0
        if not dist.is_initialized():      # a single rank without a process group
            if diverged:
                raise FloatingPointError(f"solver divergence (max |u| {st.max_u:.3g} or non-finite moment)")
            return st
        v = torch.tensor([st.mass, *st.momentum, st.n_fluid, *st.saturation, *force, *torque],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(v, group=self.group)
        # NaN max|u| would poison a MAX reduction on some backends: send it as the flag + 1e300
        m = torch.tensor([st.max_u if np.isfinite(st.max_u) else 1e300, diverged], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        v = v.cpu().numpy()
        m = m.cpu().numpy()
        st.mass = float(v[0])
        st.momentum = v[1:4]
        st.n_fluid = int(v[4])
        st.saturation = v[5:15].astype(np.int64)
        st.force = v[15:18]
        st.torque = v[18:21]
        st.max_u = float(m[0])
        if m[1] > 0:
            raise FloatingPointError("solver divergence on at least one rank (non-finite moment or "
                                     f"max |u| >= 0.9; global max |u| {st.max_u:.3g})")
        return st
