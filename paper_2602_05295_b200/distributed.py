"""x-slab domain decomposition of the HOME-LBM step over one process per GPU.

The reference is single-GPU (SPEC.md:8 lists multi-GPU as out of scope); the B200 build
partitions the global grid into contiguous x-slabs, one per rank.  Every
cell update reads only its 26 neighbours, so each step needs exactly one exchange: each
rank sends its first and last interior x-planes (all components, including the y/z ghost
layers -- planes are contiguous in the state layout) into the neighbours' ghost planes.

The exchange runs over ``torch.distributed`` point-to-point (NCCL over NVLink on the GPU
box, gloo in the CPU tests).  Ranks at a non-periodic x face have no neighbour there; their
ghost plane is resolved by the BC inside the kernels (inflow constants / outflow clamp /
wall bounce-back).
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

    ``step(n)`` = n x (exchange halos; fluid_update_step).  All ranks must call it
    together.  Statistics are reduced over ranks with an all-reduce."""

    def __init__(self, global_dims: Sequence[int], config, mask: Optional[np.ndarray] = None,
                 rank: Optional[int] = None, world: Optional[int] = None, group=None):
        import torch
        import torch.distributed as dist

        from .solver import SimGrid, Slab, Solver

        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        self.group = group
        gnx, ny, nz = (int(d) for d in global_dims)
        x_periodic = tuple(config.bc.get("x", ("periodic", "periodic"))) == ("periodic", "periodic")
        self.plan = partition(gnx, self.world, x_periodic)[self.rank]
        p = self.plan
        slab = Slab(x0=p.x0, gnx=gnx, lo_remote=p.lo is not None, hi_remote=p.hi is not None)
        self.solver = Solver(SimGrid((p.nx, ny, nz)), config, slab=slab)
        if mask is not None:
            gl, gh = mask_ghost_planes(np.asarray(mask), p)
            self.solver.set_mask(np.asarray(mask)[p.x0:p.x0 + p.nx], gl, gh)
        # kernels and NCCL transfers share torch's current stream: the exchange is ordered
        # before the step without host synchronisation
        self.solver.set_stream(torch.cuda.current_stream().cuda_stream)
        self._torch = torch

    def exchange(self):
        (send_lo, send_hi, recv_lo, recv_hi), nbytes = self.solver.halo_planes()
        t = [device_view(ptr, nbytes) for ptr in (send_lo, send_hi, recv_lo, recv_hi)]
        exchange_halos(t[0], t[1], t[2], t[3], self.plan, self.group)

    def step(self, n: int = 1, stats: bool = True):
        for k in range(n):
            self.exchange()
            last = stats and k == n - 1
            self.solver.step_async(1, with_stats=last)
        if stats:
            return self.reduce_stats(self.solver.read_stats())
        return None

    def reduce_stats(self, st):
        import torch
        import torch.distributed as dist
        v = torch.tensor([st.mass, *st.momentum, st.n_fluid, *st.saturation], dtype=torch.float64,
                         device="cuda")
        dist.all_reduce(v, group=self.group)
        m = torch.tensor([st.max_u], dtype=torch.float64, device="cuda")
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        v = v.cpu().numpy()
        st.mass = float(v[0])
        st.momentum = v[1:4]
        st.n_fluid = int(v[4])
        st.saturation = v[5:15].astype(np.int64)
        st.max_u = float(m.item())
        return st
