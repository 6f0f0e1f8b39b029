"""Host-side multi-process plumbing (torch.distributed; NCCL or gloo for the bootstrap).

Multi-GPU mode: ONE joint system whose K conditions are sharded over the
ranks in contiguous blocks; the synchronized convergence (Eq. 3.9) and the coupled alpha/beta
need one gather of the packed per-condition sums per PCG iteration, done on the device --
peer to peer over IPC-mapped memory (default, `connect_p2p`) or by NCCL.  This module holds the
partition (`shard_range`), the bench's operating-point layout (`operating_point_of`), the
max-over-ranks timing aggregation (`aggregate`) and the IPC-handle exchange (`connect_p2p`).
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_range(n_units: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n_units for this rank; the first n_units % world ranks
    get one extra unit.  Blocks tile [0, n_units) exactly, in rank order."""
    if world < 1 or not 0 <= rank < world or n_units < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def operating_point_of(rank: int, base_phi_deg: float = 90.0) -> float:
    """Shaft angle analysed by `rank` in the weak-scaling bench: rank r takes phi + r deg."""
    return base_phi_deg + float(rank)


@dataclass
class Aggregate:
    device_ms_max: float
    wall_ms_max: float
    dof_iters_total: float
    per_rank: list

    def rate(self) -> float:
        """Whole-job DOF*iter/s: all ranks' work / the slowest rank's device time."""
        return self.dof_iters_total / (self.device_ms_max * 1e-3)

    def e2e_rate(self) -> float:
        return self.dof_iters_total / (self.wall_ms_max * 1e-3)


def aggregate(device_ms: float, wall_ms: float, dof_iters: float, group=None, device=None) -> Aggregate:
    """All-gather the per-rank timings (max over ranks) and work (sum over ranks).
    Works for world = 1 without an initialised process group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([device_ms, wall_ms, dof_iters], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    if dist.is_available() and dist.is_initialized():
        parts = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, t, group=group)
        rows = [p.cpu().tolist() for p in parts]
    else:
        rows = [t.cpu().tolist()]
    return Aggregate(max(r[0] for r in rows), max(r[1] for r in rows), sum(r[2] for r in rows), rows)


def connect_p2p(solver, group=None) -> None:
    """Exchange the solvers' CUDA IPC handles over torch.distributed (any backend, e.g. gloo) and
    connect the peer-to-peer context (include/gmaf.h gmaf_p2p_handle / gmaf_p2p_connect)."""
    import torch
    import torch.distributed as dist
    # every rank's GPU must be peer-accessible from this one (the exchange kernels load and store
    # the peers' buffers over NVLink); fail loudly before connecting otherwise
    devs = [None] * solver.world
    dist.all_gather_object(devs, solver.device.index, group=group)
    mine = solver.device.index
    for r, d in enumerate(devs):
        if d is not None and d != mine and not torch.cuda.can_device_access_peer(mine, d):
            raise RuntimeError(f"rank {solver.rank}: GPU {mine} cannot access rank {r}'s GPU {d} peer to peer "
                               "(NVLink/P2P required by the peer-to-peer exchange)")
    handles = [None] * solver.world
    dist.all_gather_object(handles, solver.p2p_handle(), group=group)
    solver.p2p_connect(handles)
