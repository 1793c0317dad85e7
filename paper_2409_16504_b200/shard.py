"""Sharding independent frames / views over ranks.

Frames of a dynamic sequence and views of one scene are independent units:
each rank (one process per GPU) renders its own units end to end — it runs
P2ENet itself (≪ 1 ms) rather than receiving splats — so the data path has
no collective. The only cross-rank traffic is control: a barrier, the
max-over-ranks of the device time (bench.py), and an optional gather of
per-unit results (host objects) to rank 0 at the end.

Policies: ``"round_robin"`` (unit u -> rank u % world; bench.py's ring views
of config 2) and ``"block"`` (contiguous blocks of ceil(U/world); config 4's
frame sequence, so each rank walks consecutive frames).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(n_units: int, rank: int, world: int, policy: str = "round_robin") -> list:
    """Unit indices owned by ``rank``; the shards of all ranks partition range(n_units)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    if n_units < 0:
        raise ValueError("unit count must be non-negative")
    if policy == "round_robin":
        return list(range(rank, n_units, world))
    if policy == "block":
        per = -(-n_units // world)
        return list(range(min(n_units, rank * per), min(n_units, (rank + 1) * per)))
    raise ValueError(f"unknown sharding policy {policy!r}")


def unit_of(step: int, rank: int, world: int, n_units: int) -> int:
    """Round-robin unit of a rank's ``step``-th frame in an open-ended stream
    (global frame rank + step*world, wrapped over the units)."""
    return (rank + step * world) % n_units


def _ready() -> bool:
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(x: float) -> float:
    """Max of a per-rank scalar (device time), the only timing reduction."""
    if not _ready() or dist.get_world_size() == 1:
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(results: dict):
    """Per-unit host results of every rank -> one dict on rank 0 (None elsewhere).
    Raises if two ranks produced the same unit (a sharding bug)."""
    if not _ready() or dist.get_world_size() == 1:
        return dict(results)
    world = dist.get_world_size()
    rank = dist.get_rank()
    got = [None] * world if rank == 0 else None
    dist.gather_object(dict(results), got, dst=0)
    if rank != 0:
        return None
    merged = {}
    for part in got:
        for k, v in part.items():
            if k in merged:
                raise RuntimeError(f"unit {k} rendered by two ranks")
            merged[k] = v
    return merged


def _dtype(name: str):
    return getattr(torch, name.split(".")[-1])


def _to_host(t: torch.Tensor) -> torch.Tensor:
    if not t.is_cuda:
        return t
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def gather_planes(frames: dict, dst: int = 0, host: bool = True, out: dict = None):
    """The final gather of a sharded job: ``frames`` maps each unit this rank
    rendered to a tuple of plane tensors; rank ``dst`` receives every rank's
    planes point to point over the default process group (NCCL: device
    tensors over NVLink; gloo: host tensors) and returns {unit: planes} for
    the whole job, as pinned host tensors when ``host`` (one device->host copy
    per plane); other ranks return None. Raises if two ranks rendered the
    same unit. ``out`` (rank dst): preallocated pinned host tensors per unit
    to copy into instead of fresh allocations."""
    def to_host(u, ts):
        if out is not None and u in out:
            for h, t in zip(out[u], ts):
                h.copy_(t, non_blocking=True)
            return out[u]
        return tuple(_to_host(t) for t in ts)

    if not _ready() or dist.get_world_size() == 1:
        res = {u: (to_host(u, ts) if host else ts) for u, ts in frames.items()}
        if host and torch.cuda.is_available():
            torch.cuda.synchronize()
        return res
    world, rank = dist.get_world_size(), dist.get_rank()
    meta = {u: [(tuple(t.shape), str(t.dtype)) for t in ts] for u, ts in frames.items()}
    metas = [None] * world if rank == dst else None
    dist.gather_object(meta, metas, dst=dst)
    if rank != dst:
        reqs = [dist.isend(t.contiguous(), dst) for u in sorted(frames) for t in frames[u]]
        for r in reqs:
            r.wait()
        return None
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    got = dict(frames)
    reqs = []
    for src in range(world):
        if src == dst:
            continue
        for u in sorted(metas[src]):
            if u in got:
                raise RuntimeError(f"unit {u} rendered by two ranks")
            bufs = tuple(torch.empty(s, dtype=_dtype(d), device=dev) for s, d in metas[src][u])
            reqs += [dist.irecv(b, src) for b in bufs]
            got[u] = bufs
    for r in reqs:
        r.wait()
    if host:
        got = {u: to_host(u, ts) for u, ts in got.items()}
        if dev == "cuda":
            torch.cuda.synchronize()
    return got
