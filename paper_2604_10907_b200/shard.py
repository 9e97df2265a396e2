"""Multi-GPU sharding of the setup sweep.

Retained setups (or (setup, tau) instances) are independent (setup_search.cpp:187-211),
so rank r of W solves instances k with k % W == r on its own GPU — interleaved so the
data-dependent per-setup cost (bisection length, early exits) balances —
and the only exchange is ONE all-gather of the fixed-size per-instance records
(rw_setup_record, 336 B each), followed by the order-deterministic reduction
(setup_search.cpp:246-253).  The winner is therefore identical for any W.

torch.distributed is plumbing here: NCCL between GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

from typing import Dict, Optional, Sequence

import numpy as np

from . import _abi


def shard_of(n_items: int, rank: int, world: int) -> np.ndarray:
    """Instance indices rank `rank` solves (rw_sweep's `shard_rank/shard_count`)."""
    return np.arange(rank, n_items, world, dtype=np.int64)


def gather_records(recs: np.ndarray, group=None, device=None) -> np.ndarray:
    """All-gather every rank's record array (variable length) -> one array, rank order.

    One size exchange plus one all_gather of raw bytes; works on NCCL (device = the
    rank's cuda device) and gloo (device = cpu)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE)
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    mine = np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE).view(np.uint8)
    size = torch.tensor([mine.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, dtype=torch.uint8, device=dev)
    if mine.size:
        buf[: mine.size] = torch.from_numpy(mine.copy()).to(dev)
    outs = [torch.zeros(cap, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts = [o[:n].cpu().numpy().view(_abi.RECORD_DTYPE) for o, n in zip(outs, sizes)]
    return np.concatenate(parts) if parts else np.zeros(0, _abi.RECORD_DTYPE)


def winners_per_slo(recs: np.ndarray, taus: Optional[Sequence[float]] = None) -> Dict[float, int]:
    """Winning record index per SLO (feasible, max score, min latency, min setup id)."""
    from .routeplan import reduce_records

    recs = np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE)
    taus = sorted(set(float(t) for t in recs["tau_ms"])) if taus is None else list(taus)
    out = {}
    for t in taus:
        idx = np.nonzero(recs["tau_ms"] == t)[0]
        b = reduce_records(recs[idx]) if len(idx) else -1
        out[float(t)] = int(idx[b]) if b >= 0 else -1
    return out


def torch_gather(group=None, device=None):
    """A `gather` callable for routeplan.select_setup(..., gather=...)."""
    return lambda recs: gather_records(recs, group=group, device=device)
