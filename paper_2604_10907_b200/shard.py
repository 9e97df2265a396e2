"""Multi-GPU sharding of the setup sweep.

Retained setups (or (setup, tau) instances) are independent (setup_search.cpp:187-211),
so rank r of W solves instances k with k % W == r on its own GPU — interleaved so the
data-dependent per-setup cost (bisection length, early exits) balances —
and the only exchange is ONE all-gather of the fixed-size per-instance records
(rw_setup_record, 344 B each), followed by the order-deterministic reduction
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


def shard_capacity(n_items: int, world: int) -> int:
    """Records of the largest shard: every rank's buffer is padded to this many."""
    return max(1, (n_items + world - 1) // world)


def pad_records(recs: np.ndarray, cap: int) -> np.ndarray:
    """recs padded to cap records; padding slots carry setup_id = -1."""
    out = np.zeros(cap, _abi.RECORD_DTYPE)
    out["setup_id"] = -1
    r = np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE)
    out[: len(r)] = r
    return out


def _unpad(flat: np.ndarray) -> np.ndarray:
    return flat[flat["setup_id"] >= 0]


def gather_records(recs: np.ndarray, n_items: int, group=None, device=None) -> np.ndarray:
    """ONE all-gather of every rank's records (host array, padded to the largest shard's
    size, known from n_items) -> one array in rank order, padding dropped.  Works on NCCL
    (device = the rank's cuda device) and gloo (device = cpu)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE)
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    cap = shard_capacity(n_items, world)
    mine = torch.from_numpy(pad_records(recs, cap).view(np.uint8)).to(dev)
    out = torch.empty(world * mine.numel(), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, mine, group=group)
    return _unpad(out.cpu().numpy().view(_abi.RECORD_DTYPE))


def device_record_buffer(n_items: int, world: int, device):
    """A padded device buffer for rw_set_records_device: the sweep kernel writes this rank's
    records into it, and gather_device_records exchanges it without a host round trip."""
    import torch

    cap = shard_capacity(n_items, world)
    buf = torch.empty(cap * _abi.RECORD_DTYPE.itemsize, dtype=torch.uint8, device=device)
    return buf, cap


def reset_device_records(buf) -> None:
    buf.fill_(0xFF)  # setup_id = -1 in every slot the sweep does not write


def gather_device_records(buf, group=None) -> np.ndarray:
    """ONE all_gather_into_tensor of every rank's device record buffer (NCCL over NVLink)
    -> one host array in rank order, padding dropped."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return _unpad(buf.cpu().numpy().view(_abi.RECORD_DTYPE))
    world = dist.get_world_size(group)
    out = torch.empty(world * buf.numel(), dtype=torch.uint8, device=buf.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return _unpad(out.cpu().numpy().view(_abi.RECORD_DTYPE))


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


def torch_gather(n_items: int, group=None, device=None):
    """A `gather` callable for routeplan.select_setup(..., gather=...)."""
    return lambda recs: gather_records(recs, n_items, group=group, device=device)
