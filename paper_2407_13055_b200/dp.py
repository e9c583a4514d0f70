"""Data-parallel execution over independent ciphertexts (mode 1).

One process per GPU (torchrun), keys replicated, each rank evaluates its own
contiguous shard of the batch; there is no collective in the data path —
only the timing reduction (max over ranks) and an optional gather of results
at the end.  The helpers are backend-agnostic so the N>1 logic is exercised
with `gloo` on CPU in the test suite and with `nccl` over NVLink in bench.py.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist


def shard_bounds(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced partition of `n_items` over `world` ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def max_over_ranks(values: Sequence[float], device: Optional[torch.device] = None) -> List[float]:
    """Element-wise max over ranks (device-timed numbers are reported as the max)."""
    w, _ = world()
    if w == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def run_sharded(fn: Callable[[torch.Tensor], torch.Tensor], batch: torch.Tensor, gather: bool = True):
    """Evaluate fn on this rank's shard of `batch` (leading dimension) and
    optionally all-gather the per-rank outputs in rank order.  Shards may have
    unequal sizes; they are padded for the collective and trimmed after."""
    w, r = world()
    lo, hi = shard_bounds(batch.shape[0], w, r)
    out = fn(batch[lo:hi])
    if not gather or w == 1:
        return out
    sizes = [shard_bounds(batch.shape[0], w, k) for k in range(w)]
    cap = max(h - l for l, h in sizes)
    pad = torch.zeros((cap,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pad[: out.shape[0]] = out
    parts = [torch.empty_like(pad) for _ in range(w)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: h - l] for p, (l, h) in zip(parts, sizes)], dim=0)
