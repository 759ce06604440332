"""Multi-GPU data parallelism over frames.

Frames are independent, so ranks decode disjoint contiguous ranges of global frame
indices and exchange nothing on the data path.  After a run: one SUM all-reduce of the int64
counters (frames, bit errors, frame errors) and one MAX all-reduce of the elapsed time.  The
frames themselves are generated per rank from (seed, global frame index), so every rank
count decodes identical data.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def frame_range(rank: int, world: int, frames_per_rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns global frames [r * B, (r + 1) * B)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * frames_per_rank, frames_per_rank


def split_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Strong scaling: `total` frames split as evenly as possible, contiguous per rank."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def allreduce_counters(counters: torch.Tensor) -> torch.Tensor:
    """In-place SUM of an int64[3] (frames, bit_errors, frame_errors) over the process group."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)
    return counters


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (elapsed time) over the process group."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
