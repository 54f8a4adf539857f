"""Multi-GPU plumbing: frames / volumes are
independent units, so the path shards them across ranks (weak scaling, one
process per GPU) with no data-path collective; the one exchange is the
gather of the u8 B-mode images to rank 0 (NCCL over NVLink on B200; gloo in
the CPU tests).  Each rank builds its own handle -- table construction is
deterministic, so every replica is bitwise identical.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch
import torch.distributed as dist


def shard_frames(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of frames for ``rank``: (first, count).  Blocks
    differ in size by at most one and cover [0, total) exactly once."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_bmode(img: torch.Tensor, dst: int = 0,
                 out: Optional[List[torch.Tensor]] = None) -> Optional[List[torch.Tensor]]:
    """Gather every rank's B-mode batch (same shape on all ranks) to ``dst``.
    Returns the list of per-rank tensors on ``dst``, None elsewhere."""
    world = dist.get_world_size()
    if world == 1:
        return [img]
    rank = dist.get_rank()
    if rank == dst and out is None:
        out = [torch.empty_like(img) for _ in range(world)]
    dist.gather(img, gather_list=out if rank == dst else None, dst=dst)
    return out if rank == dst else None


def frame_max_allreduce(frame_max: torch.Tensor) -> torch.Tensor:
    """All-reduce(max) of per-frame envelope maxima -- the exchange needed
    when one volume's scanline blocks are split across ranks (the frame-max
    log reference must be global).  Non-negative floats: max is exact and
    order-independent."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(frame_max, op=dist.ReduceOp.MAX)
    return frame_max
