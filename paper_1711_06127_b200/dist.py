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


class OverlappedGather:
    """Double-buffered asynchronous gather of B-mode batches to ``dst`` so the
    transfer of step i overlaps the beamforming of step i + 1 (SURVEY 8(e):
    rank-0 ingress, not compute, bounds the frame-sharded stream beyond a few
    GPUs).  ``buffer(i)`` is the image batch step i must write; before it is
    handed out again (step i + 2) the stream waits for its previous gather.
    ``received(i)`` on ``dst`` is the list of every rank's batch of step i
    once ``drain()`` (or the wait inside ``buffer(i + 2)``) has run."""

    def __init__(self, like: torch.Tensor, dst: int = 0, nbuf: int = 2):
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.dst = dst
        self.bufs = [like if i == 0 else torch.empty_like(like) for i in range(nbuf)]
        self.recv = [[torch.empty_like(like) for _ in range(self.world)] if self.rank == dst else None
                     for _ in range(nbuf)]
        self.work = [None] * nbuf

    def buffer(self, i: int) -> torch.Tensor:
        b = i % len(self.bufs)
        if self.work[b] is not None:
            self.work[b].wait()        # stream-ordered: the current stream waits, the host does not
            self.work[b] = None
        return self.bufs[b]

    def submit(self, i: int):
        if self.world == 1:
            return
        b = i % len(self.bufs)
        self.work[b] = dist.gather(self.bufs[b], gather_list=self.recv[b], dst=self.dst, async_op=True)

    def drain(self):
        for b, w in enumerate(self.work):
            if w is not None:
                w.wait()
                self.work[b] = None

    def received(self, i: int):
        return self.recv[i % len(self.bufs)] if self.world > 1 else [self.bufs[i % len(self.bufs)]]


def frame_max_allreduce(frame_max: torch.Tensor) -> torch.Tensor:
    """All-reduce(max) of per-frame envelope maxima -- the exchange needed
    when one volume's scanline blocks are split across ranks (the frame-max
    log reference must be global).  Non-negative floats: max is exact and
    order-independent."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(frame_max, op=dist.ReduceOp.MAX)
    return frame_max


def shard_lines(L: int, world: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous block of scanlines for ``rank``: (first, count), block
    boundaries on multiples of ``align`` lines (align = lines per event block,
    so each transmit event's data is read by exactly one rank).
    Covers [0, L) exactly once; requires L % align == 0."""
    if L % align:
        raise ValueError(f"L={L} is not a multiple of align={align}")
    first, n = shard_frames(L // align, world, rank)
    return first * align, n * align


class ShardedVolume:
    """Latency mode: ONE volume beamformed by all ranks, each
    on a contiguous scanline block.  Per call:
      1. DAS + envelope of the rank's lines (supra_bf_beamform_lines),
      2. all-reduce(max) of the frame maximum (the log reference of S:267;
         skipped for a fixed reference),
      3. log compression of the rank's lines against the global maximum,
      4. all-gather of the line-domain slabs so every rank holds the volume
         (u8 for C4: 8 MiB in total) -- the scan conversion then runs on
         rank 0 (or on any rank) from the full line image.
    No input exchange: the blocks read disjoint events.  ``bf`` is a SupraBF
    handle (or any object with beamform_lines / log_compress of the same
    signature); ``y_dtype`` is the line-image dtype of its config and ``S``
    its line-image samples per line (samples_per_channel / decimation)."""

    def __init__(self, bf, L: int, S: int, y_dtype: torch.dtype, device, align: int = 1,
                 fixed_reference: bool = False):
        self.bf = bf
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.L, self.S = L, S
        self.first, self.count = shard_lines(L, self.world, self.rank, align)
        self.ranges = [shard_lines(L, self.world, r, align) for r in range(self.world)]
        counts = [c for _, c in self.ranges]
        self.chunk = max(counts)
        self.equal = all(c == self.chunk for c in counts)
        self.fixed = fixed_reference
        self.env = torch.empty((1, L, S), dtype=torch.float32, device=device)
        self.fmax = torch.zeros((1,), dtype=torch.float32, device=device)
        self.y = torch.zeros((1, L, S), dtype=y_dtype, device=device)
        self.send = torch.zeros((self.chunk, S), dtype=y_dtype, device=device)
        if not self.equal:
            self.recv = torch.zeros((self.world, self.chunk, S), dtype=y_dtype, device=device)

    def run(self, raw, stream=None) -> torch.Tensor:
        """Beamform one volume (raw [1][E][C][S] on this rank's device; only
        this rank's events are read) -> full line image [1][L][S] on every rank."""
        a, n = self.first, self.count
        self.bf.beamform_lines(raw, 1, a, n, self.env, self.fmax, stream)
        if not self.fixed:
            frame_max_allreduce(self.fmax)
        self.bf.log_compress(self.env, 1, a, n, self.fmax, self.y, stream)
        if self.world == 1:
            return self.y
        flat = self.y.view(self.L, self.S)
        self.send[:n].copy_(flat[a:a + n])
        if self.equal:       # rank r's block is rows [r*chunk, (r+1)*chunk): gather straight into y
            dist.all_gather_into_tensor(flat, self.send)
        else:
            dist.all_gather_into_tensor(self.recv.view(self.world * self.chunk, self.S), self.send)
            for r, (f, c) in enumerate(self.ranges):
                flat[f:f + c].copy_(self.recv[r, :c])
        return self.y
