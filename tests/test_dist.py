"""Multi-process plumbing on CPU (gloo, world_size 2): frame sharding covers
every frame once, the B-mode gather delivers every rank's batch to rank 0
in rank order, and the frame-max all-reduce is exact (T9)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1711_06127_b200.dist import frame_max_allreduce, gather_bmode, shard_frames


@pytest.mark.parametrize("total,world", [(100, 1), (100, 2), (100, 8), (7, 4), (3, 8)])
def test_shard_frames_partition(total, world):
    seen = []
    for r in range(world):
        first, n = shard_frames(total, world, r)
        seen.extend(range(first, first + n))
    assert seen == list(range(total))
    sizes = [shard_frames(total, world, r)[1] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, n = shard_frames(10, world, rank)
        # stand-in B-mode batch: frame f filled with f (u8)
        img = torch.stack([torch.full((3, 1, 5), first + i, dtype=torch.uint8) for i in range(n)])
        got = gather_bmode(img)
        fm = torch.tensor([float(rank + 1), 0.5 * rank], dtype=torch.float32)
        frame_max_allreduce(fm)
        q.put((rank, None if got is None else [g.tolist() for g in got], fm.tolist()))
    finally:
        dist.destroy_process_group()


def test_gather_and_allreduce_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, got, fm = q.get(timeout=120)
        res[rank] = (got, fm)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got0 = res[0][0]
    assert res[1][0] is None
    frames = [torch.tensor(b) for b in got0]
    allf = torch.cat(frames)
    assert allf.shape[0] == 10
    for f in range(10):
        assert torch.all(allf[f] == f)
    for r in range(world):
        assert res[r][1] == [2.0, 0.5]
