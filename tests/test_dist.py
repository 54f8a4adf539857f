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


@pytest.mark.parametrize("L,world,align", [(4096, 8, 256), (4096, 2, 256), (192, 4, 1), (10, 3, 2), (8, 1, 4)])
def test_shard_lines_partition(L, world, align):
    from paper_1711_06127_b200.dist import shard_lines
    seen = []
    for r in range(world):
        first, n = shard_lines(L, world, r, align)
        assert first % align == 0 and n % align == 0
        seen.extend(range(first, first + n))
    assert seen == list(range(L))


def test_c4b_line_blocks_read_disjoint_events():
    """With 4-row alignment (256 lines) every transmit event of C4b is read
    by exactly one rank: the latency-mode input needs no exchange."""
    from synth import configs
    from paper_1711_06127_b200.dist import shard_lines
    w = configs.c4("b")
    for world in (2, 4, 8):
        owners = {}
        for r in range(world):
            a, n = shard_lines(w.L, world, r, 4 * w.num_lines_x)
            for e in set(w.line_event[a:a + n].tolist()):
                assert owners.setdefault(e, r) == r
        assert len(owners) == w.num_events


class _StubBF:
    """CPU stand-in with the SupraBF line-range signatures: env[l][k] =
    (l + 1) * (k + 1) (max over a range is at its last line, last sample);
    log_compress writes env / frame_max."""

    def beamform_lines(self, raw, frames, first, count, env, fmax, stream=None):
        S = env.shape[-1]
        l = torch.arange(first, first + count, dtype=torch.float32)[:, None]
        k = torch.arange(S, dtype=torch.float32)[None]
        env[0, first:first + count] = (l + 1) * (k + 1)
        fmax[0] = env[0, first:first + count].max() if count else 0.0

    def log_compress(self, env, frames, first, count, fmax, y, stream=None):
        y[0, first:first + count] = env[0, first:first + count] / fmax[0]


def _vol_worker(rank, world, port, L, align, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_06127_b200.dist import ShardedVolume
        sv = ShardedVolume(_StubBF(), L, 8, torch.float32, "cpu", align=align)
        y = sv.run(None)
        q.put((rank, y.clone().numpy(), float(sv.fmax[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,align", [(16, 4), (12, 1)])   # equal blocks / unequal blocks (5, 4, ... )
def test_sharded_volume_gloo_world2(L, align):
    world = 2 if L == 16 else 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vol_worker, args=(r, world, port, L, align, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (y, m)) for r, y, m in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S = 8
    full = (torch.arange(L, dtype=torch.float64)[:, None] + 1) * (torch.arange(S, dtype=torch.float64)[None] + 1)
    expect = (full / full.max()).numpy()
    for r in range(world):
        y, m = res[r]
        assert m == float(L * S)                       # the global frame max on every rank
        assert abs(y[0] - expect).max() < 1e-6         # every rank holds the whole line image


def _overlap_worker(rank, world, port, q):
    from paper_1711_06127_b200.dist import OverlappedGather
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        like = torch.zeros((2, 1, 4), dtype=torch.uint8)
        g = OverlappedGather(like, dst=0)
        seen = []
        for i in range(5):
            buf = g.buffer(i)
            if i >= 2 and rank == 0:      # the gather of step i - 2 has completed
                seen.append((i - 2, [t.tolist() for t in g.received(i - 2)]))
            buf.fill_(10 * i + rank)       # "beamform" step i into the handed-out buffer
            g.submit(i)
        g.drain()
        if rank == 0:
            for i in (3, 4):
                seen.append((i, [t.tolist() for t in g.received(i)]))
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_overlapped_gather_double_buffer_gloo_world2():
    """The double-buffered asynchronous B-mode gather of bench.py: every step's
    batches arrive at rank 0 in rank order, and a buffer is not handed out
    again before its previous gather completed."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    steps = dict(res[0])
    assert sorted(steps) == [0, 1, 2, 3, 4]
    for i, got in steps.items():
        assert got == [torch.full((2, 1, 4), 10 * i + r, dtype=torch.uint8).tolist() for r in range(world)]
