"""Multi-rank host logic on CPU: world size 2 over gloo (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_16541_b200 import shard


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _allreduce(rank, world):
    g = torch.full((1000,), float(rank + 1))
    g[rank] = 100.0
    shard.allreduce_mean(g)
    return g.numpy()


def _broadcast(rank, world):
    flat = torch.arange(10, dtype=torch.float32) * (rank + 1)
    shard.broadcast_params(flat)
    return flat.numpy()


def _maxtime(rank, world):
    return shard.max_over_ranks(1.0 + rank)


def _trainer_allreduce(rank, world):
    # the Trainer's exchange on its flat gradient buffer (CPU tensor stands in for CUDA):
    # bucket [0, 11) launched asynchronously mid-backward, the rest at allreduce()
    from paper_2306_16541_b200.train import Trainer
    class T:  # minimal stand-in with the attributes Trainer.allreduce uses
        grad = torch.full((17,), float(rank * 2 + 1))
        grad[3] = 10.0 * rank
        buckets = shard.GradBuckets(grad)
    T.buckets.launch(0, 11)
    T.grad[11:] += 1.0                     # later backward kernels touch only later blocks
    Trainer.allreduce(T)
    return T.grad.numpy()


def test_allreduce_mean_world2():
    out = _run(_allreduce)
    want = np.full(1000, 1.5)
    want[0] = (100.0 + 2.0) / 2
    want[1] = (1.0 + 100.0) / 2
    for r in (0, 1):
        assert np.allclose(out[r], want)


def test_broadcast_world2():
    out = _run(_broadcast)
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[1], np.arange(10, dtype=np.float32))


def test_max_over_ranks_world2():
    out = _run(_maxtime)
    assert out[0] == out[1] == 2.0


def test_trainer_gradient_exchange_world2():
    out = _run(_trainer_allreduce)
    want = np.full(17, 2.0)
    want[3] = 5.0
    want[11:] = 3.0
    assert np.allclose(out[0], want) and np.allclose(out[1], want)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_frame_schedule_covers_each_frame_once_per_round(world):
    n = 8
    for step in range(4):
        frames = [shard.frame_of(r, world, step, n) for r in range(world)]
        assert len(set(frames)) == world
    seen = sorted(f for r in range(world) for f in shard.frames_for_rank(r, world, n))
    assert seen == list(range(n))
    tiles = sorted(t for r in range(world) for t in shard.tiles_for_rank(r, world, 64))
    assert tiles == list(range(64))


@pytest.mark.parametrize("world,height", [(1, 64), (2, 1024), (3, 64), (8, 1024), (8, 20)])
def test_row_bands_partition_the_image(world, height):
    from paper_2306_16541_b200.shard import row_bands_for_rank
    rows = np.zeros(height, int)
    for r in range(world):
        for a, b in row_bands_for_rank(r, world, height):
            rows[a:b] += 1
    assert np.all(rows == 1)


def _gather_bands(rank, world):
    h, w = 37, 5                            # uneven shares: 10 bands of 4 rows (+1) over 2 ranks
    img = torch.full((h, w, 4), -1.0)
    for y in shard.band_rows(rank, world, h):
        img[y] = float(y)
    return shard.gather_row_bands(img, world, rank).numpy()


def test_gather_row_bands_assembles_the_frame():
    out = _run(_gather_bands)
    want = np.broadcast_to(np.arange(37, dtype=np.float32)[:, None, None], (37, 5, 4))
    for r in (0, 1):
        assert np.array_equal(out[r], want)
    assert sorted(shard.band_rows(0, 2, 37) + shard.band_rows(1, 2, 37)) == list(range(37))
