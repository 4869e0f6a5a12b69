"""Data-parallel training exchange with real CUDA kernels: two ranks on one GPU over gloo
(host-mediated; the ranks' kernels never wait on each other), each rendering its own
patches.  The bucketed, backward-overlapped all-reduce (shard.GradBuckets) must give
exactly the mean of the ranks' local gradients."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from test_distributed import _run

pytestmark = pytest.mark.gpu


def _dp_grads(rank, world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    from paper_2306_16541_b200 import scene as psc
    from paper_2306_16541_b200.model import FreeviewModel
    from paper_2306_16541_b200.render import RenderSettings
    from paper_2306_16541_b200.shard import GradBuckets
    from paper_2306_16541_b200.train import Trainer
    sc = psc.make_scene(psc.config("c3", width=64, height=64, n_samples=32))
    nets = FreeviewModel(sc)
    target, mask = psc.target_image(sc)
    st = RenderSettings.from_config(sc.cfg, seed=1)
    dp = Trainer(nets, sc.camera, target, mask, st, n_patches=2, patch=16, seed=100 + rank)
    local = Trainer(nets, sc.camera, target, mask, st, n_patches=2, patch=16, seed=100 + rank)
    local.buckets = GradBuckets(local.grad)
    local.buckets.world = 1                      # no exchange: this rank's own gradient
    local.forward(step=0)
    local.backward()
    dp.forward(step=0)
    dp.backward()                                # launches the table/radiance bucket mid-backward
    dp.allreduce()
    torch.cuda.synchronize()
    mine = local.grad.clone()
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    mean = sum(gathered) / world
    return float((dp.grad - mean).abs().max()), float(mean.abs().max()), float((gathered[0] - gathered[1]).abs().max())


def test_dp_allreduce_equals_mean_of_local_gradients():
    out = _run(_dp_grads)
    for rank, (err, scale, spread) in out.items():
        print(f"rank {rank}: |dp - mean| {err:.3e}, |mean| {scale:.3e}, rank spread {spread:.3e}")
        assert spread > 0                          # the ranks really trained on different patches
        assert err <= 1e-6 * max(scale, 1e-12)
