"""How the path is spread over the GPUs of one node.

Rays are independent, so inference needs no data-path collective: each rank renders
whole frames (config 4) or interleaved image tiles (config 5 style); weights are
broadcast once.  Training is data-parallel: every rank renders its own patches and the
flat fp32 gradient is all-reduced (mean) before Adam -- the path's only exchange.
All functions work for any torch.distributed backend (NCCL on B200, gloo in CPU tests).
"""

from __future__ import annotations

from typing import List, Optional

import torch


def frame_of(rank: int, world: int, step: int, n_frames: int) -> int:
    """Frame rendered by `rank` at `step`: round-robin so a round of `world` steps covers
    consecutive frames exactly once across ranks."""
    return (rank + step * world) % n_frames


def frames_for_rank(rank: int, world: int, n_frames: int) -> List[int]:
    """Static partition of `n_frames` frames (config 4: 8 poses over 1/2/4/8 GPUs)."""
    return list(range(rank, n_frames, world))


def tiles_for_rank(rank: int, world: int, n_tiles: int) -> List[int]:
    """Interleaved image-tile assignment (uneven subject coverage balances out)."""
    return list(range(rank, n_tiles, world))


def row_bands_for_rank(rank: int, world: int, height: int, band: int = 4):
    """Image-tile sharding for config 5: interleaved bands of ``band`` rows (one 8x4 tile
    row each), rank r taking bands r, r + world, ... (subject coverage is uneven, the
    interleave balances it)."""
    return [(y, min(y + band, height)) for y in range(band * rank, height, band * world)]


def band_rows(rank: int, world: int, height: int, band: int = 4) -> List[int]:
    """Image rows of rank ``rank``'s interleaved bands (row_bands_for_rank), in order."""
    return [y for a, b in row_bands_for_rank(rank, world, height, band) for y in range(a, b)]


def gather_row_bands(image: torch.Tensor, world: int, rank: int, band: int = 4, group=None) -> torch.Tensor:
    """Assemble a frame rendered as interleaved row bands: ``image`` (H, ...) holds this rank's
    rows (others undefined); afterwards every rank holds the full frame.  One all-gather of
    the ranks' packed rows (padded to the longest share) plus an on-device row scatter."""
    import torch.distributed as dist
    if world == 1:
        return image
    h = image.shape[0]
    shares = [band_rows(r, world, h, band) for r in range(world)]
    n_max = max(len(s) for s in shares)
    idx = torch.tensor(shares[rank] + [shares[rank][-1] if shares[rank] else 0] * (n_max - len(shares[rank])),
                       device=image.device, dtype=torch.long)
    local = image.index_select(0, idx).contiguous()
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    for r in range(world):
        if r != rank and shares[r]:
            rows = torch.tensor(shares[r], device=image.device, dtype=torch.long)
            image.index_copy_(0, rows, parts[r][:len(shares[r])])
    return image


def broadcast_params(flat: torch.Tensor, src: int = 0, group=None) -> None:
    """Identical weights on every rank: one broadcast of the flat master buffer."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(flat, src=src, group=group)


def allreduce_mean(grad: torch.Tensor, group=None) -> None:
    """Data-parallel gradient exchange: sum over ranks, divide by the world size."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        n = dist.get_world_size(group)
        if n > 1:
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
            grad.mul_(1.0 / n)


class GradBuckets:
    """Data-parallel gradient exchange overlapped with the backward pass.  The flat fp32
    gradient is reduced in buckets: a bucket whose gradients are final is launched
    asynchronously (``launch``) while the backward kernels of the remaining blocks keep the
    GPU busy -- on the training path the hash table and radiance MLP (48.8 of 52.4 MB) are
    final right after the hash-grid scatter, before the residual-MLP and skinning backward --
    and ``finish`` reduces the rest, waits for every bucket and divides by the world size.
    NCCL's stream is ordered after the launching stream and ``wait`` orders the consumer
    (Adam) after NCCL, so no host synchronisation is involved.  A world of 1 is a no-op."""

    def __init__(self, grad: torch.Tensor, group=None):
        import torch.distributed as dist
        self.grad, self.group = grad, group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.pending = []
        self.done_upto = 0

    def launch(self, lo: int, hi: int) -> None:
        if self.world == 1 or hi <= lo:
            return
        import torch.distributed as dist
        self.pending.append(dist.all_reduce(self.grad[lo:hi], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        self.done_upto = max(self.done_upto, hi)

    def finish(self) -> None:
        if self.world == 1:
            return
        import torch.distributed as dist
        if self.done_upto < self.grad.numel():
            dist.all_reduce(self.grad[self.done_upto:], op=dist.ReduceOp.SUM, group=self.group)
        for w in self.pending:
            w.wait()
        self.grad.mul_(1.0 / self.world)
        self.pending, self.done_upto = [], 0


def max_over_ranks(value: float, device: Optional[torch.device] = None, group=None) -> float:
    """Job time = slowest rank (bench timing rule)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
