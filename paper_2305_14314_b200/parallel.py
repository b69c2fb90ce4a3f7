"""Data-parallel QLoRA: only the adapter gradients cross the interconnect.

The reference has no distributed code; the north star's DP
mode replicates the frozen NF4 base on every rank, shards the batch, and
all-reduces the LoRA gradients (mean over ranks) over NCCL on NVLink /
NVSwitch, bucketed and launched asynchronously so the transfer overlaps the
remaining backward work.  Optimizer steps then run replicated and
identically on every rank.  The same code runs on ``gloo`` for CPU tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


class GradBucket:
    """A flat buffer holding several gradients contiguously; one all-reduce."""

    def __init__(self, shapes: dict, device, dtype=torch.float32):
        self.names = list(shapes)
        self.sizes = [int(torch.Size(s).numel()) for s in shapes.values()]
        self.shapes = dict(shapes)
        self.flat = torch.zeros(sum(self.sizes), dtype=dtype, device=device)
        self._work = None

    def views(self) -> dict:
        out, off = {}, 0
        for name, n in zip(self.names, self.sizes):
            out[name] = self.flat[off: off + n].view(self.shapes[name])
            off += n
        return out

    def load(self, grads: dict) -> None:
        for name, v in self.views().items():
            v.copy_(grads[name].reshape(v.shape))

    def start(self, group=None) -> None:
        """Launch the (async) sum all-reduce; a no-op on a single rank."""
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            self._work = dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=True)

    def finish(self, group=None) -> dict:
        """Wait and average; returns name -> gradient view."""
        if self._work is not None:
            self._work.wait()
            self._work = None
            self.flat.div_(dist.get_world_size(group))
        return self.views()


def allreduce_mean(grads: dict, group=None) -> dict:
    """Average a dict of gradients across ranks with one bucketed all-reduce."""
    if not grads:
        return grads
    any_t = next(iter(grads.values()))
    b = GradBucket({k: tuple(v.shape) for k, v in grads.items()}, any_t.device, any_t.dtype)
    b.load(grads)
    b.start(group)
    return b.finish(group)


def shard_rows(n: int, rank: int, world: int) -> slice:
    """Contiguous batch shard of rank ``rank`` (weak scaling uses a fixed per-rank size)."""
    per = (n + world - 1) // world
    return slice(min(n, rank * per), min(n, (rank + 1) * per))


__all__ = ["GradBucket", "allreduce_mean", "shard_rows"]
