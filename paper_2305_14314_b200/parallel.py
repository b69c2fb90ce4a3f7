"""Data-parallel QLoRA: only the adapter gradients cross the interconnect.

The reference has no distributed code; the north star's
DP mode replicates the frozen NF4 base on every rank, shards the batch, and
all-reduces the LoRA gradients (mean over ranks) over NCCL on NVLink /
NVSwitch.  Optimizer steps then run replicated and identically on every rank
(every rank holds the same averaged bytes, so the bit-exact Adam keeps the
replicas identical).  The same code runs on ``gloo`` for the CPU tests.

* :class:`GradBucket` -- a flat buffer holding several gradients, one
  all-reduce (the single-linear path).
* :class:`LayerReducer` -- the training path: the adapter-gradient bucket is
  cut into groups of consecutive layers; backward runs from the last layer
  to the first, and as soon as every projection of a group has written its
  gradients (the fused backward kernels write them straight into the bucket
  views) that group's all-reduce is launched asynchronously on the NCCL
  stream, so the transfer overlaps the backward of the layers below it.
  ``wire_dtype=torch.bfloat16`` halves the bytes on the wire (the sum is
  then taken in bf16 by NCCL; fp32 is the exact default).  Launches happen
  from Python during the backward, so a CUDA-graph capture of the step
  records them in place.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world_of(group=None) -> int:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


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

    def offsets(self) -> dict:
        """name -> (offset, numel) in the flat buffer."""
        out, off = {}, 0
        for name, n in zip(self.names, self.sizes):
            out[name] = (off, n)
            off += n
        return out

    def load(self, grads: dict) -> None:
        for name, v in self.views().items():
            v.copy_(grads[name].reshape(v.shape))

    def start(self, group=None) -> None:
        """Launch the (async) sum all-reduce; a no-op on a single rank."""
        if world_of(group) > 1:
            self._work = dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=True)

    def finish(self, group=None) -> dict:
        """Wait and average; returns name -> gradient view."""
        if self._work is not None:
            self._work.wait()
            self._work = None
            self.flat.div_(world_of(group))
        return self.views()


class LayerReducer:
    """Overlapped, layer-grouped mean all-reduce of a flat gradient bucket.

    ``layer_spans[i] = (offset, numel)`` of layer i's gradients in ``flat``
    (consecutive layers are contiguous); ``group_layers`` layers share one
    collective.  Call :meth:`reset` before a backward, :meth:`layer_ready`
    as each layer's gradients land (any order), :meth:`finish` after it.
    """

    def __init__(self, flat: torch.Tensor, layer_spans: list, group_layers: int = 4, group=None,
                 wire_dtype=torch.float32):
        if group_layers < 1:
            raise ValueError("group_layers must be >= 1")
        if wire_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("wire_dtype must be float32 or bfloat16")
        self.flat = flat
        self.group = group
        self.world = world_of(group)
        self.wire_dtype = wire_dtype
        n = len(layer_spans)
        self.groups = []  # (first layer, last layer + 1, offset, numel)
        for g0 in range(0, n, group_layers):
            g1 = min(n, g0 + group_layers)
            off = layer_spans[g0][0]
            end = layer_spans[g1 - 1][0] + layer_spans[g1 - 1][1]
            self.groups.append((g0, g1, off, end - off))
        self._group_of = [li // group_layers for li in range(n)]
        self.wire = None
        if self.world > 1 and wire_dtype != flat.dtype:
            self.wire = torch.empty(flat.numel(), dtype=wire_dtype, device=flat.device)
        self.reset()

    def reset(self) -> None:
        self._left = [g1 - g0 for g0, g1, _, _ in self.groups]
        self._works: list = []
        self.launched: list[int] = []  # group indices in launch order (tests / tracing)

    def layer_ready(self, layer: int) -> None:
        gi = self._group_of[layer]
        self._left[gi] -= 1
        if self._left[gi] == 0:
            self._launch(gi)

    def _launch(self, gi: int) -> None:
        self.launched.append(gi)
        if self.world == 1:
            return
        _, _, off, n = self.groups[gi]
        buf = self.flat[off: off + n]
        if self.wire is not None:
            w = self.wire[off: off + n]
            w.copy_(buf)
            buf = w
        self._works.append((gi, dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)))

    def finish(self) -> None:
        """Launch any group not yet launched, wait for all, average."""
        for gi, left in enumerate(self._left):
            if left > 0:
                self._left[gi] = 0
                self._launch(gi)
        if self.world == 1:
            return
        for gi, work in self._works:
            work.wait()
            if self.wire is not None:
                _, _, off, n = self.groups[gi]
                self.flat[off: off + n].copy_(self.wire[off: off + n])
        self._works = []
        # mean over ranks (a power-of-two world makes this an exact scaling)
        self.flat.div_(self.world)


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


__all__ = ["GradBucket", "LayerReducer", "allreduce_mean", "shard_rows", "world_of"]
