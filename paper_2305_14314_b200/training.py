"""Optimizer step of the QLoRA finetune on the GPU -- mirror of the reference's
``TrainConfig`` / ``clip_global_norm`` / ``AdamOptimizer`` / moment stores
(pkg/src/qlrt/training.py:62-90, 354-442).

* ``AdamOptimizer.step`` launches one bit-exact fp32 Adam kernel per
  parameter (the reference's op order with the float32-rounded constants
  numpy 2 uses under NEP 50), which also refreshes the bf16 operand copies.
* ``PlainMomentStore`` keeps moments as device tensors; ``PagedMomentStore``
  keeps them in unified-memory slabs under a :class:`Pager` budget.  Both run
  the same kernel on the same bytes, so paged == plain bit for bit.
* ``clip_global_norm`` sums squares in fp64 on the device in numpy's
  pairwise order and scales in place with the float32-rounded factor
  (training.py:398-413).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ._native import SUMSQ_SCRATCH, check, lib, ptr, stream_ptr
from .errors import TrainingDivergedError
from .paging import Pager

OPTIMIZERS = ("plain", "paged")


@dataclass(frozen=True)
class TrainConfig:
    """training.py:62-90 (the optimizer-relevant fields and defaults)."""

    learning_rate: float = 0.01
    batch_size: int = 64
    steps: int = 500
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    max_grad_norm: float = 0.3
    lr_schedule: str = "constant"
    seed: int = 0

    def validate(self) -> None:
        if not (self.learning_rate > 0 and math.isfinite(self.learning_rate)):
            raise ValueError("learning_rate must be positive and finite")
        if self.batch_size < 1:
            raise ValueError("batch_size must be at least 1")
        if self.steps < 1:
            raise ValueError("steps must be at least 1")
        for name in ("adam_beta1", "adam_beta2"):
            if not 0.0 <= getattr(self, name) < 1.0:
                raise ValueError(f"{name} must lie in [0, 1)")
        if self.adam_eps <= 0:
            raise ValueError("adam_eps must be positive")
        if self.max_grad_norm <= 0:
            raise ValueError("max_grad_norm must be positive")
        if self.lr_schedule != "constant":
            raise ValueError("only the constant lr schedule is supported")


class PlainMomentStore:
    """Adam moments as resident device tensors (training.py:354-368)."""

    def __init__(self):
        self._state: dict[str, tuple[torch.Tensor, torch.Tensor]] = {}

    def update(self, name: str, param: torch.Tensor, fn) -> None:
        st = self._state.get(name)
        if st is None:
            st = (torch.zeros_like(param), torch.zeros_like(param))
            self._state[name] = st
        fn(*st)

    def close(self) -> None:
        pass


class PagedMomentStore:
    """Moments in pager slabs: first moment then second, one slab per
    parameter (training.py:371-395), resident on demand."""

    def __init__(self, pager: Pager):
        self.pager = pager
        self._slabs = {}

    def update(self, name: str, param: torch.Tensor, fn) -> None:
        slab = self._slabs.get(name)
        if slab is None:
            slab = self.pager.alloc(2 * param.numel() * param.element_size())
            self._slabs[name] = slab

        def run(view: torch.Tensor) -> None:
            flat = view.view(param.dtype)
            fn(flat[: param.numel()].view(param.shape), flat[param.numel():].view(param.shape))

        self.pager.with_slab(slab, run)

    def prefetch(self, name: str) -> None:
        """Start migrating ``name``'s moments to the device (look-ahead)."""
        slab = self._slabs.get(name)
        if slab is not None:
            self.pager.prefetch(slab)

    def close(self) -> None:
        self.pager.flush()


def _pairwise_tree(n: int):
    """numpy's pairwise-sum tree over n values (loops_utils.h.src): leaves of
    <= 128 values in order, internal nodes (dst, left, right) grouped by
    height.  Returns (leaves [L][2], ops [I][3], level_starts, root)."""
    leaves: list = []
    ops: list = []

    def rec(off: int, length: int):
        if length <= 128:
            leaves.append((off, length))
            return ("L", len(leaves) - 1), 0
        n2 = length // 2
        n2 -= n2 % 8
        a, ha = rec(off, n2)
        b, hb = rec(off + n2, length - n2)
        ops.append((a, b, max(ha, hb) + 1))
        return ("I", len(ops) - 1), max(ha, hb) + 1

    root, _ = rec(0, n)
    n_l = len(leaves)
    order = sorted(range(len(ops)), key=lambda j: ops[j][2])
    pos = {j: n_l + k for k, j in enumerate(order)}
    idx = lambda node: node[1] if node[0] == "L" else pos[node[1]]  # noqa: E731
    flat_ops, starts, h_prev = [], [0], None
    for k, j in enumerate(order):
        a, b, h = ops[j]
        if h_prev is not None and h != h_prev:
            starts.append(k)
        h_prev = h
        flat_ops += [n_l + k, idx(a), idx(b)]
    starts.append(len(order))
    if not order:
        starts = [0]
    return (np.asarray(leaves, dtype=np.int32).reshape(-1), np.asarray(flat_ops, dtype=np.int32),
            np.asarray(starts, dtype=np.int32), idx(root), n_l + len(order))


_TREES: dict = {}


def _tree_dev(n: int, device):
    key = (n, str(device))
    t = _TREES.get(key)
    if t is None:
        leaves, ops, starts, root, n_vals = _pairwise_tree(n)
        to = lambda a: torch.from_numpy(a).to(device) if a.size else torch.zeros(1, dtype=torch.int32, device=device)  # noqa: E731
        t = (to(leaves), to(ops), to(starts), len(leaves) // 2, len(starts) - 1, root,
             torch.empty(n_vals, dtype=torch.float64, device=device))
        _TREES[key] = t
    return t


def pairwise_sumsq(grads: dict, order: list) -> torch.Tensor:
    """Device fp64 sum over ``order`` of np.sum(np.square(g, dtype=float64))
    in numpy's own pairwise order per tensor, the tensors added in order from
    0.0 -- clip_global_norm's total, bit for bit (training.py:398-407)."""
    dev = grads[order[0]].device
    acc = torch.zeros(1, dtype=torch.float64, device=dev)
    for name in order:
        g = grads[name]
        if not g.is_contiguous():
            g = g.contiguous()
        if g.dtype != torch.float32:
            raise ValueError("clip_global_norm expects float32 gradients")
        if g.numel() == 0:
            continue
        leaves, ops, starts, n_leaves, n_levels, root, vals = _tree_dev(g.numel(), dev)
        check(lib().qlrt_sumsq_f64_pairwise(ptr(g), ptr(leaves), n_leaves, ptr(ops), ptr(starts), n_levels, root,
                                            ptr(vals), ptr(acc), stream_ptr()), "clip_global_norm")
    return acc


def _sumsq_scratch(device) -> torch.Tensor:
    return torch.zeros(SUMSQ_SCRATCH // 8, dtype=torch.float64, device=device)


def global_sumsq(grads: dict, order: list) -> torch.Tensor:
    """Device fp64 sum of squares over ``order`` (no host sync)."""
    dev = grads[order[0]].device
    acc = _sumsq_scratch(dev)
    for name in order:
        g = grads[name]
        if not g.is_contiguous():
            g = g.contiguous()
        if g.numel():
            check(lib().qlrt_sumsq_f64(ptr(g), g.numel(), ptr(acc), stream_ptr()), "clip_global_norm")
    return acc[:1]


def clip_global_norm(grads: dict, order: list, max_norm: float) -> float:
    """Scale every gradient in place when the joint 2-norm exceeds ``max_norm``;
    returns the pre-clip norm (training.py:398-413).  The sum of squares runs
    in numpy's pairwise order (``pairwise_sumsq``): the norm, hence the f32
    scale, is bit-identical to the reference's."""
    norm = math.sqrt(float(pairwise_sumsq(grads, order).item()))
    if norm > max_norm and norm > 0.0:
        scale = float(np.float32(max_norm / norm))
        for name in order:
            g = grads[name]
            if g.is_contiguous():
                check(lib().qlrt_scale_f32(ptr(g), g.numel(), scale, stream_ptr()), "clip_global_norm")
            else:
                g.mul_(scale)
    return norm


class AdamOptimizer:
    """Adam with bias correction; moments live wherever ``store`` puts them
    (training.py:416-442).  ``params`` maps names to float32 device tensors;
    ``shadows`` optionally maps names to bf16 copies refreshed by the kernel."""

    def __init__(self, params: dict, cfg: TrainConfig, store, shadows: dict | None = None):
        self.params = params
        self.cfg = cfg
        self.store = store
        self.shadows = shadows or {}
        self.t = 0

    def constants(self):
        """The float32 values numpy 2 (NEP 50) uses in the reference's update."""
        c = self.cfg
        f = np.float32
        bc1 = 1.0 - c.adam_beta1 ** self.t
        bc2 = 1.0 - c.adam_beta2 ** self.t
        return tuple(float(f(v)) for v in (c.adam_beta1, 1.0 - c.adam_beta1, c.adam_beta2, 1.0 - c.adam_beta2,
                                           bc1, bc2, c.adam_eps, c.learning_rate))

    def step(self, grads: dict) -> None:
        self.t += 1
        consts = self.constants()
        names = list(self.params)
        for i, name in enumerate(names):
            p = self.params[name]
            g = grads[name]
            if not g.is_contiguous():
                g = g.contiguous()
            if p.dtype != torch.float32 or g.dtype != torch.float32:
                raise ValueError("AdamOptimizer expects float32 parameters and gradients")
            shadow = self.shadows.get(name)

            def upd(m, v, p=p, g=g, shadow=shadow):
                check(lib().qlrt_adam_step(ptr(p), ptr(g), ptr(m), ptr(v), p.numel(), *consts, ptr(shadow),
                                           stream_ptr()), "AdamOptimizer.step")

            self.store.update(name, p, upd)
            # the kernel wrote p through its pointer: bump its version so the
            # layers' bf16 operand copies (LoraAdapter.bf16_operands) refresh
            torch.autograd.graph.increment_version(p)
            nxt = names[i + 1] if i + 1 < len(names) else None
            if nxt is not None and hasattr(self.store, "prefetch"):
                self.store.prefetch(nxt)  # look-ahead: the next moments migrate while this update runs


def check_finite(loss: float, norm: float, step: int) -> None:
    """The trainer's divergence guard (training.py:496-503)."""
    if not math.isfinite(loss):
        raise TrainingDivergedError(f"non-finite loss at step {step}")
    if not math.isfinite(norm):
        raise TrainingDivergedError(f"non-finite gradient norm at step {step}")


__all__ = ["TrainConfig", "PlainMomentStore", "PagedMomentStore", "AdamOptimizer", "clip_global_norm",
           "global_sumsq", "pairwise_sumsq", "check_finite", "OPTIMIZERS"]
