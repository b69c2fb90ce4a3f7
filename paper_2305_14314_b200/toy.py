"""GPU-backed toy models and trainer: the reference's desk-scale QLoRA harness
(pkg/src/qlrt/qlora.py:177-362, pkg/src/qlrt/training.py:93-572) on this
package's kernels, as the system-level parity gate of SURVEY.md §8(f) rank 3
(acceptance criteria 6-8, pkg/tests/test_acceptance.py:122-209).

What runs where:

* every frozen base is quantized by the GPU quantizer (bit-exact codes and
  double-quant constants) and dequantized by the GPU dequantizer on every
  forward, as the reference does (qlora.py:117-122);
* the toy layers (16 x 16, 2 x 16, 16 x 1) sit far below any tile of the fused
  NF4 GEMM, so ``QLinear`` runs them at the layer precision (float32, or
  float64 for the gradient gate) through cuBLAS (``QLinear._forward_exact``,
  the reference's op order);
* the optimizer is the bit-exact fp32 Adam kernel with the device fp64
  global-norm clip, moments plain or in the unified-memory ``Pager``
  (training.py:354-442);
* data comes from the reference's named numpy substreams of the run seed
  (training.py:46-60), so a seed names the same task, batches, adapter init
  and dropout masks as the reference.

``train_toy(..., graph=True)`` captures one training step in a CUDA graph
(batches pre-drawn from the data stream and indexed by a device step
counter, clip and Adam constants read on the device, loss and gradient norm
written to device arrays): the 16 000-step criterion-7 runs replay it.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Any

import numpy as np
import torch

from ._native import check, lib, ptr, stream_ptr
from .blockquant import BlockQuantized, quantize
from .codebooks import get_codebook
from .errors import TrainingDivergedError
from .paging import PagerConfig, pager_open
from .qlora import PLACEMENTS, QLinear, lora_init
from .training import (OPTIMIZERS, AdamOptimizer, PagedMomentStore, PlainMomentStore, TrainConfig, clip_global_norm,
                       pairwise_sumsq)

TASKS = ("regression", "moons")
DTYPES = ("fp32", "nf4", "nf-eq4", "fp4-e2m1", "fp4-e3m0", "int4")
_QV_LABELS = ("q", "v")
_ACTIVATIONS = ("identity", "tanh", "relu")

# substreams of the run seed; every consumer owns one stream id (training.py:46-60)
_STREAM_INIT = 0
_STREAM_TEACHER = 1
_STREAM_ADAPTER = 2
_STREAM_EVAL = 3
_STREAM_DATA = 4
_STREAM_DROPOUT = 5


def _stream(seed: int, stream_id: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((seed, stream_id)))


def _dev(a, dtype=None) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    return t if dtype is None else t.to(dtype)


# ---------------------------------------------------------------------------
# layers and model (qlora.py:177-362)


class DenseLinear:
    """Full-precision linear layer; trainable unless frozen (qlora.py:177-216)."""

    def __init__(self, weight, trainable: bool = True, dtype=torch.float32):
        self.dtype = dtype
        self.w = torch.as_tensor(weight).to(device="cuda", dtype=dtype).contiguous()
        self.trainable_flag = trainable

    @property
    def in_dim(self) -> int:
        return int(self.w.shape[0])

    @property
    def out_dim(self) -> int:
        return int(self.w.shape[1])

    def forward(self, x, train: bool = False, rng=None):
        x = torch.as_tensor(x).to(device="cuda", dtype=self.dtype)
        return x @ self.w, {"x": x}

    def backward(self, d_y, cache):
        d_y = torch.as_tensor(d_y).to(device="cuda", dtype=self.dtype)
        d_x = d_y @ self.w.T
        grads = {"w": cache["x"].T @ d_y} if self.trainable_flag else {}
        return d_x, grads

    def trainable(self) -> dict:
        return {"w": self.w} if self.trainable_flag else {}


@dataclass
class Layer:
    label: str
    linear: Any
    activation: str = "identity"

    def __post_init__(self) -> None:
        if self.activation not in _ACTIVATIONS:
            raise ValueError(f"unknown activation {self.activation!r}")


class ToyModel:
    """A stack of labeled linear layers with elementwise nonlinearities
    (qlora.py:229-303)."""

    def __init__(self, layers: list, placement: str = "none"):
        if placement not in PLACEMENTS:
            raise ValueError(f"placement must be one of {PLACEMENTS}")
        self.layers = layers
        self.placement = placement

    def forward(self, x, train: bool = False, rng=None):
        caches = []
        h = x
        for layer in self.layers:
            z, lin_cache = layer.linear.forward(h, train=train, rng=rng)
            if layer.activation == "tanh":
                h = torch.tanh(z)
            elif layer.activation == "relu":
                h = torch.clamp_min(z, 0)
            else:
                h = z
            caches.append({"lin": lin_cache, "z": z, "h": h})
        return h, caches

    def backward(self, d_out, caches) -> dict:
        grads: dict = {}
        d_h = d_out
        for layer, cache in zip(reversed(self.layers), reversed(caches)):
            if layer.activation == "tanh":
                d_z = d_h * (1.0 - cache["h"] * cache["h"])
            elif layer.activation == "relu":
                d_z = d_h * (cache["z"] > 0)
            else:
                d_z = d_h
            d_h, lin_grads = layer.linear.backward(d_z, cache["lin"])
            for name, g in lin_grads.items():
                grads[f"{layer.label}.{name}"] = g
        return grads

    def trainable_params(self) -> dict:
        params: dict = {}
        for layer in self.layers:
            for name, arr in layer.linear.trainable().items():
                params[f"{layer.label}.{name}"] = arr
        return params

    def base_fingerprint(self) -> bytes:
        """Byte snapshot of every frozen quantized base (qlora.py:285-303)."""
        parts = []
        for layer in self.layers:
            lin = layer.linear
            if not isinstance(lin, QLinear):
                continue
            b = lin.base
            if not isinstance(b, BlockQuantized):
                parts.append(torch.as_tensor(b).cpu().numpy().tobytes())
                continue
            parts.append(b.codes.cpu().numpy().tobytes())
            if b.constants is not None:
                parts.append(b.constants.cpu().numpy().tobytes())
            if b.dq is not None:
                parts += [b.dq.c1.cpu().numpy().tobytes(), b.dq.codes.cpu().numpy().tobytes(),
                          b.dq.mu.cpu().numpy().astype(np.float32).tobytes()]
        return b"".join(parts)


def attach_adapters(model: ToyModel, placement: str, rank: int, alpha: float, rng: np.random.Generator,
                    dropout_p: float = 0.0) -> None:
    """Adapters on the layers ``placement`` selects, drawn from ``rng`` in
    layer order; rank clamped to min(in, out) (qlora.py:306-344)."""
    if placement not in PLACEMENTS:
        raise ValueError(f"placement must be one of {PLACEMENTS}")
    model.placement = placement
    if placement == "none":
        return
    for layer in model.layers:
        if not isinstance(layer.linear, QLinear):
            continue
        if placement == "qv_only" and layer.label.split(".")[-1] not in _QV_LABELS:
            continue
        lin = layer.linear
        layer_rank = min(rank, lin.in_dim, lin.out_dim)
        lin.adapters.append(lora_init(lin.in_dim, lin.out_dim, layer_rank, alpha, rng, dropout_p=dropout_p,
                                      dtype=lin.dtype))


def quantize_dense_stack(weights: list, codebook, blocksize: int = 64, double_quant: bool = True,
                         dtype=torch.float32) -> list:
    """Adapter-less QLinear layers over GPU-quantized dense weights (qlora.py:347-362)."""
    return [QLinear(quantize(torch.as_tensor(w).to("cuda"), codebook, blocksize, double_quant=double_quant),
                    adapters=[], dtype=dtype) for w in weights]


# ---------------------------------------------------------------------------
# tasks (training.py:148-292)


def _mse_loss(pred: torch.Tensor, target: torch.Tensor):
    """(device fp64 loss, gradient) -- training.py:148-152."""
    diff = pred - target.to(pred.dtype)
    loss = torch.mean(torch.square(diff.double()))
    return loss, (2.0 / diff.numel()) * diff


def _logistic_loss(pred: torch.Tensor, target: torch.Tensor):
    """Mean log(1 + exp(-y z)), labels in {-1, +1} -- training.py:155-161."""
    y = target.to(pred.dtype)
    margin = -y * pred
    loss = torch.mean(torch.logaddexp(torch.zeros((), dtype=pred.dtype, device=pred.device), margin).double())
    grad = (-y * torch.sigmoid(margin)) / float(pred.numel())
    return loss, grad


class RegressionTask:
    """Linear teacher-student regression over six square layers (training.py:164-225)."""

    name = "regression"
    labels = ("q", "k", "v", "o", "ffn_up", "ffn_down")

    def __init__(self, seed: int = 0, width: int = 16, teacher_rank: int = 2, teacher_delta_std: float = 0.05,
                 noise_std: float = 0.02, eval_size: int = 1024):
        self.seed = seed
        self.width = width
        self.noise_std = float(noise_std)
        self.activations = ("identity",) * len(self.labels)
        rng_init, rng_teacher, rng_eval = (_stream(seed, s) for s in (_STREAM_INIT, _STREAM_TEACHER, _STREAM_EVAL))
        w = width
        self.base_weights = [rng_init.standard_normal((w, w)) / math.sqrt(w) for _ in self.labels]
        self.teacher_weights = []
        for base in self.base_weights:
            a = rng_teacher.standard_normal((w, teacher_rank))
            b = rng_teacher.standard_normal((teacher_rank, w))
            self.teacher_weights.append(base + (teacher_delta_std / math.sqrt(teacher_rank)) * (a @ b))
        ex = rng_eval.standard_normal((eval_size, w))
        ey = self._teacher(ex) + self.noise_std * rng_eval.standard_normal((eval_size, w))
        self.eval_x, self.eval_y = _dev(ex), _dev(ey)

    def _teacher(self, x: np.ndarray) -> np.ndarray:
        h = x
        for wt in self.teacher_weights:
            h = h @ wt
        return h

    def sample_host(self, rng: np.random.Generator, n: int):
        x = rng.standard_normal((n, self.width))
        y = self._teacher(x) + self.noise_std * rng.standard_normal((n, self.width))
        return x.astype(np.float32), y.astype(np.float32)

    def sample_batch(self, rng: np.random.Generator, n: int):
        x, y = self.sample_host(rng, n)
        return _dev(x), _dev(y)

    def loss_and_grad(self, pred, target):
        return _mse_loss(pred, target)

    def eval_loss(self, model: ToyModel) -> float:
        pred, _ = model.forward(self.eval_x)
        diff = pred.double() - self.eval_y
        return float(torch.mean(diff * diff))


def _sample_moons(rng: np.random.Generator, n: int, noise: float):
    """Two interleaved half-circles, labels -1 / +1 (training.py:228-241)."""
    cls = rng.integers(0, 2, size=n)
    theta = rng.random(n) * math.pi
    x = np.empty((n, 2))
    pos = cls == 1
    x[pos, 0] = np.cos(theta[pos])
    x[pos, 1] = np.sin(theta[pos])
    x[~pos, 0] = 1.0 - np.cos(theta[~pos])
    x[~pos, 1] = 0.5 - np.sin(theta[~pos])
    x += noise * rng.standard_normal((n, 2))
    x -= np.array([0.5, 0.25])
    return x, (2.0 * cls - 1.0).reshape(n, 1)


class MoonsTask:
    """Two-moons classification under a 3-layer tanh MLP (training.py:244-280)."""

    name = "moons"
    labels = ("q", "v", "o")

    def __init__(self, seed: int = 0, hidden: int = 16, noise: float = 0.1, eval_size: int = 512):
        self.seed = seed
        self.noise = float(noise)
        self.activations = ("tanh", "tanh", "identity")
        dims = [(2, hidden), (hidden, hidden), (hidden, 1)]
        rng_init = _stream(seed, _STREAM_INIT)
        self.base_weights = [rng_init.standard_normal(d) / math.sqrt(d[0]) for d in dims]
        ex, ey = _sample_moons(_stream(seed, _STREAM_EVAL), eval_size, self.noise)
        self.eval_x, self.eval_y = _dev(ex), _dev(ey)

    def sample_host(self, rng: np.random.Generator, n: int):
        x, y = _sample_moons(rng, n, self.noise)
        return x.astype(np.float32), y.astype(np.float32)

    def sample_batch(self, rng: np.random.Generator, n: int):
        x, y = self.sample_host(rng, n)
        return _dev(x), _dev(y)

    def loss_and_grad(self, pred, target):
        return _logistic_loss(pred, target)

    def eval_loss(self, model: ToyModel) -> float:
        pred, _ = model.forward(self.eval_x)
        loss, _ = _logistic_loss(pred.double(), self.eval_y.double())
        return float(loss)


def make_task(name: str, seed: int = 0, **kwargs):
    if name == "regression":
        return RegressionTask(seed=seed, **kwargs)
    if name == "moons":
        return MoonsTask(seed=seed, **kwargs)
    raise ValueError(f"unknown task {name!r}; expected one of {TASKS}")


def build_model(task, dtype: str = "nf4", placement: str = "all_linear", rank: int = 4, alpha: float = 4.0,
                blocksize: int = 64, double_quant: bool = True, dropout_p: float = 0.0, seed: int = 0,
                precision: str = "low") -> ToyModel:
    """A ToyModel over the task's base weights (training.py:295-347): fp32 +
    none is the dense full finetune; any other dtype freezes a GPU-quantized
    base and trains adapters only."""
    if dtype not in DTYPES:
        raise ValueError(f"unknown dtype {dtype!r}; expected one of {DTYPES}")
    if precision not in ("low", "high"):
        raise ValueError("precision must be 'low' or 'high'")
    tdt = torch.float64 if precision == "high" else torch.float32
    layers = []
    for label, activation, w in zip(task.labels, task.activations, task.base_weights):
        if dtype == "fp32":
            lin = (DenseLinear(w, trainable=True, dtype=tdt) if placement == "none"
                   else QLinear(_dev(w, tdt), adapters=[], dtype=tdt))
        else:
            q = quantize(_dev(w), get_codebook(dtype), blocksize, double_quant=double_quant)
            lin = QLinear(q, adapters=[], dtype=tdt)
        layers.append(Layer(label=label, linear=lin, activation=activation))
    model = ToyModel(layers)
    attach_adapters(model, placement, rank, alpha, _stream(seed, _STREAM_ADAPTER), dropout_p=dropout_p)
    model.dtype_label = dtype
    return model


# ---------------------------------------------------------------------------
# report and trainer (training.py:93-141, 449-572)


@dataclass(frozen=True)
class TrainReport:
    task: str
    dtype: str
    placement: str
    optimizer: str
    seed: int
    steps: int
    learning_rate: float
    losses: tuple
    grad_norms: tuple
    initial_eval_loss: float
    final_eval_loss: float
    pager_stats: dict | None = None

    @property
    def final_train_loss(self) -> float:
        return self.losses[-1] if self.losses else float("nan")

    def summary(self) -> dict:
        return {"task": self.task, "dtype": self.dtype, "placement": self.placement, "optimizer": self.optimizer,
                "seed": self.seed, "steps": self.steps, "learning_rate": self.learning_rate,
                "initial_eval_loss": self.initial_eval_loss, "final_eval_loss": self.final_eval_loss,
                "final_train_loss": self.final_train_loss, "pager_stats": self.pager_stats}

    def to_jsonl(self) -> str:
        rows = [json.dumps({"step": i + 1, "loss": l, "grad_norm": g})
                for i, (l, g) in enumerate(zip(self.losses, self.grad_norms))]
        return "\n".join(rows + [json.dumps({"summary": self.summary()})]) + "\n"


def _train_graph(model: ToyModel, task, cfg: TrainConfig, params: dict, order: list, store, rng_data):
    """The step as one CUDA graph: batches pre-drawn from the data stream
    (the same draws as the eager loop), a device step counter selecting the
    batch and the Adam constants, the fused clip + Adam kernel per parameter,
    loss and norm recorded on the device.  Returns (losses, norms)."""
    n = cfg.steps
    xs, ys = zip(*(task.sample_host(rng_data, cfg.batch_size) for _ in range(n)))
    xs, ys = _dev(np.stack(xs)), _dev(np.stack(ys))
    c = cfg
    f32 = np.float32
    rows = np.empty((n, 8), dtype=np.float32)
    rows[:, 0], rows[:, 1] = f32(c.adam_beta1), f32(1.0 - c.adam_beta1)
    rows[:, 2], rows[:, 3] = f32(c.adam_beta2), f32(1.0 - c.adam_beta2)
    rows[:, 4] = [f32(1.0 - c.adam_beta1 ** t) for t in range(1, n + 1)]
    rows[:, 5] = [f32(1.0 - c.adam_beta2 ** t) for t in range(1, n + 1)]
    rows[:, 6], rows[:, 7] = f32(c.adam_eps), f32(c.learning_rate)
    table = _dev(rows)
    t_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    hyper = torch.zeros(8, dtype=torch.float32, device="cuda")
    losses = torch.zeros(n, dtype=torch.float64, device="cuda")
    norms = torch.zeros(n, dtype=torch.float64, device="cuda")
    moments = {}
    for name in order:
        p = params[name]
        moments[name] = (torch.zeros_like(p), torch.zeros_like(p))

    def step():
        x = xs.index_select(0, t_dev).squeeze(0)
        y = ys.index_select(0, t_dev).squeeze(0)
        pred, caches = model.forward(x, train=True, rng=None)
        loss, d_pred = task.loss_and_grad(pred, y)
        grads = model.backward(d_pred, caches)
        for name in order:
            grads[name] = grads[name].contiguous()
        acc = pairwise_sumsq(grads, order)  # (clip_global_norm's numpy-order total)
        hyper.copy_(table.index_select(0, t_dev).view(-1))
        for name in order:
            p, g = params[name], grads[name]
            m, v = moments[name]
            check(lib().qlrt_adam_step_dev(ptr(p), ptr(g), ptr(m), ptr(v), p.numel(), ptr(hyper), ptr(acc),
                                           float(cfg.max_grad_norm), None, stream_ptr()), "adam")
        losses.index_copy_(0, t_dev, loss.view(1))
        norms.index_copy_(0, t_dev, torch.sqrt(acc[:1]))
        t_dev.add_(1)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    snap = {k: v.clone() for k, v in params.items()}
    with torch.cuda.stream(s):
        step()  # warm-up (allocations); undone below
    torch.cuda.current_stream().wait_stream(s)
    for k, v in params.items():
        v.copy_(snap[k])
    for m, v in moments.values():
        m.zero_()
        v.zero_()
    t_dev.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(n):
        g.replay()
    torch.cuda.synchronize()
    return losses.cpu().tolist(), norms.cpu().tolist()


def train_toy(model: ToyModel, task, cfg: TrainConfig, optimizer: str = "plain",
              pager_config: PagerConfig | None = None, graph: bool = False) -> TrainReport:
    """Adam with global grad-norm clipping on the GPU; the full trajectory
    (training.py:449-542).  ``graph=True`` replays one captured step
    (plain optimizer, no dropout)."""
    cfg.validate()
    if optimizer not in OPTIMIZERS:
        raise ValueError(f"optimizer must be one of {OPTIMIZERS}")
    params = model.trainable_params()
    order = list(params)
    for name, p in params.items():
        if p.dtype != torch.float32:
            raise ValueError(f"train_toy runs the fp32 Adam kernel: {name} is {p.dtype} (use precision='low')")
    rng_data = _stream(cfg.seed, _STREAM_DATA)
    rng_dropout = _stream(cfg.seed, _STREAM_DROPOUT)
    fingerprint = model.base_fingerprint()
    pager = None
    if optimizer == "paged":
        pager = pager_open(pager_config or PagerConfig(budget_bytes=1 << 20, page_bytes=4096))
        store = PagedMomentStore(pager)
    else:
        store = PlainMomentStore()
    try:
        initial_eval = task.eval_loss(model)
        if graph:
            if optimizer != "plain" or any(getattr(ad, "dropout_p", 0.0) > 0.0 for layer in model.layers
                                           for ad in getattr(layer.linear, "adapters", [])):
                raise ValueError("graph mode needs the plain optimizer and no dropout")
            losses, norms = _train_graph(model, task, cfg, params, order, store, rng_data)
            for i, (l, gn) in enumerate(zip(losses, norms)):
                if not math.isfinite(l):
                    raise TrainingDivergedError(f"non-finite loss at step {i + 1}")
                if not math.isfinite(gn):
                    raise TrainingDivergedError(f"non-finite gradient norm at step {i + 1}")
        else:
            opt = AdamOptimizer(params, cfg, store)
            losses, norms = [], []
            for step in range(1, cfg.steps + 1):
                x, y = task.sample_batch(rng_data, cfg.batch_size)
                pred, caches = model.forward(x, train=True, rng=rng_dropout)
                loss_t, d_pred = task.loss_and_grad(pred, y)
                loss = float(loss_t)
                if not math.isfinite(loss):
                    raise TrainingDivergedError(f"non-finite loss at step {step}")
                grads = {k: v.contiguous() for k, v in model.backward(d_pred, caches).items()}
                grad_norm = clip_global_norm(grads, order, cfg.max_grad_norm)
                if not math.isfinite(grad_norm):
                    raise TrainingDivergedError(f"non-finite gradient norm at step {step}")
                opt.step(grads)
                losses.append(loss)
                norms.append(grad_norm)
        final_eval = task.eval_loss(model)
    finally:
        store.close()
        if pager is not None:
            pager.close()
    if model.base_fingerprint() != fingerprint:
        raise RuntimeError("frozen base weights changed during training")
    pager_stats = None
    if pager is not None:
        pager_stats = {"budget_bytes": pager.config.budget_bytes, "page_bytes": pager.config.page_bytes,
                       "faults": pager.faults, "evictions": pager.evictions, "bytes_read": pager.bytes_read,
                       "bytes_written": pager.bytes_written, "peak_resident_bytes": pager.peak_resident_bytes}
    return TrainReport(task=task.name, dtype=getattr(model, "dtype_label", "fp32"), placement=model.placement,
                       optimizer=optimizer, seed=cfg.seed, steps=cfg.steps, learning_rate=cfg.learning_rate,
                       losses=tuple(losses), grad_norms=tuple(norms), initial_eval_loss=initial_eval,
                       final_eval_loss=final_eval, pager_stats=pager_stats)


def run_toy_training(task_name: str, dtype: str, placement: str, cfg: TrainConfig, optimizer: str = "plain",
                     pager_config: PagerConfig | None = None, rank: int = 4, alpha: float = 4.0,
                     blocksize: int = 64, double_quant: bool = True, dropout_p: float = 0.0,
                     task_kwargs: dict | None = None, graph: bool = False) -> TrainReport:
    """Task and model from the config seed, then train (training.py:545-572)."""
    task = make_task(task_name, seed=cfg.seed, **(task_kwargs or {}))
    model = build_model(task, dtype=dtype, placement=placement, rank=rank, alpha=alpha, blocksize=blocksize,
                        double_quant=double_quant, dropout_p=dropout_p, seed=cfg.seed)
    return train_toy(model, task, cfg, optimizer=optimizer, pager_config=pager_config, graph=graph)


__all__ = ["DenseLinear", "Layer", "ToyModel", "attach_adapters", "quantize_dense_stack", "RegressionTask",
           "MoonsTask", "make_task", "build_model", "TrainReport", "train_toy", "run_toy_training", "TASKS",
           "DTYPES"]
