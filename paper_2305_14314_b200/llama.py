"""LLaMA-shaped QLoRA finetuning harness on the B200 kernels (SURVEY.md §8(f)
rank 1; BASELINE configs C3 = LLaMA-7B shapes on 1 GPU and C5 = LLaMA-33B
shapes data-parallel).

The reference trains a toy MLP (pkg/src/qlrt/qlora.py:229-303) and has no
transformer; this harness exists to *measure* the hot path at LLaMA scale:
every linear layer (q, k, v, o, gate, up, down) is a frozen NF4 + DQ base with
a bf16-operand LoRA adapter running through the fused tcgen05 kernels
(``QLinear``, qlora.py:91-167 semantics); the glue -- RMSNorm, RoPE, SwiGLU,
causal attention (PyTorch SDPA), the frozen bf16 embedding and lm_head
(cuBLAS) and the loss -- is PyTorch.  Weights are random N(0, 0.02) (no
checkpoints offline), tokens synthetic.

Training step = forward, backward (adapter gradients written straight into
one flat fp32 bucket), data-parallel mean all-reduce of that bucket only
(NCCL over NVLink; per group of layers, launched as soon as the group's
gradients land so it overlaps the rest of the backward --
``parallel.LayerReducer``), fused global-norm clip + bit-exact Adam
(``qlrt_adam_step_dev``), bf16 operand shadows refreshed in the same pass.

Optimizer state: ``optimizer="plain"`` keeps the Adam moments in one flat
device buffer and the whole step captures into one CUDA graph;
``optimizer="paged"`` keeps them in unified-memory pages under a
:class:`~paper_2305_14314_b200.paging.Pager` budget (the reference's
PagedMomentStore, training.py:371-395: one slab per layer holding its m then
v), the forward/backward still one CUDA graph and the optimizer walking the
layer slabs with look-ahead prefetch on the pager's side streams; once every
slab is resident under a budget that holds them all
(``optimizer_resident()``) the optimizer issues no migration and the whole
step captures into one graph.  The walk
alternates direction every step (an elevator scan), so the reference's LRU
keeps exactly the slabs the next step needs first and evicts the ones it has
finished with; each parameter's update is independent, so the order changes
no bit of the result (paged == plain).

``checkpoint=True`` recomputes each decoder layer's forward in the backward
(activation memory O(1 layer) instead of O(layers); +2P FLOPs per token).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F
import torch.utils.checkpoint as _ckpt

from . import _native
from ._native import check, lib, ptr, stream_ptr
from .blockquant import quantize
from .codebooks import get_codebook
from .paging import Pager, PagerConfig
from .parallel import GradBucket, LayerReducer
from .qlora import LoraAdapter, QLinear, QLinearGroup, side_join
from .training import TrainConfig, _sumsq_scratch

PROJS = ("q", "k", "v", "o", "gate", "up", "down")
# the projections as issued: siblings that read the same input form one unit
UNITS_GROUPED = (("qkv", ("q", "k", "v")), ("o", ("o",)), ("gu", ("gate", "up")), ("down", ("down",)))


@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int = 32
    hidden: int = 4096
    ffn: int = 11008
    n_heads: int = 32
    vocab: int = 32000
    seq: int = 512
    rank: int = 64
    alpha: float = 16.0
    rms_eps: float = 1e-6
    rope_theta: float = 10000.0

    @staticmethod
    def llama7b(**kw) -> "LlamaConfig":
        return LlamaConfig(**kw)

    @staticmethod
    def llama33b(**kw) -> "LlamaConfig":
        return LlamaConfig(n_layers=60, hidden=6656, ffn=17920, n_heads=52, **kw)

    @staticmethod
    def tiny(**kw) -> "LlamaConfig":
        base = dict(n_layers=2, hidden=256, ffn=512, n_heads=4, vocab=512, seq=64, rank=16)
        base.update(kw)
        return LlamaConfig(**base)

    def proj_shape(self, name: str) -> tuple[int, int]:
        h, f = self.hidden, self.ffn
        return {"q": (h, h), "k": (h, h), "v": (h, h), "o": (h, h), "gate": (h, f), "up": (h, f),
                "down": (f, h)}[name]

    @property
    def linear_params(self) -> int:
        return self.n_layers * sum(a * b for a, b in map(self.proj_shape, PROJS))

    @property
    def lora_params(self) -> int:
        return self.n_layers * sum(self.rank * (a + b) for a, b in map(self.proj_shape, PROJS))

    def flops_per_token(self) -> float:
        """fwd 2P + bwd-to-input 2P over the frozen linears, 6 P_lora for the
        adapters, causal attention (QK^T and PV, fwd + bwd 3x, half masked
        counted in full as the SDPA kernels do the work) and the lm_head
        (fwd + bwd-to-input): SURVEY.md §8(d) C3."""
        p, pl = self.linear_params, self.lora_params
        attn = 3 * self.n_layers * 4 * self.seq * self.hidden
        head = 4 * self.vocab * self.hidden
        return 2 * p + 2 * p + 6 * pl + attn + head


class _QLinearFn(torch.autograd.Function):
    """Autograd bridge to QLinear.forward / backward (qlora.py:124-167); the
    adapter gradients go to the bucket views, not to autograd."""

    @staticmethod
    def forward(ctx, x, anchor, layer, gviews, notify, defer):
        y, cache = layer.forward(x)
        ctx.layer, ctx.cache, ctx.gviews, ctx.notify, ctx.defer = layer, cache, gviews, notify, defer
        return y

    @staticmethod
    def backward(ctx, dy):
        dx, _ = ctx.layer.backward(dy.contiguous(), ctx.cache, grads_out=ctx.gviews,
                                   defer=ctx.defer() if ctx.defer is not None else None)
        ctx.cache = None
        if ctx.notify is not None:  # this projection's adapter gradients are issued
            ctx.notify()
        return dx, None, None, None, None, None


class _QKVFn(torch.autograd.Function):
    """q | k | v as one grouped NF4 linear (QLinearGroup: one Ts GEMM, one
    fused grid, one dl1 GEMM), RoPE applied to the q and k column slices of
    the concatenated output; the backward builds d[q | k | v] in place
    (inverse RoPE into the slices) and runs the grouped backward once."""

    @staticmethod
    def forward(ctx, x, anchor, grp, gviews, notify, defer, cos_sin, nh):
        b, s, h = x.shape
        d = h // nh
        ycat, cache = grp.forward(x)
        q = torch.empty(b, s, nh, d, dtype=ycat.dtype, device=ycat.device)
        k, v = torch.empty_like(q), torch.empty_like(q)
        check(lib().qlrt_rope_qkv_fwd(ptr(ycat), ptr(q), ptr(k), ptr(v), ptr(cos_sin), b * s, nh, d, s, stream_ptr()),
              "rope qkv")
        ctx.grp, ctx.cache, ctx.gviews, ctx.notify, ctx.defer = grp, cache, gviews, notify, defer
        ctx.save_for_backward(cos_sin)
        ctx.dims = (b, s, h, nh, d)
        return q, k, v

    @staticmethod
    def backward(ctx, dq, dk, dv):
        (cos_sin,) = ctx.saved_tensors
        b, s, h, nh, d = ctx.dims
        dq, dk, dv = dq.contiguous(), dk.contiguous(), dv.contiguous()
        dycat = torch.empty(b * s, 3 * h, dtype=dq.dtype, device=dq.device)
        check(lib().qlrt_rope_qkv_bwd(ptr(dq), ptr(dk), ptr(dv), ptr(dycat), ptr(cos_sin), b * s, nh, d, s,
                                      stream_ptr()), "rope qkv bwd")
        dx = ctx.grp.backward(dycat, ctx.cache, ctx.gviews["l1"], ctx.gviews["l2"],
                              defer=ctx.defer() if ctx.defer is not None else None)
        ctx.cache = None
        if ctx.notify is not None:
            ctx.notify()
        return dx.view(b, s, h), None, None, None, None, None, None, None


class _GateUpFn(torch.autograd.Function):
    """gate | up as one grouped NF4 linear, SwiGLU over the concatenated
    output; the backward writes d[gate | up] in place and runs the grouped
    backward once."""

    @staticmethod
    def forward(ctx, x, anchor, grp, gviews, notify, defer):
        b, s, h = x.shape
        f = grp.n_member
        ycat, cache = grp.forward(x)
        out = torch.empty(b * s, f, dtype=ycat.dtype, device=ycat.device)
        check(lib().qlrt_swiglu_cat_fwd(ptr(ycat), ptr(out), b * s, f, stream_ptr()), "swiglu")
        ctx.grp, ctx.cache, ctx.gviews, ctx.notify, ctx.defer = grp, cache, gviews, notify, defer
        ctx.save_for_backward(ycat)
        ctx.dims = (b, s, h, f)
        return out.view(b, s, f)

    @staticmethod
    def backward(ctx, dout):
        (ycat,) = ctx.saved_tensors
        b, s, h, f = ctx.dims
        dgu = torch.empty_like(ycat)
        check(lib().qlrt_swiglu_cat_bwd(ptr(ycat), ptr(dout.contiguous()), ptr(dgu), b * s, f, stream_ptr()),
              "swiglu bwd")
        dx = ctx.grp.backward(dgu, ctx.cache, ctx.gviews["l1"], ctx.gviews["l2"],
                              defer=ctx.defer() if ctx.defer is not None else None)
        ctx.cache = None
        if ctx.notify is not None:
            ctx.notify()
        return dx.view(b, s, h), None, None, None, None, None


class _RMSNormFn(torch.autograd.Function):
    """y = x * rsqrt(mean(x^2) + eps) (frozen unit weight), fused kernels."""

    @staticmethod
    def forward(ctx, x, eps):
        x = x.contiguous()
        h = x.shape[-1]
        rows = x.numel() // h
        y = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        check(lib().qlrt_rmsnorm_fwd(ptr(x), ptr(y), ptr(rstd), rows, h, float(eps), stream_ptr()), "rmsnorm")
        ctx.save_for_backward(x, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, rstd = ctx.saved_tensors
        dy = dy.contiguous()
        dx = torch.empty_like(x)
        h = x.shape[-1]
        check(lib().qlrt_rmsnorm_bwd(ptr(dy), ptr(x), ptr(rstd), ptr(dx), x.numel() // h, h, stream_ptr()),
              "rmsnorm bwd")
        return dx, None


class _SwiGLUFn(torch.autograd.Function):
    """silu(g) * u, fused kernels."""

    @staticmethod
    def forward(ctx, g, u):
        g, u = g.contiguous(), u.contiguous()
        out = torch.empty_like(g)
        check(lib().qlrt_swiglu_fwd(ptr(g), ptr(u), ptr(out), g.numel(), stream_ptr()), "swiglu")
        ctx.save_for_backward(g, u)
        return out

    @staticmethod
    def backward(ctx, dout):
        g, u = ctx.saved_tensors
        dout = dout.contiguous()
        dg, du = torch.empty_like(g), torch.empty_like(u)
        check(lib().qlrt_swiglu_bwd(ptr(g), ptr(u), ptr(dout), ptr(dg), ptr(du), g.numel(), stream_ptr()),
              "swiglu bwd")
        return dg, du


class _RoPEFn(torch.autograd.Function):
    """Rotary embedding of adjacent pairs on [b, s, heads, d]; the backward
    rotates the gradient back."""

    @staticmethod
    def forward(ctx, t, cos_sin):
        t = t.contiguous()
        b, s, nh, d = t.shape
        y = torch.empty_like(t)
        check(lib().qlrt_rope(ptr(t), ptr(y), ptr(cos_sin), b * s, nh, d, s, 0, stream_ptr()), "rope")
        ctx.save_for_backward(cos_sin)
        ctx.shape = (b, s, nh, d)
        return y

    @staticmethod
    def backward(ctx, dy):
        (cos_sin,) = ctx.saved_tensors
        b, s, nh, d = ctx.shape
        dy = dy.contiguous()
        dx = torch.empty_like(dy)
        check(lib().qlrt_rope(ptr(dy), ptr(dx), ptr(cos_sin), b * s, nh, d, s, 1, stream_ptr()), "rope bwd")
        return dx, None


class _XentFn(torch.autograd.Function):
    """Mean cross entropy straight from the bf16 logits (no fp32 copy of the
    [tokens x vocab] matrix): per-row logsumexp in one pass; the backward
    recomputes softmax - onehot from the saved logsumexp."""

    @staticmethod
    def forward(ctx, logits, targets):
        rows, vocab = logits.shape
        logits = logits.contiguous()
        tg = targets.reshape(-1).to(torch.int64).contiguous()
        loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
        lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
        check(lib().qlrt_xent_fwd(ptr(logits), ptr(tg), rows, vocab, ptr(loss), ptr(lse), stream_ptr()), "xent")
        ctx.save_for_backward(logits, tg, lse)
        return loss.mean()

    @staticmethod
    def backward(ctx, g):
        logits, tg, lse = ctx.saved_tensors
        rows, vocab = logits.shape
        d = torch.empty_like(logits)
        g = g.to(torch.float32).reshape(1).contiguous()
        check(lib().qlrt_xent_bwd(ptr(logits), ptr(tg), ptr(lse), ptr(g), rows, vocab, ptr(d), stream_ptr()),
              "xent bwd")
        return d, None


class _AddRMSNormFn(torch.autograd.Function):
    """Residual add fused into the following RMSNorm: s = x + d, y =
    rmsnorm(s) in one kernel; the backward adds the norm's gradient and the
    residual stream's own gradient in one kernel, for both inputs."""

    @staticmethod
    def forward(ctx, x, d, eps):
        x, d = x.contiguous(), d.contiguous()
        h = x.shape[-1]
        rows = x.numel() // h
        s = torch.empty_like(x)
        y = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        check(lib().qlrt_add_rmsnorm_fwd(ptr(x), ptr(d), ptr(s), ptr(y), ptr(rstd), rows, h, float(eps),
                                         stream_ptr()), "add + rmsnorm")
        ctx.save_for_backward(s, rstd)
        return s, y

    @staticmethod
    def backward(ctx, ds, dy):
        s, rstd = ctx.saved_tensors
        h = s.shape[-1]
        rows = s.numel() // h
        if dy is None:
            return ds, ds, None
        dx = torch.empty_like(s)
        dy = dy.contiguous()
        if ds is None:
            check(lib().qlrt_rmsnorm_bwd(ptr(dy), ptr(s), ptr(rstd), ptr(dx), rows, h, stream_ptr()), "rmsnorm bwd")
        else:
            check(lib().qlrt_rmsnorm_bwd_add(ptr(dy), ptr(s), ptr(rstd), ptr(ds.contiguous()), ptr(dx), rows, h,
                                             stream_ptr()), "rmsnorm bwd + residual")
        return dx, dx, None


def _rmsnorm(x: torch.Tensor, eps: float) -> torch.Tensor:
    return _RMSNormFn.apply(x, eps)


def _rope(t: torch.Tensor, cos_sin: torch.Tensor) -> torch.Tensor:
    """Rotary embedding on [b, s, heads, d]; cos_sin fp32 [s, d/2, 2]."""
    return _RoPEFn.apply(t, cos_sin)


def rope_reference(t: torch.Tensor, cos_sin: torch.Tensor) -> torch.Tensor:
    """Plain PyTorch statement of the same rotation (tests)."""
    tt = t.float().reshape(*t.shape[:-1], -1, 2)
    c, s_ = cos_sin[None, :, None, :, 0], cos_sin[None, :, None, :, 1]
    x0, x1 = tt[..., 0], tt[..., 1]
    return torch.stack((x0 * c - x1 * s_, x0 * s_ + x1 * c), dim=-1).flatten(-2)


class LlamaQLoRA:
    """Frozen NF4 LLaMA-shaped decoder with LoRA on every linear layer.

    group: the data-parallel process group (None = the default group when
    torch.distributed is initialized, else single rank).  optimizer:
    "plain" | "paged"; pager_budget_bytes bounds the device-resident moment
    bytes of the paged store (default: all of them).  bucket_layers: layers
    per overlapped all-reduce; wire_dtype: float32 (exact) or bfloat16.
    """

    def __init__(self, cfg: LlamaConfig, device="cuda", seed: int = 0, train_cfg: TrainConfig | None = None, *,
                 group=None, optimizer: str = "plain", pager_budget_bytes: int | None = None,
                 page_bytes: int = 2 << 20, lookahead: int = 2, checkpoint: bool = False, bucket_layers: int = 4,
                 wire_dtype=torch.float32, max_steps: int = 100_000, defer_lag: int | None = 1,
                 grouped: bool | None = None):
        if optimizer not in ("plain", "paged"):
            raise ValueError(f"optimizer must be 'plain' or 'paged', got {optimizer!r}")
        self.cfg = cfg
        self.dev = torch.device(device)
        self.train_cfg = train_cfg or TrainConfig()
        self.checkpoint = checkpoint
        self.optimizer = optimizer
        # deferred adapter gradients: each projection's dl2 / dl1 GEMMs stay on
        # the library's side stream (QLRT_BWD_DEFER) and run beside the next
        # projections' fused grids; layer li's are waited for (and its bucket
        # span handed to the all-reduce) once layer li - defer_lag has issued
        # its backward.  None: every backward joins its own side work.
        self.defer_lag = defer_lag
        self._inflight: dict = {}
        self._side_ev: dict = {}
        self._ready_q: list = []
        self.lookahead = lookahead
        g = torch.Generator(device=self.dev).manual_seed(seed)
        cb = get_codebook("nf4")
        h, v = cfg.hidden, cfg.vocab
        self.embed = (torch.randn(v, h, device=self.dev, generator=g) * 0.02).to(torch.bfloat16)
        self.lm_head = (torch.randn(h, v, device=self.dev, generator=g) * 0.02).to(torch.bfloat16)
        # sibling projections that share their input run as one grouped call
        # (q | k | v, gate | up: QLinearGroup) when the shapes allow it
        if grouped is None:
            grouped = cfg.rank % 64 == 0 and h % 256 == 0 and cfg.ffn % 256 == 0
        self.grouped = bool(grouped)
        self.units = (UNITS_GROUPED if self.grouped else tuple((pj, (pj,)) for pj in PROJS))
        # one flat fp32 buffer each for adapter parameters and gradients (layer
        # after layer, so a layer's -- and a group of layers' -- tensors are
        # contiguous; a unit's l1 [K][G r] / l2 [r][G N] blocks are contiguous);
        # a flat bf16 buffer for the MMA operand shadows (same layout)
        r = cfg.rank
        ushapes = {}
        for li in range(cfg.n_layers):
            for un, members in self.units:
                a_, b_ = cfg.proj_shape(members[0])
                ushapes[f"{li}.{un}.l1"] = (a_, len(members) * r)
                ushapes[f"{li}.{un}.l2"] = (r, len(members) * b_)
        self.bucket = GradBucket(ushapes, self.dev)         # gradients (all-reduced)
        pbuf = GradBucket(ushapes, self.dev)                # parameters
        self.params_flat = pbuf.flat
        self.shadow_flat = torch.zeros(self.params_flat.numel(), dtype=torch.bfloat16, device=self.dev)
        self.uparams, self.ugrads = pbuf.views(), self.bucket.views()
        ushadows, off = {}, 0
        for n, shp in ushapes.items():
            k_ = int(np.prod(shp))
            ushadows[n] = self.shadow_flat[off: off + k_].view(shp)
            off += k_
        # per-projection names / views (member g = column slice g of its unit)
        names, self.params, self.gviews, shadows = [], {}, {}, {}
        for li in range(cfg.n_layers):
            for un, members in self.units:
                a_, b_ = cfg.proj_shape(members[0])
                for g_, pj in enumerate(members):
                    for src, dst in ((self.uparams, self.params), (self.ugrads, self.gviews), (ushadows, shadows)):
                        dst[f"{li}.{pj}.l1"] = src[f"{li}.{un}.l1"][:, g_ * r:(g_ + 1) * r]
                        dst[f"{li}.{pj}.l2"] = src[f"{li}.{un}.l2"][:, g_ * b_:(g_ + 1) * b_]
                    names += [f"{li}.{pj}.l1", f"{li}.{pj}.l2"]
        self.names = names
        offs = self.bucket.offsets()
        self.layer_spans = []
        for li in range(cfg.n_layers):
            first = offs[f"{li}.{self.units[0][0]}.l1"][0]
            last_off, last_n = offs[f"{li}.{self.units[-1][0]}.l2"]
            self.layer_spans.append((first, last_off + last_n - first))
        self.pager = None
        if optimizer == "plain":
            self.m_flat = torch.zeros_like(self.params_flat)
            self.v_flat = torch.zeros_like(self.params_flat)
        else:
            # default budget: every slab resident (page-rounded), i.e. no eviction
            state = sum((2 * n * 4 + page_bytes - 1) // page_bytes * page_bytes for _, n in self.layer_spans)
            self.pager = Pager(PagerConfig(budget_bytes=pager_budget_bytes or state, page_bytes=page_bytes))
            self.mslabs = [self.pager.alloc(2 * n * 4) for _, n in self.layer_spans]
        self.reducer = LayerReducer(self.bucket.flat, self.layer_spans, bucket_layers, group, wire_dtype)
        self._pending = [len(self.units)] * cfg.n_layers
        self.layers = []
        for li in range(cfg.n_layers):
            lay = {}
            qs = {}
            for pj in PROJS:
                a_, b_ = cfg.proj_shape(pj)
                w = torch.randn(a_, b_, device=self.dev, generator=g) * 0.02
                qs[pj] = quantize(w, cb, 64, double_quant=True)
                del w
                l1, l2 = self.params[f"{li}.{pj}.l1"], self.params[f"{li}.{pj}.l2"]
                l1.copy_(torch.randn(a_, r, device=self.dev, generator=g) / math.sqrt(r))
                l2.zero_()  # lora_init: l2 = 0 (qlora.py:63-80)
                ad = LoraAdapter(r, cfg.alpha, l1, l2)
                if r % 8 == 0 and not self.grouped:  # the kernels read the shadows in place; Adam refreshes them
                    s1, s2 = shadows[f"{li}.{pj}.l1"], shadows[f"{li}.{pj}.l2"]
                    s1.copy_(l1)
                    s2.copy_(l2)
                    ad.adopt_shadows(s1, s2)
                lay[pj] = QLinear(qs[pj], [ad])
                lay[pj + ".g"] = {"adapter0.l1": self.gviews[f"{li}.{pj}.l1"],
                                  "adapter0.l2": self.gviews[f"{li}.{pj}.l2"]}
            if self.grouped:
                for un, members in self.units:
                    if len(members) == 1:
                        pj = members[0]
                        lay[un] = QLinear(qs[pj], [LoraAdapter(r, cfg.alpha, self.uparams[f"{li}.{un}.l1"],
                                                               self.uparams[f"{li}.{un}.l2"])])
                        lay[un].adapters[0].adopt_shadows(ushadows[f"{li}.{un}.l1"], ushadows[f"{li}.{un}.l2"])
                        lay[un + ".g"] = {"adapter0.l1": self.ugrads[f"{li}.{un}.l1"],
                                          "adapter0.l2": self.ugrads[f"{li}.{un}.l2"]}
                    else:
                        lay[un] = QLinearGroup([qs[pj] for pj in members], self.uparams[f"{li}.{un}.l1"],
                                               self.uparams[f"{li}.{un}.l2"], r, cfg.alpha,
                                               l1b=ushadows[f"{li}.{un}.l1"], l2b=ushadows[f"{li}.{un}.l2"])
                        lay[un + ".g"] = {"l1": self.ugrads[f"{li}.{un}.l1"], "l2": self.ugrads[f"{li}.{un}.l2"]}
            lay["notify"] = (lambda li=li: self._proj_done(li))
            lay["index"] = li
            self.layers.append(lay)
        if self.grouped:
            self.shadow_flat.copy_(self.params_flat)
        self._build_constant_jobs()
        d = h // cfg.n_heads
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, d, 2, device=self.dev, dtype=torch.float32) / d))
        ang = torch.outer(torch.arange(cfg.seq, device=self.dev, dtype=torch.float32), inv)
        self.cos_sin = torch.stack((torch.cos(ang), torch.sin(ang)), dim=-1).contiguous()  # fp32 [seq, d/2, 2]
        self.anchor = torch.zeros(1, device=self.dev, requires_grad=True)
        self.t = 0
        self._scans = 0
        # the Adam constants of every step t = 1..max_steps, as the float32
        # values numpy 2 uses in the reference update (training.py:426-442);
        # a device step counter selects the row, so a captured step replays
        # with the right bias corrections and no host write races the GPU
        c = self.train_cfg
        f32 = np.float32
        rows = np.empty((max_steps, 8), dtype=np.float32)
        rows[:, 0], rows[:, 1] = f32(c.adam_beta1), f32(1.0 - c.adam_beta1)
        rows[:, 2], rows[:, 3] = f32(c.adam_beta2), f32(1.0 - c.adam_beta2)
        rows[:, 4] = [f32(1.0 - c.adam_beta1 ** t) for t in range(1, max_steps + 1)]
        rows[:, 5] = [f32(1.0 - c.adam_beta2 ** t) for t in range(1, max_steps + 1)]
        rows[:, 6], rows[:, 7] = f32(c.adam_eps), f32(c.learning_rate)
        self.hyper_table = torch.from_numpy(rows).to(self.dev)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)  # steps taken
        self.hyper = torch.zeros(8, dtype=torch.float32, device=self.dev)
        self.sumsq = _sumsq_scratch(self.dev)

    # ------------------------------------------------------------------ model
    def _build_constant_jobs(self) -> None:
        """The frozen bases' block constants are double-dequantized once per
        step for every linear in ONE launch (qlrt_nf4_constants_batch) into
        per-unit caches the fused kernels read (the per-call prepass chain --
        one or more small launches in front of every fused GEMM -- leaves the
        critical path).  The caches hold what the forward kept for the
        backward anyway (the reference keeps cache['w'], qlora.py:146-147)."""
        L = lib()
        jobs, self._consts = [], []
        max_elems = 1
        for lay in self.layers:
            for un, members in self.units:
                lin = lay[un] if self.grouped else lay[members[0]]
                a_, b_ = self.cfg.proj_shape(members[0])
                pitch = int(L.qlrt_nf4_constants_bytes(a_, len(members) * b_)) // 4 // a_
                buf = torch.zeros(a_, pitch, dtype=torch.float32, device=self.dev)
                lin.consts_cache = buf
                self._consts.append(buf)
                nbr = b_ // 64
                for g_, pj in enumerate(members):
                    q = lay[pj].base
                    j = _native.ConstJob()
                    j.dq_codes, j.c1, j.mu = ptr(q.dq.codes), ptr(q.dq.c1), ptr(q.dq.mu)
                    j.out = ptr(buf) + 4 * g_ * nbr
                    j.rows, j.nbr, j.pitch, j.blocksize2 = a_, nbr, pitch, q.dq.blocksize2
                    j.spec = q.dq.spec.to_c()
                    jobs.append(j)
                    max_elems = max(max_elems, a_ * nbr)
        arr = (_native.ConstJob * len(jobs))(*jobs)
        self._const_jobs = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(self.dev)
        self._const_n, self._const_max = len(jobs), max_elems

    def refresh_constants(self) -> None:
        """The step-level block-constant prepass (one launch, capturable)."""
        check(lib().qlrt_nf4_constants_batch(ptr(self._const_jobs), self._const_n, self._const_max, stream_ptr()),
              "constants prepass")

    def _proj_done(self, li: int) -> None:
        self._pending[li] -= 1
        if self._pending[li] != 0:
            return
        if self.defer_lag is None:
            self.reducer.layer_ready(li)
            return
        # mark the side work issued through layer li; wait for (and release) the
        # layers issued defer_lag layers earlier
        ev = torch.cuda.Event()
        ev.record(self._side_stream())
        self._side_ev[li] = ev
        self._ready_q.append(li)
        while len(self._ready_q) > self.defer_lag:
            self._land(self._ready_q.pop(0))

    def _land(self, li: int) -> None:
        torch.cuda.current_stream().wait_event(self._side_ev.pop(li))
        self._inflight.pop(li, None)
        self.reducer.layer_ready(li)

    def _land_all(self) -> None:
        """Wait for every deferred adapter-gradient GEMM (end of backward)."""
        if self.defer_lag is None:
            return
        side_join()
        for li in self._ready_q:
            self._side_ev.pop(li, None)
            self._inflight.pop(li, None)
            self.reducer.layer_ready(li)
        self._ready_q = []
        self._inflight.clear()

    def _side_stream(self) -> torch.cuda.ExternalStream:
        cur = torch.cuda.current_stream()
        h = lib().qlrt_side_stream(cur.cuda_stream)
        if not h:
            raise RuntimeError("deferred adapter gradients need the library's side streams (QLRT_SIDE=1)")
        return torch.cuda.ExternalStream(h)

    def _lin(self, x, lay, pj, anchor):
        li = lay["index"]
        defer = None if self.defer_lag is None else (lambda li=li: self._inflight.setdefault(li, []))
        return _QLinearFn.apply(x, anchor, lay[pj], lay[pj + ".g"], lay["notify"], defer)

    def _layer(self, x, delta, li, anchor):
        """One decoder layer on the residual stream x + delta (the previous
        layer's last residual add is fused into this layer's first norm);
        returns (x, delta) with the layer output x + delta."""
        cfg = self.cfg
        lay = self.layers[li]
        b, s = x.shape[0], x.shape[1]
        nh, d = cfg.n_heads, cfg.hidden // cfg.n_heads
        if delta is None:
            hn = _rmsnorm(x, cfg.rms_eps)
        else:
            x, hn = _AddRMSNormFn.apply(x, delta, cfg.rms_eps)
        cs = self.cos_sin[:s]
        if self.grouped:
            defer = None if self.defer_lag is None else (lambda li=li: self._inflight.setdefault(li, []))
            q, k, v = _QKVFn.apply(hn, anchor, lay["qkv"], lay["qkv.g"], lay["notify"], defer, cs, nh)
            a = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               is_causal=True).transpose(1, 2).reshape(b, s, cfg.hidden)
            x, hn = _AddRMSNormFn.apply(x, self._lin(a, lay, "o", anchor), cfg.rms_eps)
            act = _GateUpFn.apply(hn, anchor, lay["gu"], lay["gu.g"], lay["notify"], defer)
            return x, self._lin(act, lay, "down", anchor)
        q = _rope(self._lin(hn, lay, "q", anchor).view(b, s, nh, d), cs).transpose(1, 2)
        k = _rope(self._lin(hn, lay, "k", anchor).view(b, s, nh, d), cs).transpose(1, 2)
        v = self._lin(hn, lay, "v", anchor).view(b, s, nh, d).transpose(1, 2)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(b, s, cfg.hidden)
        x, hn = _AddRMSNormFn.apply(x, self._lin(a, lay, "o", anchor), cfg.rms_eps)
        gt = self._lin(hn, lay, "gate", anchor)
        up = self._lin(hn, lay, "up", anchor)
        return x, self._lin(_SwiGLUFn.apply(gt, up), lay, "down", anchor)

    def loss(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        cfg = self.cfg
        b, s = tokens.shape
        self.refresh_constants()
        x = F.embedding(tokens, self.embed)
        delta = None
        for li in range(cfg.n_layers):
            if self.checkpoint:
                # reentrant: the layer reruns under grad in the backward; the
                # anchor (requires_grad) carries the graph through it
                x, delta = _ckpt.checkpoint(self._layer, x, delta, li, self.anchor, use_reentrant=True,
                                            preserve_rng_state=False)
            else:
                x, delta = self._layer(x, delta, li, self.anchor)
        _, x = _AddRMSNormFn.apply(x, delta, cfg.rms_eps)
        logits = x.reshape(b * s, cfg.hidden) @ self.lm_head
        if cfg.vocab % 8 == 0:
            return _XentFn.apply(logits, targets)
        return F.cross_entropy(logits.float(), targets.reshape(-1))

    # ------------------------------------------------------------------ step
    def set_step_constants(self) -> None:
        """Host mirror of the step counter (the paged optimizer's scan
        direction follows it); the constants themselves come from the device
        table row the device counter selects inside the step."""
        self.t += 1

    def forward_backward(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """Loss, backward with the overlapped adapter-gradient all-reduce, and
        the global fp64 sum of squares for the clip (capturable: no host sync)."""
        self._pending = [len(self.units)] * self.cfg.n_layers
        self._ready_q, self._side_ev = [], {}
        self.reducer.reset()
        loss = self.loss(tokens, targets)
        loss.backward()
        self._land_all()
        self.reducer.finish()
        # step t + 1's Adam constants from the table (device-side counter)
        self.hyper.copy_(self.hyper_table.index_select(0, self.t_dev).view(-1))
        self.t_dev.add_(1)
        self.sumsq.zero_()
        check(lib().qlrt_sumsq_f64(ptr(self.bucket.flat), self.bucket.flat.numel(), ptr(self.sumsq), stream_ptr()),
              "clip")
        return loss.detach()

    def _adam(self, off: int, n: int, m: torch.Tensor, v: torch.Tensor) -> None:
        check(lib().qlrt_adam_step_dev(ptr(self.params_flat) + 4 * off, ptr(self.bucket.flat) + 4 * off, ptr(m),
                                       ptr(v), n, ptr(self.hyper), ptr(self.sumsq),
                                       float(self.train_cfg.max_grad_norm), ptr(self.shadow_flat) + 2 * off,
                                       stream_ptr()), "adam")

    def optimizer_step(self) -> None:
        """Fused clip + Adam over every adapter parameter.  Plain: one launch
        over the flat buffers (capturable).  Paged: one launch per layer slab,
        elevator order, the next ``lookahead`` slabs prefetched while the
        current one updates (host-driven: the pager decides faults and
        evictions per step)."""
        if self.pager is None:
            self._adam(0, self.params_flat.numel(), self.m_flat, self.v_flat)
            return
        n_l = self.cfg.n_layers
        self._scans += 1
        order = list(range(n_l)) if self._scans % 2 == 1 else list(range(n_l - 1, -1, -1))
        for i, li in enumerate(order):
            off, n = self.layer_spans[li]
            st = self.pager.acquire(self.mslabs[li]).view(torch.float32)
            self._adam(off, n, st[:n], st[n:])
            self.pager.release(self.mslabs[li])
            for j in order[i + 1: i + 1 + self.lookahead]:
                self.pager.prefetch(self.mslabs[j])

    def optimizer_resident(self) -> bool:
        """Plain moments, or paged moments whose budget holds every slab and
        every slab's pages resident: the optimizer step issues no migration
        and makes no host decision that could differ between steps, so the
        whole train step (optimizer included) may be captured in one graph."""
        if self.pager is None:
            return True
        pb = self.pager.config.page_bytes
        pages = [p for sl in self.mslabs for p in sl.pages(pb)]
        return (len(pages) * pb <= self.pager.config.budget_bytes
                and all(self.pager.table.is_resident(p) for p in pages))

    def train_step(self, tokens: torch.Tensor, targets: torch.Tensor, group=None) -> torch.Tensor:
        """One QLoRA step; call set_step_constants() first.  Capturable as a
        whole with the plain optimizer (``group`` is accepted for backward
        compatibility; the process group is fixed at construction)."""
        loss = self.forward_backward(tokens, targets)
        self.optimizer_step()
        return loss

    def state_bytes(self) -> int:
        """Adam moment bytes (m + v, fp32) of all adapter parameters."""
        return 8 * self.params_flat.numel()

    def moments(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(m, v) as flat fp32 tensors in parameter order (a copy when paged)."""
        if self.pager is None:
            return self.m_flat, self.v_flat
        ms, vs = [], []
        for li, (off, n) in enumerate(self.layer_spans):
            st = self.pager.view(self.mslabs[li]).view(torch.float32)
            ms.append(st[:n].clone())
            vs.append(st[n:].clone())
        return torch.cat(ms), torch.cat(vs)

    def close(self) -> None:
        if self.pager is not None:
            self.pager.close()
            self.pager = None


__all__ = ["LlamaConfig", "LlamaQLoRA", "PROJS"]
