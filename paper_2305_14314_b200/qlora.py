"""Frozen NF4 linear layer with a LoRA adapter on the B200 kernels -- mirror of
``qlrt.qlora`` (pkg/src/qlrt/qlora.py:48-167).

    Y   = X W + s (Xa L1) L2                     s = alpha / rank
    dX  = dY W^T + (s dY L2^T) L1^T (masked)     dL2 = s (Xa L1)^T dY
    dL1 = Xa^T (s dY L2^T)

Same names and semantics as the reference: ``forward(x, train, rng) ->
(y, cache)`` and ``backward(d_y, cache) -> (d_x, {"adapter0.l1", "adapter0.l2"})``,
no gradient for the frozen base, the base is re-dequantized on every use and
never cached on the layer.  On the GPU "re-dequantized" means: the packed
NF4 tiles are decoded inside the tcgen05 GEMM (``qlrt_nf4_linear_fwd/bwd``);
W is never materialized in HBM.

Compute precision is bf16 operands with fp32 accumulation (the reference's
"low" float32 mode is the closest host analogue); the adapter's trainable
master copies are float32, mirrored to bf16 for the MMAs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

from . import _native
from ._native import check, lib, ptr, stream_ptr
from .blockquant import BlockQuantized, dequantize

PLACEMENTS = ("all_linear", "qv_only", "none")
_LINEAR_WS: dict = {}


def _pad8(r: int) -> int:
    return (r + 7) // 8 * 8


@dataclass
class LoraAdapter:
    """Trainable low-rank delta s * (X l1) l2 (qlora.py:48-60); fp32 device masters."""

    rank: int
    alpha: float
    l1: torch.Tensor  # (in_dim, rank) float32
    l2: torch.Tensor  # (rank, out_dim) float32
    dropout_p: float = 0.0
    _shadow: dict = field(default_factory=dict, repr=False)

    @property
    def scaling(self) -> float:
        return self.alpha / self.rank

    def bf16_operands(self):
        """bf16 copies of l1 / l2, zero-padded to a rank multiple of 8 (the
        optimizer refreshes them in place after every step)."""
        rp = _pad8(self.rank)
        key = (self.l1.data_ptr(), self.l2.data_ptr(), rp)
        sh = self._shadow.get("ops")
        if sh is None or sh[0] != key:
            l1b = torch.zeros(self.l1.shape[0], rp, dtype=torch.bfloat16, device=self.l1.device)
            l2b = torch.zeros(rp, self.l2.shape[1], dtype=torch.bfloat16, device=self.l2.device)
            sh = (key, l1b, l2b)
            self._shadow["ops"] = sh
            self.refresh_bf16()
        return sh[1], sh[2]

    def refresh_bf16(self) -> None:
        sh = self._shadow.get("ops")
        if sh is None:
            return
        sh[1][:, : self.rank].copy_(self.l1)
        sh[2][: self.rank].copy_(self.l2)


def lora_init(in_dim: int, out_dim: int, rank: int, alpha: float, rng: np.random.Generator,
              dropout_p: float = 0.0, dtype=torch.float32, device="cuda") -> LoraAdapter:
    """l1 ~ N(0, 1/rank), l2 = 0 (qlora.py:63-80); the same numpy draws as the
    reference, so a seed names the same adapter."""
    if rank < 1:
        raise ValueError(f"rank must be >= 1, got {rank}")
    if not 0.0 <= dropout_p < 1.0:
        raise ValueError(f"dropout_p must lie in [0, 1), got {dropout_p}")
    l1 = (rng.standard_normal((in_dim, rank)) / np.sqrt(rank)).astype(np.float32)
    return LoraAdapter(rank=rank, alpha=alpha, l1=torch.from_numpy(l1).to(device=device, dtype=dtype),
                       l2=torch.zeros(rank, out_dim, dtype=dtype, device=device), dropout_p=dropout_p)


class QLinear:
    """Frozen base (NF4 ``BlockQuantized`` or a dense tensor) plus trainable adapters."""

    def __init__(self, base, adapters: list[LoraAdapter] | None = None, dtype=torch.bfloat16):
        if len(base.shape) != 2:
            raise ValueError(f"base weight must be 2-d, got shape {tuple(base.shape)}")
        self.base = base
        self.adapters = adapters if adapters is not None else []
        self.dtype = dtype
        for ad in self.adapters:
            if ad.l1.shape[0] != base.shape[0] or ad.l2.shape[1] != base.shape[1]:
                raise ValueError(f"adapter ({tuple(ad.l1.shape)} x {tuple(ad.l2.shape)}) does not match "
                                 f"base shape {tuple(base.shape)}")
        if len(self.adapters) > 1:
            raise ValueError("the fused GPU layer carries at most one adapter per layer")
        self._ws = None
        self._wdesc = None

    @property
    def in_dim(self) -> int:
        return int(self.base.shape[0])

    @property
    def out_dim(self) -> int:
        return int(self.base.shape[1])

    # -- base access -------------------------------------------------------
    def fused(self) -> bool:
        b = self.base
        return (isinstance(b, BlockQuantized) and b.dq is not None and b.blocksize == 64
                and b.codebook.bits == 4 and self.out_dim % 64 == 0 and self.in_dim % 8 == 0)

    def weight_desc(self, consts: torch.Tensor | None = None) -> _native.NF4Weight:
        """C descriptor of the base; ``consts`` = the per-forward fp32
        block-constant cache shared with the matching backward."""
        if self._wdesc is None:
            b = self.base
            w = _native.NF4Weight()
            w.codes, w.dq_codes, w.c1, w.mu = ptr(b.codes), ptr(b.dq.codes), ptr(b.dq.c1), ptr(b.dq.mu)
            w.k_in, w.n_out, w.blocksize2 = self.in_dim, self.out_dim, b.dq.blocksize2
            w.spec = b.dq.spec.to_c()
            for i in range(16):
                w.values[i] = float(b.codebook.values[i])
            self._wdesc = w
        self._wdesc.consts = ptr(consts)
        return self._wdesc

    def _constants(self) -> torch.Tensor:
        """Double-dequantize the block constants once per forward (kept in the
        cache for backward, like the reference keeps cache['w'])."""
        L = lib()
        out = torch.empty(int(L.qlrt_nf4_constants_bytes(self.in_dim, self.out_dim)) // 4, dtype=torch.float32,
                          device="cuda")
        check(L.qlrt_nf4_constants(self.weight_desc(None), ptr(out), stream_ptr()), "QLinear constants")
        return out

    def dequant_weight(self) -> torch.Tensor:
        """Base weight at compute precision (qlora.py:117-122); only the
        non-fused shapes use it -- the fused kernels never materialize W."""
        if isinstance(self.base, BlockQuantized):
            return dequantize(self.base, torch.float32).to(self.dtype)
        return torch.as_tensor(self.base).to(device="cuda", dtype=self.dtype)

    def _workspace(self, m: int) -> torch.Tensor:
        """Scratch of the fused entry points.  Layers share one buffer per
        device (their launches are stream-ordered); it only grows."""
        r = _pad8(self.adapters[0].rank) if self.adapters else 0
        need = int(lib().qlrt_linear_workspace_bytes(max(m, 1), self.in_dim, self.out_dim, r))
        dev = torch.cuda.current_device()
        ws = _LINEAR_WS.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device="cuda")  # stream-K flags start at 0
            _LINEAR_WS[dev] = ws
        return ws

    # -- forward / backward -------------------------------------------------
    def forward(self, x, train: bool = False, rng=None) -> tuple[torch.Tensor, dict[str, Any]]:
        x = torch.as_tensor(x).to(device="cuda", dtype=self.dtype).contiguous()
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.in_dim)
        m = x2.shape[0]
        ad = self.adapters[0] if self.adapters else None
        mask = None
        xa = x2
        if ad is not None and train and ad.dropout_p > 0.0:
            if rng is None:
                raise ValueError("dropout needs an rng in train mode")
            keep = 1.0 - ad.dropout_p
            if isinstance(rng, torch.Generator):
                draw = torch.rand(x2.shape, generator=rng, device=x2.device)
            else:  # numpy Generator: the reference's exact mask (qlora.py:140-142)
                draw = torch.from_numpy(rng.random(tuple(x2.shape))).to(x2.device)
            mask = ((draw >= ad.dropout_p).to(torch.float32) / keep)
            xa = (x2.float() * mask).to(self.dtype).contiguous()
        y = torch.empty(m, self.out_dim, dtype=self.dtype, device=x2.device)
        rp = _pad8(ad.rank) if ad else 0
        ts = torch.empty(m, 2 * rp, dtype=self.dtype, device=x2.device) if ad else None  # bf16 hi | lo
        # the GEMV decodes the DQ constants itself; at m > 1 the fp32 constants are
        # built once here and shared with backward (None -> backward rebuilds them)
        consts = self._constants() if self.fused() and m > 1 else None
        if self.fused() and m > 1:
            l1b, l2b = ad.bf16_operands() if ad else (None, None)
            check(lib().qlrt_nf4_linear_fwd(self.weight_desc(consts), ptr(x2), ptr(xa) if mask is not None else None, m,
                                            ptr(l1b), ptr(l2b), rp, float(ad.scaling) if ad else 0.0, ptr(ts),
                                            ptr(y), ptr(self._workspace(m)), stream_ptr()), "QLinear.forward")
        elif self.fused() and m == 1:
            l1b, l2b = ad.bf16_operands() if ad else (None, None)
            if ad is not None:
                _split_into(gemm_bf16(xa, l1b, alpha=ad.scaling, out_dtype=torch.float32), ts)
            check(lib().qlrt_nf4_gemv(self.weight_desc(None), ptr(x2), ptr(l1b), ptr(l2b), rp,
                                      float(ad.scaling) if ad else 0.0, ptr(y), ptr(self._workspace(m)),
                                      stream_ptr()), "QLinear.forward(gemv)")
        else:
            w = self.dequant_weight().contiguous()
            gemm_bf16(x2, w, out=y)
            if ad is not None:
                l1b, l2b = ad.bf16_operands()
                _split_into(gemm_bf16(xa, l1b, alpha=ad.scaling, out_dtype=torch.float32), ts)
                y.copy_((y.float() + gemm_bf16(ts[:, :rp], l2b, out_dtype=torch.float32)
                         + gemm_bf16(ts[:, rp:], l2b, out_dtype=torch.float32)).to(self.dtype))
        cache = {"x": x2, "xa": xa, "ts": ts, "mask": mask, "lead": lead, "consts": consts}
        return y.reshape(*lead, self.out_dim), cache

    def backward(self, d_y, cache: dict[str, Any], grads_out: dict | None = None
                 ) -> tuple[torch.Tensor, dict[str, torch.Tensor]]:
        """``grads_out`` optionally names fp32 buffers ([in, rank], [rank, out],
        e.g. views of a data-parallel gradient bucket) the fused kernels write
        the adapter gradients into directly."""
        d_y = torch.as_tensor(d_y).to(device="cuda", dtype=self.dtype).reshape(-1, self.out_dim).contiguous()
        m = d_y.shape[0]
        ad = self.adapters[0] if self.adapters else None
        grads: dict[str, torch.Tensor] = {}
        d_x = torch.empty(m, self.in_dim, dtype=self.dtype, device=d_y.device)
        mask = cache["mask"]
        if ad is not None:
            rp = _pad8(ad.rank)
            l1b, l2b = ad.bf16_operands()
            dt = torch.empty(m, 2 * rp, dtype=self.dtype, device=d_y.device)  # bf16 hi | lo
            go = grads_out or {}
            g1, g2 = go.get("adapter0.l1"), go.get("adapter0.l2")
            direct = (rp == ad.rank and g1 is not None and g2 is not None and g1.is_contiguous()
                      and g2.is_contiguous() and g1.dtype == torch.float32 and g2.dtype == torch.float32
                      and tuple(g1.shape) == (self.in_dim, rp) and tuple(g2.shape) == (rp, self.out_dim))
            dl1 = g1 if direct else torch.empty(self.in_dim, rp, dtype=torch.float32, device=d_y.device)
            dl2 = g2 if direct else torch.empty(rp, self.out_dim, dtype=torch.float32, device=d_y.device)
        if self.fused() and mask is None:
            if ad is None:
                check(lib().qlrt_nf4_linear_bwd(self.weight_desc(cache.get("consts")), ptr(d_y), m, None, None, None, None, 0, 0.0,
                                                None, ptr(d_x), None, None, ptr(self._workspace(m)), stream_ptr()),
                      "QLinear.backward")
            else:
                check(lib().qlrt_nf4_linear_bwd(self.weight_desc(cache.get("consts")), ptr(d_y), m, ptr(cache["xa"]), ptr(cache["ts"]),
                                                ptr(l1b), ptr(l2b), rp, float(ad.scaling), ptr(dt), ptr(d_x),
                                                ptr(dl1), ptr(dl2), ptr(self._workspace(m)), stream_ptr()),
                      "QLinear.backward")
        else:
            if self.fused():
                check(lib().qlrt_nf4_linear_bwd(self.weight_desc(cache.get("consts")), ptr(d_y), m, None, None, None, None, 0, 0.0,
                                                None, ptr(d_x), None, None, ptr(self._workspace(m)), stream_ptr()),
                      "QLinear.backward")
            else:
                w = self.dequant_weight().contiguous()
                gemm_bf16(d_y, w, out=d_x, b_t=True)
            if ad is not None:
                _split_into(gemm_bf16(d_y, l2b, alpha=ad.scaling, b_t=True, out_dtype=torch.float32), dt)
                d_xa = (gemm_bf16(dt[:, :rp], l1b, b_t=True, out_dtype=torch.float32)
                        + gemm_bf16(dt[:, rp:], l1b, b_t=True, out_dtype=torch.float32))
                if mask is not None:
                    d_xa = d_xa * mask
                d_x.copy_((d_x.float() + d_xa).to(self.dtype))
                ts = cache["ts"]
                dl2.copy_(gemm_bf16(ts[:, :rp], d_y, a_t=True, out_dtype=torch.float32)
                          + gemm_bf16(ts[:, rp:], d_y, a_t=True, out_dtype=torch.float32))
                dl1.copy_(gemm_bf16(cache["xa"], dt[:, :rp], a_t=True, out_dtype=torch.float32)
                          + gemm_bf16(cache["xa"], dt[:, rp:], a_t=True, out_dtype=torch.float32))
        if ad is not None:
            grads["adapter0.l1"] = dl1[:, : ad.rank]
            grads["adapter0.l2"] = dl2[: ad.rank]
            if grads_out and not direct:
                for k in ("adapter0.l1", "adapter0.l2"):
                    if grads_out.get(k) is not None:
                        grads_out[k].copy_(grads[k])
                        grads[k] = grads_out[k]
        return d_x.reshape(*cache["lead"], self.in_dim), grads

    def trainable(self) -> dict[str, torch.Tensor]:
        out = {}
        for i, ad in enumerate(self.adapters):
            out[f"adapter{i}.l1"] = ad.l1
            out[f"adapter{i}.l2"] = ad.l2
        return out


def _split_into(v: torch.Tensor, pair: torch.Tensor) -> None:
    """fp32 [m, r] -> bf16 hi/lo pair stored as pair[:, :r] | pair[:, r:]."""
    r = v.shape[1]
    hi = v.to(torch.bfloat16)
    pair[:, :r].copy_(hi)
    pair[:, r:].copy_((v - hi.float()).to(torch.bfloat16))


_GEMM_WS: dict = {}


def _pad2(t: torch.Tensor, r: int, c: int) -> torch.Tensor:
    if t.shape[0] == r and t.shape[1] == c:
        return t
    out = torch.zeros(r, c, dtype=t.dtype, device=t.device)
    out[: t.shape[0], : t.shape[1]] = t
    return out


def gemm_bf16(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, alpha: float = 1.0,
              a_t: bool = False, b_t: bool = False, out_dtype=None) -> torch.Tensor:
    """out = alpha * op(a) @ op(b) on the tcgen05 engine (fp32 accumulate).

    ``a`` is [M, K] (or [K, M] with ``a_t``), ``b`` is [K, N] (or [N, K] with
    ``b_t``); operands are bf16.  Row pitches must be 16-byte multiples for
    TMA: unaligned extents are zero-padded (exact) and the result sliced.
    """
    a = a.to(torch.bfloat16).contiguous()
    b = b.to(torch.bfloat16).contiguous()
    m, k = (a.shape[1], a.shape[0]) if a_t else (a.shape[0], a.shape[1])
    n = b.shape[0] if b_t else b.shape[1]
    if out is None:
        out = torch.empty(m, n, dtype=out_dtype or torch.bfloat16, device=a.device)
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("gemm_bf16 writes bf16 or fp32")
    r8 = lambda v: (v + 7) // 8 * 8  # noqa: E731
    mp, kp, np_ = r8(m), r8(k), r8(n)
    if (mp, kp, np_) != (m, k, n) or not out.is_contiguous():
        a = _pad2(a, kp, mp) if a_t else _pad2(a, mp, kp)
        b = _pad2(b, np_, kp) if b_t else _pad2(b, kp, np_)
        tmp = gemm_bf16(a, b, alpha=alpha, a_t=a_t, b_t=b_t, out_dtype=out.dtype)
        out.copy_(tmp[:m, :n])
        return out
    dev = a.device
    ws = _GEMM_WS.get(dev)
    need = 16 * m * n * 4 + 4096 + (20 << 20)  # split-K partials + the stream-K region
    if ws is None or ws.numel() < need:
        ws = torch.zeros(need, dtype=torch.uint8, device=dev)  # stream-K flags start at 0
        _GEMM_WS[dev] = ws
    # a_mn: A stored [K][M]; b_mn: B stored [K][N]
    check(lib().qlrt_gemm_bf16(ptr(a), ptr(b), ptr(out), m, n, k, int(a_t), int(not b_t), float(alpha),
                               int(out.dtype == torch.float32), 0, ptr(ws), ws.numel(), stream_ptr()), "gemm_bf16")
    return out


__all__ = ["LoraAdapter", "lora_init", "QLinear", "PLACEMENTS", "gemm_bf16"]
