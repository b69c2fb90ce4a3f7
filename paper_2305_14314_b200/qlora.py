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

import ctypes

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

    def _versions(self):
        return (self.l1._version, self.l2._version)

    def bf16_operands(self):
        """bf16 copies of l1 / l2, zero-padded to a rank multiple of 8.  They
        follow the fp32 masters: any in-place change of l1 / l2 (a torch op, or
        ``AdamOptimizer.step``, which bumps their version counters) refreshes
        them before the next use."""
        rp = _pad8(self.rank)
        key = (self.l1.data_ptr(), self.l2.data_ptr(), rp)
        sh = self._shadow.get("ops")
        if sh is None or sh[0] != key:
            l1b = torch.zeros(self.l1.shape[0], rp, dtype=torch.bfloat16, device=self.l1.device)
            l2b = torch.zeros(rp, self.l2.shape[1], dtype=torch.bfloat16, device=self.l2.device)
            sh = [key, l1b, l2b, None]
            self._shadow["ops"] = sh
        if sh[3] != self._versions():
            self.refresh_bf16()
        return sh[1], sh[2]

    def adopt_shadows(self, l1b: torch.Tensor, l2b: torch.Tensor) -> None:
        """Use caller-owned bf16 copies (kept current by the caller, e.g. the
        fused Adam kernel of the LLaMA harness) as the MMA operands."""
        self._shadow["ops"] = [(self.l1.data_ptr(), self.l2.data_ptr(), _pad8(self.rank)), l1b, l2b,
                               self._versions()]

    def refresh_bf16(self) -> None:
        sh = self._shadow.get("ops")
        if sh is None:
            return
        sh[1][:, : self.rank].copy_(self.l1)
        sh[2][: self.rank].copy_(self.l2)
        sh[3] = self._versions()


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
        self._cat = None
        self._ws = None
        self._wdesc = None
        # a block-constant cache kept current by the caller (a step-level
        # prepass, qlrt_nf4_constants_batch); None: rebuilt every forward
        self.consts_cache: torch.Tensor | None = None

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

    def _rank_total(self) -> int:
        return sum(_pad8(ad.rank) for ad in self.adapters)

    def _workspace(self, m: int) -> torch.Tensor:
        """Scratch of the fused entry points.  Layers share one buffer per
        device (their launches are stream-ordered); it only grows."""
        need = int(lib().qlrt_linear_workspace_bytes(max(m, 1), self.in_dim, self.out_dim, self._rank_total()))
        dev = torch.cuda.current_device()
        ws = _LINEAR_WS.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device="cuda")  # stream-K flags start at 0
            _LINEAR_WS[dev] = ws
        return ws

    def _operands(self):
        """bf16 MMA operands of all adapters: one adapter -> its own copies;
        several -> l1c = [l1_0 | l1_1 | ...] ([in, R]) and l2c = [l2_0; l2_1; ...]
        ([R, out]), each rank zero-padded to a multiple of 8, rebuilt when any
        master changes.  A sum of adapters is one adapter of the summed rank
        once each Ts_i / dT_i carries its own scaling (qlora.py:133-146)."""
        if len(self.adapters) == 1:
            return self.adapters[0].bf16_operands()
        key = tuple((ad.l1.data_ptr(), ad.l2.data_ptr()) + ad._versions() for ad in self.adapters)
        if self._cat is None or self._cat[0] != key:
            R = self._rank_total()
            l1c = torch.zeros(self.in_dim, R, dtype=torch.bfloat16, device=self.adapters[0].l1.device)
            l2c = torch.zeros(R, self.out_dim, dtype=torch.bfloat16, device=self.adapters[0].l1.device)
            o = 0
            for ad in self.adapters:
                l1c[:, o: o + ad.rank].copy_(ad.l1)
                l2c[o: o + ad.rank].copy_(ad.l2)
                o += _pad8(ad.rank)
            self._cat = (key, l1c, l2c)
        return self._cat[1], self._cat[2]

    def _pairs(self, inputs, ts: torch.Tensor, transpose_l2: bool) -> None:
        """Per-adapter s_i * inputs_i @ l1_i (or s_i * dY @ l2_i^T) as bf16 hi/lo
        pairs into ts[:, o_i : o_i + r_i] (hi) and ts[:, R + o_i : ...] (lo)."""
        R = ts.shape[1] // 2
        o = 0
        for ad, inp in zip(self.adapters, inputs):
            rp = _pad8(ad.rank)
            l1b, l2b = ad.bf16_operands()
            v = (gemm_bf16(inp, l2b, alpha=ad.scaling, b_t=True, out_dtype=torch.float32) if transpose_l2
                 else gemm_bf16(inp, l1b, alpha=ad.scaling, out_dtype=torch.float32))
            hi = v.to(torch.bfloat16)
            ts[:, o: o + rp].copy_(hi)
            ts[:, R + o: R + o + rp].copy_((v - hi.float()).to(torch.bfloat16))
            o += rp

    def _masks(self, x2: torch.Tensor, train: bool, rng) -> list:
        """Dropout masks on the adapter inputs, drawn adapter by adapter from
        ``rng`` as the reference does (qlora.py:137-143); None = no dropout."""
        masks = []
        for ad in self.adapters:
            if not (train and ad.dropout_p > 0.0):
                masks.append(None)
                continue
            if rng is None:
                raise ValueError("dropout needs an rng in train mode")
            keep = 1.0 - ad.dropout_p
            if isinstance(rng, torch.Generator):
                draw = torch.rand(x2.shape, generator=rng, device=x2.device)
            else:  # numpy Generator: the reference's exact mask (qlora.py:140-142)
                draw = torch.from_numpy(rng.random(tuple(x2.shape))).to(x2.device)
            masks.append((draw >= ad.dropout_p).to(torch.float32) / keep)
        return masks

    # -- exact-precision path (float32 / float64 layers) ---------------------
    def _exact(self) -> bool:
        return self.dtype in (torch.float32, torch.float64)

    def _forward_exact(self, x, train: bool, rng) -> tuple[torch.Tensor, dict[str, Any]]:
        """The reference's own op order at its precision (qlora.py:117-148): W
        = dequantize(q) (float64, the bit-exact kernel) cast to the layer
        dtype, then cuBLAS GEMMs in that dtype (TF32 off).  The toy layers
        (16 x 16, 2 x 16, ...) are far below any tile of the fused kernels;
        this is the path the GPU ToyModel / train_toy gates run through."""
        if torch.backends.cuda.matmul.allow_tf32:
            raise RuntimeError("exact-precision QLinear needs torch.backends.cuda.matmul.allow_tf32 = False")
        dt = self.dtype
        x = torch.as_tensor(x).to(device="cuda", dtype=dt)
        if isinstance(self.base, BlockQuantized):
            w = dequantize(self.base, torch.float64).to(dt)
        else:
            w = torch.as_tensor(self.base).to(device="cuda", dtype=dt)
        y = x @ w
        branches = []
        for ad in self.adapters:
            xa, mask = x, None
            if train and ad.dropout_p > 0.0:
                if rng is None:
                    raise ValueError("dropout needs an rng in train mode")
                keep = 1.0 - ad.dropout_p
                if isinstance(rng, torch.Generator):
                    draw = torch.rand(x.shape, generator=rng, device=x.device, dtype=torch.float64)
                else:  # numpy Generator: the reference's exact mask (qlora.py:140-142)
                    draw = torch.from_numpy(rng.random(tuple(x.shape))).to(x.device)
                mask = (draw >= ad.dropout_p).to(dt) / keep
                xa = x * mask
            t = xa @ ad.l1.to(dt)
            y = y + ad.scaling * (t @ ad.l2.to(dt))
            branches.append({"xa": xa, "t": t, "mask": mask})
        return y, {"x": x, "w": w, "branches": branches, "exact": True}

    def _backward_exact(self, d_y, cache) -> tuple[torch.Tensor, dict[str, torch.Tensor]]:
        """qlora.py:150-167 at the layer precision."""
        dt = self.dtype
        d_y = torch.as_tensor(d_y).to(device="cuda", dtype=dt)
        d_x = d_y @ cache["w"].T
        grads: dict[str, torch.Tensor] = {}
        for i, (ad, br) in enumerate(zip(self.adapters, cache["branches"])):
            s = ad.scaling
            l1, l2 = ad.l1.to(dt), ad.l2.to(dt)
            d_t = s * (d_y @ l2.T)
            grads[f"adapter{i}.l2"] = s * (br["t"].T @ d_y)
            grads[f"adapter{i}.l1"] = br["xa"].T @ d_t
            d_xa = d_t @ l1.T
            if br["mask"] is not None:
                d_xa = d_xa * br["mask"]
            d_x = d_x + d_xa
        return d_x, grads

    # -- forward / backward -------------------------------------------------
    def forward(self, x, train: bool = False, rng=None) -> tuple[torch.Tensor, dict[str, Any]]:
        """y = x W + sum_i s_i (xa_i l1_i) l2_i (qlora.py:124-148).  One
        adapter without dropout is the fully fused path (Ts and the NF4 GEMM
        with the adapter term in its accumulator, all in the C ABI); several
        adapters or dropout compute the Ts pairs here and still join the same
        accumulator; M = 1 runs the HBM-streaming GEMV.  A float32 / float64
        layer computes at that precision (``_forward_exact``)."""
        if self._exact():
            return self._forward_exact(x, train, rng)
        x = torch.as_tensor(x).to(device="cuda", dtype=self.dtype).contiguous()
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.in_dim)
        m = x2.shape[0]
        masks = self._masks(x2, train, rng)
        xas = [x2 if mk is None else (x2.float() * mk).to(self.dtype).contiguous() for mk in masks]
        y = torch.empty(m, self.out_dim, dtype=self.dtype, device=x2.device)
        n_ad = len(self.adapters)
        R = self._rank_total()
        ts = torch.empty(m, 2 * R, dtype=self.dtype, device=x2.device) if n_ad else None  # bf16 hi | lo
        consts = None
        if self.fused() and m == 1 and n_ad <= 1:
            # the GEMV decodes the DQ constants itself; Ts (needed only by a
            # backward) is left to backward -- inference pays nothing for it
            ad = self.adapters[0] if n_ad else None
            l1b, l2b = self._operands() if n_ad else (None, None)
            check(lib().qlrt_nf4_gemv(self.weight_desc(None), ptr(x2), ptr(xas[0]) if masks and masks[0] is not None
                                      else None, ptr(l1b), ptr(l2b), R, float(ad.scaling) if ad else 0.0, ptr(y),
                                      ptr(self._workspace(m)), stream_ptr()), "QLinear.forward(gemv)")
            ts_ready = False
        elif self.fused():
            # fp32 block constants built once here and shared with backward
            consts = self.consts_cache if self.consts_cache is not None else self._constants()
            l1b, l2b = self._operands() if n_ad else (None, None)
            if n_ad == 1:
                ad = self.adapters[0]
                check(lib().qlrt_nf4_linear_fwd(self.weight_desc(consts), ptr(x2),
                                                ptr(xas[0]) if masks[0] is not None else None, m, ptr(l1b),
                                                ptr(l2b), R, float(ad.scaling), ptr(ts), ptr(y),
                                                ptr(self._workspace(m)), stream_ptr()), "QLinear.forward")
            else:
                if n_ad:
                    self._pairs(xas, ts, False)  # Ts given: l1 = NULL
                check(lib().qlrt_nf4_linear_fwd(self.weight_desc(consts), ptr(x2), None, m, None, ptr(l2b), R, 0.0,
                                                ptr(ts), ptr(y), ptr(self._workspace(m)), stream_ptr()),
                      "QLinear.forward")
            ts_ready = True
        else:
            w = self.dequant_weight().contiguous()
            y32 = gemm_bf16(x2, w, out_dtype=torch.float32)
            if n_ad:
                self._pairs(xas, ts, False)
                o = 0
                for ad in self.adapters:
                    rp = _pad8(ad.rank)
                    _, l2b = ad.bf16_operands()
                    y32 += gemm_bf16(ts[:, o: o + rp], l2b, out_dtype=torch.float32)
                    y32 += gemm_bf16(ts[:, R + o: R + o + rp], l2b, out_dtype=torch.float32)
                    o += rp
            y.copy_(y32.to(self.dtype))
            ts_ready = True
        cache = {"x": x2, "xas": xas, "masks": masks, "ts": ts, "ts_ready": ts_ready, "lead": lead,
                 "consts": consts}
        return y.reshape(*lead, self.out_dim), cache

    def _side_workspace(self, m: int) -> torch.Tensor:
        """Split-K scratch of the deferred adapter-gradient GEMMs (side stream)."""
        need = int(lib().qlrt_linear_workspace_bytes(max(m, 1), self.in_dim, self.out_dim, self._rank_total()))
        dev = torch.cuda.current_device()
        ws = _SIDE_WS.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
            _SIDE_WS[dev] = ws
        return ws

    def backward(self, d_y, cache: dict[str, Any], grads_out: dict | None = None, defer: list | None = None
                 ) -> tuple[torch.Tensor, dict[str, torch.Tensor]]:
        """dX = dY W^T + sum_i (s_i dY l2_i^T) l1_i^T (masked), dl2_i = s_i t_i^T dY,
        dl1_i = xa_i^T (s_i dY l2_i^T) (qlora.py:150-167).  ``grads_out``
        optionally names fp32 buffers ([in, rank], [rank, out], e.g. views of a
        data-parallel gradient bucket) the fused kernels write the adapter
        gradients into directly.

        ``defer`` (a list): on the fused single-adapter path the adapter-gradient
        GEMMs stay on the library's side stream (QLRT_BWD_DEFER) and overlap
        whatever the caller issues next; the tensors they read are appended to
        ``defer``.  The gradients are valid only after :func:`side_join`, and
        the caller keeps the list alive until it has called it."""
        if cache.get("exact"):
            return self._backward_exact(d_y, cache)
        d_y = torch.as_tensor(d_y).to(device="cuda", dtype=self.dtype).reshape(-1, self.out_dim).contiguous()
        m = d_y.shape[0]
        n_ad = len(self.adapters)
        R = self._rank_total()
        dev = d_y.device
        grads: dict[str, torch.Tensor] = {}
        d_x = torch.empty(m, self.in_dim, dtype=self.dtype, device=dev)
        masks, xas, ts = cache["masks"], cache["xas"], cache["ts"]
        if n_ad and not cache["ts_ready"]:
            self._pairs(xas, ts, False)  # the GEMV forward left Ts to backward
            cache["ts_ready"] = True
        any_mask = any(mk is not None for mk in masks)
        wd = self.weight_desc(cache.get("consts")) if self.fused() else None
        ws = self._workspace(m) if self.fused() else None
        if n_ad == 0 or (self.fused() and not any_mask):
            go = grads_out or {}
            single = n_ad == 1
            g1, g2 = go.get("adapter0.l1"), go.get("adapter0.l2")
            direct = (single and R == self.adapters[0].rank and g1 is not None and g2 is not None
                      and g1.is_contiguous() and g2.is_contiguous() and g1.dtype == torch.float32
                      and g2.dtype == torch.float32 and tuple(g1.shape) == (self.in_dim, R)
                      and tuple(g2.shape) == (R, self.out_dim))
            if n_ad == 0:
                if self.fused():
                    check(lib().qlrt_nf4_linear_bwd(wd, ptr(d_y), m, None, None, None, None, 0, 0.0, None, ptr(d_x),
                                                    None, None, ptr(ws), stream_ptr()), "QLinear.backward")
                else:
                    gemm_bf16(d_y, self.dequant_weight().contiguous(), out=d_x, b_t=True)
                return d_x.reshape(*cache["lead"], self.in_dim), grads
            dt = torch.empty(m, 2 * R, dtype=self.dtype, device=dev)  # bf16 hi | lo
            dl1 = g1 if direct else torch.empty(self.in_dim, R, dtype=torch.float32, device=dev)
            dl2 = g2 if direct else torch.empty(R, self.out_dim, dtype=torch.float32, device=dev)
            l1b, l2b = self._operands()
            if single:
                ad = self.adapters[0]
                defer_ok = defer is not None and (direct or not grads_out)
                check(lib().qlrt_nf4_linear_bwd_ex(wd, ptr(d_y), m, ptr(xas[0]), ptr(ts), ptr(l1b), ptr(l2b), R,
                                                   float(ad.scaling), ptr(dt), ptr(d_x), ptr(dl1), ptr(dl2), ptr(ws),
                                                   ptr(self._side_workspace(m)) if defer_ok else None,
                                                   _native.QLRT_BWD_DEFER if defer_ok else 0, stream_ptr()),
                      "QLinear.backward")
                if defer_ok:
                    defer.extend((d_y, xas[0], ts, dt, dl1, dl2))
            else:
                self._pairs([d_y] * n_ad, dt, True)  # dT given: l2 = NULL
                check(lib().qlrt_nf4_linear_bwd(wd, ptr(d_y), m, ptr(cache["x"]), ptr(ts), ptr(l1b), None, R, 0.0,
                                                ptr(dt), ptr(d_x), ptr(dl1), ptr(dl2), ptr(ws), stream_ptr()),
                      "QLinear.backward")
            o = 0
            for i, ad in enumerate(self.adapters):
                grads[f"adapter{i}.l1"] = dl1[:, o: o + ad.rank]
                grads[f"adapter{i}.l2"] = dl2[o: o + ad.rank]
                o += _pad8(ad.rank)
        else:
            # dropout (or a base the fused kernels do not take): the base product
            # through the engine, the masked adapter terms added in fp32
            if self.fused():
                check(lib().qlrt_nf4_linear_bwd(wd, ptr(d_y), m, None, None, None, None, 0, 0.0, None, ptr(d_x),
                                                None, None, ptr(ws), stream_ptr()), "QLinear.backward")
                dx32 = d_x.float()
            else:
                dx32 = gemm_bf16(d_y, self.dequant_weight().contiguous(), b_t=True, out_dtype=torch.float32)
            dt = torch.empty(m, 2 * R, dtype=self.dtype, device=dev)
            self._pairs([d_y] * n_ad, dt, True)
            o = 0
            for i, (ad, mk, xa) in enumerate(zip(self.adapters, masks, xas)):
                rp = _pad8(ad.rank)
                l1b, _ = ad.bf16_operands()
                hi, lo = dt[:, o: o + rp], dt[:, R + o: R + o + rp]
                d_xa = (gemm_bf16(hi, l1b, b_t=True, out_dtype=torch.float32)
                        + gemm_bf16(lo, l1b, b_t=True, out_dtype=torch.float32))
                dx32 += d_xa if mk is None else d_xa * mk
                t_hi, t_lo = ts[:, o: o + rp], ts[:, R + o: R + o + rp]
                grads[f"adapter{i}.l2"] = (gemm_bf16(t_hi, d_y, a_t=True, out_dtype=torch.float32)
                                           + gemm_bf16(t_lo, d_y, a_t=True, out_dtype=torch.float32))[: ad.rank]
                grads[f"adapter{i}.l1"] = (gemm_bf16(xa, hi, a_t=True, out_dtype=torch.float32)
                                           + gemm_bf16(xa, lo, a_t=True, out_dtype=torch.float32))[:, : ad.rank]
                o += rp
            d_x.copy_(dx32.to(self.dtype))
        if grads_out:
            for k, v in list(grads.items()):
                tgt = grads_out.get(k)
                if tgt is not None and tgt.data_ptr() != v.data_ptr():
                    tgt.copy_(v)
                    grads[k] = tgt
        return d_x.reshape(*cache["lead"], self.in_dim), grads

    def trainable(self) -> dict[str, torch.Tensor]:
        out = {}
        for i, ad in enumerate(self.adapters):
            out[f"adapter{i}.l1"] = ad.l1
            out[f"adapter{i}.l2"] = ad.l2
        return out


class QLinearGroup:
    """Sibling projections that read the same input (q | k | v, gate | up) as
    ONE call of the fused kernels -- the same math per member as a QLinear
    with one adapter (qlora.py:124-167).

    Every member keeps its own NF4 + DQ quantization (the reference's
    per-layer QLinear; its DQ codes / c1 / mu stay per member); the packed
    codes are concatenated along N into one buffer so one fused grid covers
    all members (``release_member_codes`` drops the members' own copies).  ``l1`` [K][G r] and ``l2``
    [r][G N_g] are fp32 masters (member g's adapter = column slice g), ``l1b``
    / ``l2b`` their bf16 operand copies (kept current by the caller's fused
    Adam, as the LLaMA harness does, or refreshed here on a version change).
    """

    def __init__(self, bases: list, l1: torch.Tensor, l2: torch.Tensor, rank: int, alpha: float,
                 l1b: torch.Tensor | None = None, l2b: torch.Tensor | None = None,
                 release_member_codes: bool = False):
        g = len(bases)
        k, ng = int(bases[0].shape[0]), int(bases[0].shape[1])
        for b in bases:
            if not (isinstance(b, BlockQuantized) and b.dq is not None and b.blocksize == 64
                    and b.codebook.bits == 4 and tuple(b.shape) == (k, ng)):
                raise ValueError("group members must be NF4 + DQ, blocksize 64, of one shape")
        if ng % 256 or rank % 64:
            raise ValueError(f"grouped projections need N_g % 256 == 0 and rank % 64 == 0 (got {ng}, {rank})")
        if tuple(l1.shape) != (k, g * rank) or tuple(l2.shape) != (rank, g * ng):
            raise ValueError("l1 must be [K][G r] and l2 [r][G N_g]")
        self.groups, self.in_dim, self.n_member, self.rank, self.alpha = g, k, ng, rank, alpha
        self.out_dim = g * ng
        self.l1, self.l2 = l1, l2
        self.codes = torch.empty(k, self.out_dim // 2, dtype=torch.uint8, device=l1.device)
        for i, b in enumerate(bases):
            self.codes[:, i * ng // 2: (i + 1) * ng // 2].copy_(b.codes.view(k, ng // 2))
            if release_member_codes:  # (the concatenated buffer stays the only copy)
                b.codes = None
        self.bases = bases
        self._ops = [l1b, l2b, None] if l1b is not None else None
        self._wdesc = None
        self.consts_cache: torch.Tensor | None = None  # (as QLinear.consts_cache)
        self._member_desc = (_native.NF4Weight * g)()
        for i, b in enumerate(bases):
            d = self._member_desc[i]
            d.dq_codes, d.c1, d.mu = ptr(b.dq.codes), ptr(b.dq.c1), ptr(b.dq.mu)
            d.k_in, d.n_out, d.blocksize2 = k, ng, b.dq.blocksize2
            d.spec = b.dq.spec.to_c()

    @property
    def scaling(self) -> float:
        return self.alpha / self.rank

    def operands(self):
        """bf16 copies of l1 / l2 (caller-owned ones are used as they are)."""
        if self._ops is None or (self._ops[2] is not None and self._ops[2] != (self.l1._version, self.l2._version)):
            if self._ops is None:
                self._ops = [torch.empty_like(self.l1, dtype=torch.bfloat16),
                             torch.empty_like(self.l2, dtype=torch.bfloat16), None]
            self._ops[0].copy_(self.l1)
            self._ops[1].copy_(self.l2)
            self._ops[2] = (self.l1._version, self.l2._version)
        return self._ops[0], self._ops[1]

    def _desc(self, consts: torch.Tensor):
        if self._wdesc is None:
            b = self.bases[0]
            w = _native.NF4Weight()
            w.codes, w.dq_codes, w.c1, w.mu = ptr(self.codes), ptr(b.dq.codes), ptr(b.dq.c1), ptr(b.dq.mu)
            w.k_in, w.n_out, w.blocksize2 = self.in_dim, self.out_dim, b.dq.blocksize2
            w.spec = b.dq.spec.to_c()
            for i in range(16):
                w.values[i] = float(b.codebook.values[i])
            self._wdesc = w
        self._wdesc.consts = ptr(consts)
        return self._wdesc

    def _constants(self) -> torch.Tensor:
        """The members' block constants into one [K][round4(N/64)] cache (per
        forward, shared with the backward; padding columns stay zero)."""
        L = lib()
        pitch = int(L.qlrt_nf4_constants_bytes(self.in_dim, self.out_dim)) // 4 // self.in_dim
        nbr = self.n_member // 64
        alloc = torch.empty if pitch == self.groups * nbr else torch.zeros  # (padding columns must read 0)
        out = alloc(self.in_dim, pitch, dtype=torch.float32, device=self.l1.device)
        if self.groups <= 4:
            check(L.qlrt_nf4_constants_group(self._member_desc, self.groups, ptr(out), pitch, stream_ptr()),
                  "QLinearGroup constants")
        else:
            for i in range(self.groups):
                check(L.qlrt_nf4_constants_into(ctypes.byref(self._member_desc[i]), ptr(out) + 4 * i * nbr, pitch,
                                                stream_ptr()), "QLinearGroup constants")
        return out

    def _workspace(self, m: int, side: bool = False) -> torch.Tensor:
        need = int(lib().qlrt_linear_workspace_bytes(max(m, 1), self.in_dim, self.out_dim, self.groups * self.rank))
        table = _SIDE_WS if side else _LINEAR_WS
        dev = torch.cuda.current_device()
        ws = table.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
            table[dev] = ws
        return ws

    def forward(self, x: torch.Tensor):
        """Y_cat [M][G N_g] = X W_cat + per member s (X l1_g) l2_g."""
        x2 = x.reshape(-1, self.in_dim)
        if x2.dtype != torch.bfloat16 or not x2.is_contiguous():
            x2 = x2.to(torch.bfloat16).contiguous()
        m = x2.shape[0]
        consts = self.consts_cache if self.consts_cache is not None else self._constants()
        l1b, l2b = self.operands()
        ts = torch.empty(m, 2 * self.groups * self.rank, dtype=torch.bfloat16, device=x2.device)
        y = torch.empty(m, self.out_dim, dtype=torch.bfloat16, device=x2.device)
        check(lib().qlrt_nf4_linear_group_fwd(self._desc(consts), self.groups, ptr(x2), m, ptr(l1b), ptr(l2b),
                                              self.rank, float(self.scaling), ptr(ts), ptr(y),
                                              ptr(self._workspace(m)), stream_ptr()), "QLinearGroup.forward")
        return y, {"x": x2, "ts": ts, "consts": consts}

    def backward(self, d_y: torch.Tensor, cache: dict, dl1: torch.Tensor, dl2: torch.Tensor,
                 defer: list | None = None) -> torch.Tensor:
        """dX = sum_g (dY_g W_g^T + s dY_g l2_g^T l1_g^T); dl1 [K][G r] and dl2
        [r][G N_g] (fp32, contiguous) receive every member's adapter
        gradients.  ``defer``: as QLinear.backward."""
        d_y = d_y.reshape(-1, self.out_dim)
        if d_y.dtype != torch.bfloat16 or not d_y.is_contiguous():
            d_y = d_y.to(torch.bfloat16).contiguous()
        m = d_y.shape[0]
        if not (dl1.is_contiguous() and dl2.is_contiguous() and dl1.dtype == torch.float32
                and dl2.dtype == torch.float32):
            raise ValueError("dl1 / dl2 must be contiguous float32")
        l1b, l2b = self.operands()
        dt = torch.empty(m, 2 * self.groups * self.rank, dtype=torch.bfloat16, device=d_y.device)
        d_x = torch.empty(m, self.in_dim, dtype=torch.bfloat16, device=d_y.device)
        check(lib().qlrt_nf4_linear_group_bwd(self._desc(cache["consts"]), self.groups, ptr(d_y), m, ptr(cache["x"]),
                                              ptr(cache["ts"]), ptr(l1b), ptr(l2b), self.rank, float(self.scaling),
                                              ptr(dt), ptr(d_x), ptr(dl1), ptr(dl2), ptr(self._workspace(m)),
                                              ptr(self._workspace(m, side=True)) if defer is not None else None,
                                              _native.QLRT_BWD_DEFER if defer is not None else 0, stream_ptr()),
              "QLinearGroup.backward")
        if defer is not None:
            defer.extend((d_y, cache["x"], cache["ts"], dt, dl1, dl2))
        return d_x


_GEMM_WS: dict = {}
_SIDE_WS: dict = {}


def side_join(stream: torch.cuda.Stream | None = None) -> None:
    """The (current) stream waits for the adapter-gradient GEMMs deferred by
    ``QLinear.backward(defer=...)`` on it (qlrt_side_join)."""
    check(lib().qlrt_side_join(stream_ptr() if stream is None else stream.cuda_stream), "side_join")


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


__all__ = ["LoraAdapter", "lora_init", "QLinear", "QLinearGroup", "PLACEMENTS", "gemm_bf16", "side_join"]
