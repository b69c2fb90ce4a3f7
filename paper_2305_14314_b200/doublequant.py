"""Double quantization on the GPU -- mirror of ``qlrt.doublequant``
(pkg/src/qlrt/doublequant.py:33-223).

Tensors live on the CUDA device; ``mu`` is a 1-element float32 device tensor
(kept on the device so dequantization never syncs).  Codes, ``c1`` and
``mu`` are bit-exact with the reference: the mean follows numpy 2.3's
buffered pairwise summation order, the 8-bit float encoder is the
reference's nearest-with-ties-away-from-zero on the E4M3/bias-7/no-NaN grid
(max 480), not the hardware e4m3 converter.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import check, lib, ptr, stream_ptr


@dataclass(frozen=True)
class Fp8Spec:
    """Sign/exponent/mantissa layout of the 8-bit constant quantizer (doublequant.py:33-77)."""

    exp_bits: int = 4
    mant_bits: int = 3
    bias: int = 7

    def __post_init__(self) -> None:
        if self.exp_bits + self.mant_bits != 7:
            raise ValueError("exp_bits + mant_bits must equal 7 (one sign bit)")
        if self.exp_bits < 1 or self.bias < 0:
            raise ValueError("need at least one exponent bit and bias >= 0")

    @property
    def max_value(self) -> float:
        return (2.0 - 2.0 ** -self.mant_bits) * 2.0 ** (2 ** self.exp_bits - 1 - self.bias)

    def to_c(self) -> _native.Fp8SpecC:
        return _native.Fp8SpecC(self.exp_bits, self.mant_bits, self.bias)

    def grid(self):
        """(sorted distinct values, canonical byte codes) -- host-side, like the reference."""
        table = decode_table_host(self)
        order = np.argsort(table, kind="stable")
        vals, codes = table[order], np.arange(256, dtype=np.uint8)[order]
        keep = np.concatenate([[True], vals[1:] != vals[:-1]])
        return vals[keep], codes[keep]


def decode_table_host(spec: Fp8Spec) -> np.ndarray:
    out = np.empty(256)
    for b in range(256):
        e = (b >> spec.mant_bits) & (2 ** spec.exp_bits - 1)
        m = b & (2 ** spec.mant_bits - 1)
        mag = m * 2.0 ** (1 - spec.bias - spec.mant_bits) if e == 0 else \
            (2 ** spec.mant_bits + m) * 2.0 ** (e - spec.bias - spec.mant_bits)
        out[b] = -mag if b >> 7 else mag
    return out


@dataclass
class DQConstants:
    """Compressed first-level constants (doublequant.py:129-145)."""

    mu: torch.Tensor         # float32 [1], device
    blocksize2: int
    spec: Fp8Spec
    c1: torch.Tensor         # float32 [ceil(n / blocksize2)], device
    codes: torch.Tensor      # uint8 [n], device

    @property
    def n_constants(self) -> int:
        return int(self.codes.numel())


def _cuda(t, dtype=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.from_numpy(np.ascontiguousarray(t))
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.cuda().contiguous()


def encode_fp8(x, spec: Fp8Spec | None = None) -> torch.Tensor:
    """Nearest 8-bit float code, ties away from zero, clamped (doublequant.py:103-113)."""
    spec = spec or Fp8Spec()
    x = _cuda(x, torch.float64)
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    if x.numel():
        check(lib().qlrt_fp8_encode(ptr(x), x.numel(), spec.to_c(), ptr(out), stream_ptr()), "encode_fp8")
    return out


def decode_fp8(codes, spec: Fp8Spec | None = None) -> torch.Tensor:
    """Byte codes -> float64 grid values, total over all 256 patterns (doublequant.py:116-121)."""
    spec = spec or Fp8Spec()
    c = _cuda(codes, torch.uint8)
    out = torch.empty(c.shape, dtype=torch.float64, device=c.device)
    if c.numel():
        check(lib().qlrt_fp8_decode(ptr(c), c.numel(), spec.to_c(), ptr(out), stream_ptr()), "decode_fp8")
    return out


def dq_compress(constants, blocksize2: int = 256, spec: Fp8Spec | None = None) -> DQConstants:
    """Mean-centre and block-quantize the constants (doublequant.py:148-187)."""
    spec = spec or Fp8Spec()
    c = _cuda(constants, torch.float32)
    if c.dim() != 1 or c.numel() == 0:
        raise ValueError("constants must be a non-empty 1-d array")
    if blocksize2 < 1:
        raise ValueError(f"blocksize2 must be >= 1, got {blocksize2}")
    if bool((c < 0).any()) or not bool(torch.isfinite(c).all()):
        raise ValueError("constants must be finite and nonnegative")
    return _dq_compress_unchecked(c, blocksize2, spec)


def _dq_compress_unchecked(c: torch.Tensor, blocksize2: int, spec: Fp8Spec) -> DQConstants:
    L = lib()
    nb = c.numel()
    n2 = -(-nb // blocksize2)
    ws = torch.empty(max(1, int(L.qlrt_dq_workspace_bytes(nb))), dtype=torch.uint8, device=c.device)
    mu = torch.empty(1, dtype=torch.float32, device=c.device)
    c1 = torch.empty(n2, dtype=torch.float32, device=c.device)
    codes = torch.empty(nb, dtype=torch.uint8, device=c.device)
    check(L.qlrt_dq_compress(ptr(c), nb, blocksize2, spec.to_c(), ptr(ws), ptr(mu), ptr(c1), ptr(codes),
                             stream_ptr()), "dq_compress")
    return DQConstants(mu=mu, blocksize2=blocksize2, spec=spec, c1=c1, codes=codes)


def dq_decompress(dq: DQConstants) -> torch.Tensor:
    """max(decode(code) * c1 + mu, 0) in two fp64 roundings -> float32 (doublequant.py:190-195)."""
    out = torch.empty(dq.n_constants, dtype=torch.float32, device=dq.codes.device)
    check(lib().qlrt_dq_decompress(ptr(dq.codes), ptr(dq.c1), ptr(dq.mu), dq.n_constants, dq.blocksize2,
                                   dq.spec.to_c(), ptr(out), stream_ptr()), "dq_decompress")
    return out


def bits_per_param(k: int, blocksize: int, dq: tuple[int, int] | None = None) -> float:
    """Storage accounting (doublequant.py:203-223): 4.126953125 for NF4/64/DQ(256, 8)."""
    if k < 1 or blocksize < 1:
        raise ValueError("k and blocksize must be positive")
    if dq is None:
        return k + 32.0 / blocksize
    b2, bits2 = dq
    if b2 < 1 or bits2 < 1:
        raise ValueError("blocksize2 and bits2 must be positive")
    return k + bits2 / blocksize + 32.0 / (blocksize * b2)


__all__ = ["Fp8Spec", "DQConstants", "encode_fp8", "decode_fp8", "dq_compress", "dq_decompress",
           "bits_per_param"]
