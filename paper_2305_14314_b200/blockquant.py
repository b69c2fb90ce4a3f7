"""Block-wise NF4 quantization on the GPU -- mirror of ``qlrt.blockquant``
(pkg/src/qlrt/blockquant.py:34-213) with the reference's names, argument
meaning and errors; arrays are CUDA tensors instead of numpy arrays.

Bit-exactness: codes (packed, even index in the low nibble), float32
constants, the double-quant fields and the float64 dequantization are
identical to the reference on the same inputs (float32, bfloat16 or float64).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._native import BF16, F32, F64, check, lib, ptr, stream_ptr
from .codebooks import Codebook
from .doublequant import DQConstants, Fp8Spec, _dq_compress_unchecked, dq_decompress
from .errors import CorruptDataError

_IN_DTYPES = {torch.float32: F32, torch.bfloat16: BF16, torch.float64: F64}
_OUT_DTYPES = {torch.float32: F32, torch.bfloat16: BF16, torch.float64: F64}


@dataclass
class BlockQuantized:
    """Packed codes + per-block constants (or their DQ form) + codebook (blockquant.py:34-73)."""

    shape: tuple
    blocksize: int
    codebook: Codebook
    codes: torch.Tensor                 # uint8, device, ceil(n_blocks*blocksize/2)
    constants: torch.Tensor | None      # float32, device, [n_blocks] (None under DQ)
    dq: DQConstants | None = None

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def n_blocks(self) -> int:
        return (self.numel + self.blocksize - 1) // self.blocksize

    def block_constants(self) -> torch.Tensor:
        if self.dq is not None:
            return dq_decompress(self.dq)
        assert self.constants is not None
        return self.constants

    def unpacked_codes(self) -> torch.Tensor:
        return unpack_codes(self.codes, self.codebook.bits, self.n_blocks * self.blocksize)

    def to_numpy(self) -> dict:
        """Host copies of every field, named as on the reference object."""
        out = {"shape": self.shape, "blocksize": self.blocksize, "codes": self.codes.cpu().numpy()}
        if self.constants is not None:
            out["constants"] = self.constants.cpu().numpy()
        if self.dq is not None:
            out["dq.codes"] = self.dq.codes.cpu().numpy()
            out["dq.c1"] = self.dq.c1.cpu().numpy()
            out["dq.mu"] = np.float32(self.dq.mu.item())
        return out


def _as_input(x) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if x.dtype not in _IN_DTYPES:
        # float16 embeds exactly in float32; everything else follows the
        # reference's float64 cast (blockquant.py:153)
        x = x.to(torch.float32 if x.dtype == torch.float16 else torch.float64)
    return x.cuda().contiguous()


def pack_codes(codes, k: int) -> torch.Tensor:
    """Two 4-bit codes per byte, even index low nibble, odd tail -> 0 (blockquant.py:81-98)."""
    if k not in (4, 8):
        raise ValueError(f"pack_codes supports k in {{4, 8}}, got {k}")
    c = codes if isinstance(codes, torch.Tensor) else torch.from_numpy(np.asarray(codes))
    c = c.reshape(-1)
    if c.numel() and (int(c.min()) < 0 or int(c.max()) >= 2 ** k):
        raise ValueError(f"codes out of range for k={k}")
    c = c.to(torch.uint8).cuda().contiguous()
    if k == 8:
        return c.clone()
    out = torch.empty((c.numel() + 1) // 2, dtype=torch.uint8, device=c.device)
    if c.numel():
        check(lib().qlrt_pack4(ptr(c), c.numel(), ptr(out), stream_ptr()), "pack_codes")
    return out


def unpack_codes(packed, k: int, count: int) -> torch.Tensor:
    """Inverse of :func:`pack_codes`; exactly ``count`` codes (blockquant.py:101-115)."""
    if k not in (4, 8):
        raise ValueError(f"unpack_codes supports k in {{4, 8}}, got {k}")
    p = packed if isinstance(packed, torch.Tensor) else torch.from_numpy(np.asarray(packed, dtype=np.uint8))
    p = p.to(torch.uint8).cuda().contiguous().reshape(-1)
    if (p.numel() if k == 8 else 2 * p.numel()) < count:
        raise ValueError("packed buffer shorter than requested count")
    if k == 8:
        return p[:count].clone()
    out = torch.empty(count, dtype=torch.uint8, device=p.device)
    if count:
        check(lib().qlrt_unpack4(ptr(p), count, ptr(out), stream_ptr()), "unpack_codes")
    return out


def quantize_async(x, codebook: Codebook, blocksize: int = 64, double_quant: bool = False, blocksize2: int = 256,
                   fp8_spec: Fp8Spec | None = None):
    """Launch-only quantize (no host sync, CUDA-graph capturable): returns the
    ``BlockQuantized`` and the device int64 holding the first non-finite flat
    index (0x7F7F... when none).  :func:`quantize` adds the check."""
    L = lib()  # no CUDA library / device -> RuntimeError before touching the data
    shape = tuple(x.shape) if hasattr(x, "shape") else ()
    xt = _as_input(x)
    if xt.numel() == 0:
        raise ValueError("cannot quantize an empty tensor")
    if blocksize < 1:
        raise ValueError(f"blocksize must be >= 1, got {blocksize}")
    if codebook.bits != 4:
        raise ValueError(f"the GPU quantizer handles 4-bit codebooks only, got k={codebook.bits}")
    if double_quant and blocksize2 < 1:
        raise ValueError(f"blocksize2 must be >= 1, got {blocksize2}")
    n = xt.numel()
    nb = (n + blocksize - 1) // blocksize
    n_pad = nb * blocksize
    codes = torch.empty((n_pad + 1) // 2 + 3 & ~3, dtype=torch.uint8, device=xt.device)
    absmax = torch.empty(nb, dtype=torch.float32, device=xt.device)
    bad = torch.empty(1, dtype=torch.int64, device=xt.device)
    check(L.qlrt_quantize4(ptr(xt), _IN_DTYPES[xt.dtype], n, blocksize, codebook.to_c(), ptr(codes), ptr(absmax),
                           ptr(bad), stream_ptr()), "quantize")
    codes = codes[: (n_pad + 1) // 2]
    dq = _dq_compress_unchecked(absmax, blocksize2, fp8_spec or Fp8Spec()) if double_quant else None
    q = BlockQuantized(shape=shape, blocksize=blocksize, codebook=codebook, codes=codes,
                       constants=None if double_quant else absmax, dq=dq)
    return q, bad


def quantize(x, codebook: Codebook, blocksize: int = 64, double_quant: bool = False, blocksize2: int = 256,
             fp8_spec: Fp8Spec | None = None) -> BlockQuantized:
    """Block-wise absmax quantization against ``codebook`` (blockquant.py:132-195).

    Raises ``ValueError`` for an empty tensor, ``blocksize < 1`` and the first
    non-finite flat index -- the reference's messages (one host sync).
    """
    q, bad = quantize_async(x, codebook, blocksize, double_quant, blocksize2, fp8_spec)
    first = int(bad.item())
    if first < q.numel:
        raise ValueError(f"non-finite input at flat index {first}")
    return q


def dequantize(q: BlockQuantized, dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """``values[code] * f64(constant)`` in the original shape (blockquant.py:198-213).

    ``dtype=float64`` is the reference's own output, bit-exact; float32 is
    ``f32`` of it and bfloat16 is ``bf16(f32(.))`` (what QLinear consumes).
    """
    if dtype not in _OUT_DTYPES:
        raise ValueError(f"dequantize writes float64, float32 or bfloat16, got {dtype}")
    if q.codebook.bits != 4:
        raise ValueError(f"the GPU dequantizer handles 4-bit codebooks only, got k={q.codebook.bits}")
    nb = q.n_blocks
    if q.dq is not None:
        if q.dq.n_constants != nb:
            raise CorruptDataError(f"expected {nb} block constants, got ({q.dq.n_constants},)")
    elif q.constants is None or tuple(q.constants.shape) != (nb,):
        got = None if q.constants is None else tuple(q.constants.shape)
        raise CorruptDataError(f"expected {nb} block constants, got {got}")
    if q.codes.numel() * 2 < nb * q.blocksize - 1:
        raise CorruptDataError("packed code buffer shorter than the block grid")
    n = q.numel
    out = torch.empty(n, dtype=dtype, device=q.codes.device)
    dq = q.dq
    check(lib().qlrt_dequantize4(
        ptr(q.codes), n, q.blocksize, q.codebook.to_c(),
        None if dq is not None else ptr(q.constants),
        ptr(dq.codes) if dq else None, ptr(dq.c1) if dq else None, ptr(dq.mu) if dq else None,
        dq.blocksize2 if dq else 1, (dq.spec if dq else Fp8Spec()).to_c(),
        ptr(out), _OUT_DTYPES[dtype], stream_ptr()), "dequantize")
    return out.reshape(q.shape)


__all__ = ["BlockQuantized", "quantize", "quantize_async", "dequantize", "pack_codes", "unpack_codes"]
