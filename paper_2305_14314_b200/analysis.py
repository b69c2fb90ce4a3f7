"""Data-type comparison on the GPU kernels -- mirror of
``qlrt.analysis.quant_error_report`` (pkg/src/qlrt/analysis.py:140-205), the
Table-3 style report (NF4 vs FP4 vs Int4, with and without double
quantization) computed at LLaMA scale through the sm_100a quantize /
dequantize kernels.

Same dataclasses and semantics: MSE is ``mean((x - dequantize(quantize(x)))**2)``
in float64 (the dequantized values are the reference's bit-exact float64),
entropy is the Shannon entropy in bits of the emitted-code histogram.  The
reductions run on the GPU in float64 (a different summation order than
numpy's pairwise sum: agreement to ~1e-12 relative, not bit-exact).
4-bit codebooks only (the GPU quantizer is 4-bit; int8 / nf3 stay with the
reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .blockquant import _as_input, dequantize, quantize, unpack_codes
from .codebooks import get_codebook
from .doublequant import bits_per_param


@dataclass(frozen=True)
class QuantConfig:
    """One quantization configuration to evaluate (analysis.py:140-151)."""

    codebook: str
    blocksize: int = 64
    double_quant: bool = False
    blocksize2: int = 256

    @property
    def label(self) -> str:
        tag = f"{self.codebook}/b{self.blocksize}"
        return tag + (f"/dq{self.blocksize2}" if self.double_quant else "")


@dataclass(frozen=True)
class QuantErrorRow:
    label: str
    bits_per_param: float
    mse: float
    max_abs_err: float
    entropy_bits: float
    occupancy: tuple[int, ...]


def quant_error_report(x, configs: list[QuantConfig]) -> list[QuantErrorRow]:
    """Quantize ``x`` under each config on the GPU and report reconstruction
    error and code usage (analysis.py:164-205)."""
    xt = _as_input(x)
    x64 = xt.to(torch.float64).reshape(-1)
    rows = []
    for cfg in configs:
        cb = get_codebook(cfg.codebook)
        q = quantize(xt, cb, blocksize=cfg.blocksize, double_quant=cfg.double_quant,
                     blocksize2=cfg.blocksize2)
        err = x64 - dequantize(q).reshape(-1)
        n = q.numel
        codes = unpack_codes(q.codes, 4, n).to(torch.int64)
        counts = torch.bincount(codes, minlength=cb.n_emitted)
        probs = counts[counts > 0].to(torch.float64) / n
        entropy = float(-(probs * torch.log2(probs)).sum())
        sq = (err * err).sum() / n
        rows.append(QuantErrorRow(
            label=cfg.label,
            bits_per_param=bits_per_param(cb.bits, cfg.blocksize,
                                          (cfg.blocksize2, 8) if cfg.double_quant else None),
            mse=float(sq),
            max_abs_err=float(err.abs().max()),
            entropy_bits=entropy,
            occupancy=tuple(int(c) for c in counts.cpu().tolist()),
        ))
    return rows


__all__ = ["QuantConfig", "QuantErrorRow", "quant_error_report"]
