"""4-bit codebooks (NF4 and the table-driven ablation types) for the GPU path.

Mirrors ``qlrt.codebooks`` (pkg/src/qlrt/codebooks.py:86-323): the same
float64 construction -- inverse normal CDF by rational approximation plus
one Newton step against ``erfc`` (codebooks.py:86-117), NF-k asymmetric
quantiles with the omega offset (:184-206) -- so the table the kernels embed
is bit-identical to the reference's (pinned by tests against golden hex
values; the paper's fp32 table differs by up to 1.9e-7 and is NOT used).

``Codebook.to_c()`` produces the ``qlrt_codebook4`` struct: values, fp64
midpoints, and the fp32 brackets the quantize kernel's fast path uses.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

from . import _native

# rational-approximation coefficients (central / tail) -- published constants
_CA = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
       1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_CB = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
       6.680131188771972e+01, -1.328068155288572e+01)
_TC = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
       -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_TD = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
       3.754408661907416e+00)


def _poly(cs, t):
    out = cs[0]
    for c in cs[1:]:
        out = out * t + c
    return out


def inv_normal_cdf(p: float) -> float:
    """Standard-normal quantile; evaluation order matches codebooks.py:86-117."""
    p = float(p)
    if not 0.0 < p < 1.0:
        raise ValueError(f"inv_normal_cdf domain is the open interval (0, 1), got {p!r}")
    if p == 0.5:
        return 0.0
    if p < 0.02425 or p > 1.0 - 0.02425:
        t = math.sqrt(-2.0 * math.log(p if p < 0.5 else 1.0 - p))
        x = _poly(_TC, t) / (_poly(_TD, t) * t + 1.0)
        if p > 0.5:
            x = -x
    else:
        q = p - 0.5
        r = q * q
        x = _poly(_CA, r) * q / (_poly(_CB, r) * r + 1.0)
    x -= (0.5 * math.erfc(-x / math.sqrt(2.0)) - p) / (math.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)) \
        if math.exp(-0.5 * x * x) > 0.0 else 0.0
    return x


@dataclass(frozen=True, eq=False)
class Codebook:
    """Decode table of a k-bit data type (codebooks.py:125-176)."""

    name: str
    bits: int
    values: np.ndarray
    n_emitted: int

    @property
    def emitted_values(self) -> np.ndarray:
        return self.values[: self.n_emitted]

    @property
    def zero_code(self):
        z = np.flatnonzero(self.emitted_values == 0.0)
        return int(z[0]) if z.size else None

    @property
    def max_gap(self) -> float:
        return float(np.diff(self.emitted_values).max())

    def midpoints(self) -> np.ndarray:
        ev = self.emitted_values
        return (ev[:-1] + ev[1:]) / 2.0

    @property
    def pad_code(self) -> int:
        """Code for padding and all-zero blocks (blockquant.py:173-176)."""
        if self.zero_code is not None:
            return self.zero_code
        return int(np.searchsorted(self.midpoints(), 0.0, side="right"))

    @functools.cached_property
    def _c_struct(self) -> "_native.Codebook4":
        if self.bits != 4:
            raise ValueError(f"the GPU kernels handle 4-bit codebooks only, got k={self.bits}")
        cb = _native.Codebook4()
        mids = self.midpoints()
        for i in range(16):
            cb.values[i] = float(self.values[i])
            cb.lo[i] = np.inf
            cb.hi[i] = np.inf
        for i, m in enumerate(mids):
            cb.mids[i] = float(m)
            d = max(abs(float(m)) * 2.0 ** -19, 2.0 ** -100)
            lo = np.float32(m - d)
            if float(lo) > m - d:
                lo = np.nextafter(lo, np.float32(-np.inf))
            hi = np.float32(m + d)
            if float(hi) < m + d:
                hi = np.nextafter(hi, np.float32(np.inf))
            cb.lo[i], cb.hi[i] = float(lo), float(hi)
        cb.n_mids = mids.size
        cb.pad_code = self.pad_code
        return cb

    def to_c(self) -> "_native.Codebook4":
        return self._c_struct


def make_nf_codebook(k: int = 4) -> Codebook:
    """NF-k: asymmetric quantiles, exact 0, endpoints +-1 (codebooks.py:184-206)."""
    if not 2 <= k <= 8:
        raise ValueError(f"k must be in [2, 8], got {k}")
    omega = 0.5 * ((1.0 - 1.0 / (2.0 * 2 ** k)) + (1.0 - 1.0 / (2.0 * (2 ** k - 1))))
    upper = [inv_normal_cdf(p) for p in np.linspace(0.5, omega, 2 ** (k - 1) + 1)[1:]]
    lower = [-inv_normal_cdf(p) for p in np.linspace(0.5, omega, 2 ** (k - 1))[1:]]
    v = np.array(sorted(lower) + [0.0] + upper, dtype=np.float64)
    return Codebook(f"nf{k}", k, v / v[-1], 2 ** k)


def make_nf_midpoint_codebook(k: int = 4) -> Codebook:
    """nf-eq: averaged adjacent quantiles, no exact zero (codebooks.py:209-224)."""
    if not 2 <= k <= 8:
        raise ValueError(f"k must be in [2, 8], got {k}")
    pos = np.arange(1, 2 ** k + 2, dtype=np.float64) / (2 ** k + 2.0)
    q = np.array([inv_normal_cdf(p) for p in pos])
    m = 0.5 * (q[:-1] + q[1:])
    return Codebook(f"nf-eq{k}", k, m / np.max(np.abs(m)), 2 ** k)


def _float_grid(e_bits: int, m_bits: int, bias: int) -> list:
    out = set()
    for e in range(2 ** e_bits):
        for m in range(2 ** m_bits):
            out.add((m / 2.0 ** m_bits) * 2.0 ** (1 - bias) if e == 0
                    else (1.0 + m / 2.0 ** m_bits) * 2.0 ** (e - bias))
    return sorted(out)


def make_fp4_codebook(variant: str = "e2m1") -> Codebook:
    """fp4-e2m1 (bias 1) / fp4-e3m0 (bias 3), spare code = 0 (codebooks.py:251-271)."""
    variant = str(getattr(variant, "value", variant))
    if variant not in ("e2m1", "e3m0"):
        raise ValueError(f"unknown fp4 variant {variant!r}")
    mags = _float_grid(2, 1, 1) if variant == "e2m1" else _float_grid(3, 0, 3)
    top = mags[-1]
    vals = sorted({sgn * m / top for m in mags for sgn in (-1.0, 1.0)})
    return Codebook(f"fp4-{variant}", 4, np.array(vals + [0.0], dtype=np.float64), len(vals))


def make_int_codebook(k: int = 4) -> Codebook:
    """Symmetric integer grid, spare code = 0 (codebooks.py:279-290)."""
    if not 2 <= k <= 8:
        raise ValueError(f"k must be in [2, 8], got {k}")
    m = 2 ** (k - 1) - 1
    return Codebook(f"int{k}", k, np.append(np.arange(-m, m + 1, dtype=np.float64) / m, 0.0), 2 ** k - 1)


CODEBOOK_NAMES = ("nf4", "fp4-e2m1", "fp4-e3m0", "int4", "nf-eq4", "int8")


@functools.lru_cache(maxsize=None)
def _cached(name: str, bits) -> Codebook:
    if name.startswith("fp4-"):
        if bits not in (None, 4):
            raise ValueError("fp4 variants are 4-bit only")
        return make_fp4_codebook(name[4:])
    for fam, maker in (("nf-eq", make_nf_midpoint_codebook), ("nf", make_nf_codebook),
                       ("int", make_int_codebook)):
        if name.startswith(fam):
            suf = name[len(fam):]
            if suf and not suf.isdigit():
                break
            if suf and bits is not None and int(suf) != bits:
                raise ValueError(f"type {name!r} conflicts with bits={bits}")
            return maker(bits if bits is not None else (int(suf) if suf else 4))
    raise ValueError(f"unknown codebook type {name!r}")


def get_codebook(name: str, bits: int | None = None) -> Codebook:
    """Resolve a codebook by type string (codebooks.py:300-323)."""
    return _cached(name.lower(), bits)


__all__ = ["Codebook", "inv_normal_cdf", "make_nf_codebook", "make_nf_midpoint_codebook",
           "make_fp4_codebook", "make_int_codebook", "get_codebook", "CODEBOOK_NAMES"]
