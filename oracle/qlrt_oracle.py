"""CPU oracle for the NF4 / double-quant / QLoRA-linear hot path.

TEST INFRASTRUCTURE ONLY.  This module is a numpy restatement of the
reference package ``qlrt`` 0.1.0 (``/root/reference/pkg/src/qlrt``).  It is
imported by ``tests/``, by ``__graft_entry__.smoke()`` and by the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- as the
*checker* and as the timed CPU baseline, never as the product.  The product
(``paper_2305_14314_b200``) never imports it; the product path runs on the
CUDA library and fails loudly without it.

Parity pinning: every function here is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the real reference in
the build container (``tests/test_oracle.py``).  The one quantity the
reference tests do not pin -- the summation order of the double-quant mean
-- is pinned by running the reference's own ``dq_compress`` on the same
numpy (2.3.5, bufsize 8192) over adversarial inputs (``tests/golden``).

Each function cites the reference ``file:line`` it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

REF = "pkg/src/qlrt"  # all citations below are relative to /root/reference

# ---------------------------------------------------------------------------
# codebooks  (restates pkg/src/qlrt/codebooks.py)
# ---------------------------------------------------------------------------

# Acklam-style rational approximation + one Newton step against erfc
# (codebooks.py:55-117).  Coefficients are the published constants.
_A = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
      1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_B = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
      6.680131188771972e+01, -1.328068155288572e+01)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
      -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
      3.754408661907416e+00)
_PLOW = 0.02425


def _horner(coeffs, t):
    acc = coeffs[0]
    for c in coeffs[1:]:
        acc = acc * t + c
    return acc


def inv_normal_cdf(p: float) -> float:
    """codebooks.py:86-117 -- evaluation order kept term-for-term so the
    float64 result is identical (the NF4 table is built from it)."""
    p = float(p)
    if not 0.0 < p < 1.0:
        raise ValueError(f"inv_normal_cdf domain is the open interval (0, 1), got {p!r}")
    if p == 0.5:
        return 0.0
    if p < _PLOW:
        t = math.sqrt(-2.0 * math.log(p))
        x = _horner(_C, t) / (_horner(_D, t) * t + 1.0)
    elif p > 1.0 - _PLOW:
        t = math.sqrt(-2.0 * math.log(1.0 - p))
        x = -(_horner(_C, t) / (_horner(_D, t) * t + 1.0))
    else:
        q = p - 0.5
        r = q * q
        x = _horner(_A, r) * q / (_horner(_B, r) * r + 1.0)
    err = 0.5 * math.erfc(-x / math.sqrt(2.0)) - p
    pdf = math.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    if pdf > 0.0:
        x -= err / pdf
    return x


@dataclass(frozen=True, eq=False)
class Codebook:
    """codebooks.py:125-176 (values f64, n_emitted, zero_code, midpoints)."""
    name: str
    bits: int
    values: np.ndarray
    n_emitted: int

    def emitted(self) -> np.ndarray:
        return self.values[: self.n_emitted]

    def midpoints(self) -> np.ndarray:          # codebooks.py:173-176
        e = self.emitted()
        return (e[:-1] + e[1:]) / 2.0

    @property
    def zero_code(self):                        # codebooks.py:162-166
        hit = np.flatnonzero(self.emitted() == 0.0)
        return int(hit[0]) if hit.size else None

    @property
    def max_gap(self) -> float:                 # codebooks.py:168-171
        return float(np.max(np.diff(self.emitted())))

    def pad_code(self) -> int:                  # blockquant.py:173-176
        if self.zero_code is not None:
            return self.zero_code
        return int(nearest_codes(np.zeros(1), self)[0])


def make_nf_codebook(k: int = 4) -> Codebook:
    """codebooks.py:184-206: asymmetric two-range quantiles, omega offset."""
    omega = 0.5 * ((1.0 - 1.0 / (2.0 * 2 ** k)) + (1.0 - 1.0 / (2.0 * (2 ** k - 1))))
    pos = [inv_normal_cdf(p) for p in np.linspace(0.5, omega, 2 ** (k - 1) + 1)[1:]]
    neg = [-inv_normal_cdf(p) for p in np.linspace(0.5, omega, 2 ** (k - 1))[1:]]
    vals = np.array(sorted(neg) + [0.0] + pos, dtype=np.float64)
    vals /= vals[-1]
    return Codebook(f"nf{k}", k, vals, 2 ** k)


def make_nf_midpoint_codebook(k: int = 4) -> Codebook:
    """codebooks.py:209-224 (nf-eq family, no exact zero)."""
    pos = np.arange(1, 2 ** k + 2, dtype=np.float64) / (2 ** k + 2.0)
    qs = np.array([inv_normal_cdf(p) for p in pos])
    mids = 0.5 * (qs[:-1] + qs[1:])
    return Codebook(f"nf-eq{k}", k, mids / np.max(np.abs(mids)), 2 ** k)


def _fp_mags(e_bits, m_bits, bias):
    out = set()
    for e in range(2 ** e_bits):
        for m in range(2 ** m_bits):
            if e == 0:
                out.add((m / 2.0 ** m_bits) * 2.0 ** (1 - bias))
            else:
                out.add((1.0 + m / 2.0 ** m_bits) * 2.0 ** (e - bias))
    return sorted(out)


def make_fp4_codebook(variant: str = "e2m1") -> Codebook:
    """codebooks.py:237-271."""
    mags = _fp_mags(2, 1, 1) if variant == "e2m1" else _fp_mags(3, 0, 3)
    top = mags[-1]
    distinct = sorted({s * m / top for m in mags for s in (-1.0, 1.0)})
    return Codebook(f"fp4-{variant}", 4, np.array(distinct + [0.0]), len(distinct))


def make_int_codebook(k: int = 4) -> Codebook:
    """codebooks.py:279-290."""
    m = 2 ** (k - 1) - 1
    grid = np.arange(-m, m + 1, dtype=np.float64) / m
    return Codebook(f"int{k}", k, np.concatenate([grid, [0.0]]), 2 ** k - 1)


def get_codebook(name: str) -> Codebook:
    """codebooks.py:300-323 (subset: the spellings the hot path uses)."""
    name = name.lower()
    if name.startswith("fp4-"):
        return make_fp4_codebook(name[4:])
    if name.startswith("nf-eq"):
        return make_nf_midpoint_codebook(int(name[5:] or 4))
    if name.startswith("nf"):
        return make_nf_codebook(int(name[2:] or 4))
    if name.startswith("int"):
        return make_int_codebook(int(name[3:] or 4))
    raise ValueError(f"unknown codebook type {name!r}")


# ---------------------------------------------------------------------------
# 8-bit float grid of the double quantizer (restates doublequant.py:33-121)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Fp8Spec:
    """doublequant.py:33-51; E4M3, bias 7, no NaN/Inf -> max 480."""
    exp_bits: int = 4
    mant_bits: int = 3
    bias: int = 7

    @property
    def max_value(self) -> float:
        return (2.0 - 2.0 ** -self.mant_bits) * 2.0 ** (2 ** self.exp_bits - 1 - self.bias)


def fp8_decode_table(spec: Fp8Spec = Fp8Spec()) -> np.ndarray:
    """doublequant.py:83-100: all 256 byte patterns -> float64."""
    t = np.empty(256)
    for b in range(256):
        e = (b >> spec.mant_bits) & (2 ** spec.exp_bits - 1)
        m = b & (2 ** spec.mant_bits - 1)
        mag = (m / 2.0 ** spec.mant_bits) * 2.0 ** (1 - spec.bias) if e == 0 else \
            (1.0 + m / 2.0 ** spec.mant_bits) * 2.0 ** (e - spec.bias)
        t[b] = -mag if b >> 7 else mag
    return t


def fp8_grid(spec: Fp8Spec = Fp8Spec()):
    """doublequant.py:53-77: sorted distinct values + canonical byte codes
    (+0 wins over -0 through the stable sort)."""
    table = fp8_decode_table(spec)
    order = np.argsort(table, kind="stable")
    vals, codes = table[order], np.arange(256, dtype=np.uint8)[order]
    keep = np.concatenate([[True], vals[1:] != vals[:-1]])
    return vals[keep], codes[keep]


def encode_fp8(x, spec: Fp8Spec = Fp8Spec()) -> np.ndarray:
    """doublequant.py:103-113: nearest grid value, ties away from zero,
    clamping at +-max."""
    vals, codes = fp8_grid(spec)
    x = np.asarray(x, dtype=np.float64)
    mids = (vals[:-1] + vals[1:]) / 2.0
    idx = np.where(x >= 0, np.searchsorted(mids, x, "right"),
                   np.searchsorted(mids, x, "left"))
    return codes[idx]


def decode_fp8(codes, spec: Fp8Spec = Fp8Spec()) -> np.ndarray:
    """doublequant.py:116-121."""
    return fp8_decode_table(spec)[np.asarray(codes, dtype=np.uint8)]


# ---------------------------------------------------------------------------
# numpy's float32->float64 add-reduce order (what ``constants.mean(dtype=
# np.float64)`` in doublequant.py:164 executes on numpy 2.3.5, bufsize 8192)
# ---------------------------------------------------------------------------

def _pairwise(a: np.ndarray) -> float:
    """numpy loops_utils.h.src pairwise_sum over float64 values."""
    n = a.size
    if n < 8:
        s = 0.0
        for v in a:
            s += float(v)
        return s
    if n <= 128:
        r = [float(a[j]) for j in range(8)]
        m = n - n % 8
        for i in range(8, m, 8):
            for j in range(8):
                r[j] += float(a[i + j])
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(m, n):
            s += float(a[i])
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a[:n2]) + _pairwise(a[n2:])


def numpy_order_sum_f64(c32: np.ndarray, chunk: int = 8192) -> float:
    """Buffered reduction: 8192-element chunks from index 0, each chunk
    pairwise-summed, chunk sums accumulated sequentially from 0.0."""
    a = np.asarray(c32, dtype=np.float32).astype(np.float64)
    acc = 0.0
    for s in range(0, a.size, chunk):
        acc += _pairwise(a[s:s + chunk])
    return acc


# ---------------------------------------------------------------------------
# double quantization (restates doublequant.py:129-223)
# ---------------------------------------------------------------------------

@dataclass
class DQConstants:
    """doublequant.py:129-145."""
    mu: np.float32
    blocksize2: int
    spec: Fp8Spec
    c1: np.ndarray
    codes: np.ndarray


def dq_compress(constants, blocksize2: int = 256, spec: Fp8Spec = Fp8Spec(),
                emulate_order: bool = False) -> DQConstants:
    """doublequant.py:148-187.  ``emulate_order`` swaps numpy's mean for the
    explicit buffered-pairwise restatement above (tests assert they agree)."""
    c = np.asarray(constants, dtype=np.float32)
    if c.ndim != 1 or c.size == 0:
        raise ValueError("constants must be a non-empty 1-d array")
    if blocksize2 < 1:
        raise ValueError(f"blocksize2 must be >= 1, got {blocksize2}")
    if np.any(c < 0) or not np.all(np.isfinite(c)):
        raise ValueError("constants must be finite and nonnegative")
    if emulate_order:
        mu = np.float32(numpy_order_sum_f64(c) / c.size)
    else:
        mu = np.float32(c.mean(dtype=np.float64))
    centered = c.astype(np.float64) - float(mu)
    n2 = -(-c.size // blocksize2)
    c1 = np.zeros(n2, dtype=np.float32)
    codes = np.zeros(c.size, dtype=np.uint8)
    top = spec.max_value
    for b in range(n2):
        sl = slice(b * blocksize2, (b + 1) * blocksize2)
        amax = np.abs(centered[sl]).max()
        if amax == 0.0:
            codes[sl] = encode_fp8(np.zeros(centered[sl].size), spec)
            continue
        s = np.float32(amax / top)
        if s == 0.0:
            continue
        c1[b] = s
        codes[sl] = encode_fp8(centered[sl] / np.float64(s), spec)
    return DQConstants(mu, blocksize2, spec, c1, codes)


def dq_decompress(dq: DQConstants) -> np.ndarray:
    """doublequant.py:190-195 (two fp64 roundings, clamp at 0, -> f32)."""
    dec = decode_fp8(dq.codes, dq.spec)
    scale = np.repeat(dq.c1.astype(np.float64), dq.blocksize2)[: dq.codes.size]
    return np.maximum(dec * scale + np.float64(dq.mu), 0.0).astype(np.float32)


def bits_per_param(k: int, blocksize: int, dq=None) -> float:
    """doublequant.py:203-223."""
    if k < 1 or blocksize < 1:
        raise ValueError("k and blocksize must be positive")
    if dq is None:
        return k + 32.0 / blocksize
    b2, bits2 = dq
    if b2 < 1 or bits2 < 1:
        raise ValueError("blocksize2 and bits2 must be positive")
    return k + bits2 / blocksize + 32.0 / (blocksize * b2)


# ---------------------------------------------------------------------------
# block-wise quantization (restates blockquant.py:34-213)
# ---------------------------------------------------------------------------

@dataclass
class BlockQuantized:
    """blockquant.py:34-73."""
    shape: tuple
    blocksize: int
    codebook: Codebook
    codes: np.ndarray
    constants: np.ndarray | None
    dq: DQConstants | None = None

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64)) if self.shape else 1

    @property
    def n_blocks(self) -> int:
        return -(-self.numel // self.blocksize)

    def block_constants(self) -> np.ndarray:
        return dq_decompress(self.dq) if self.dq is not None else self.constants

    def unpacked_codes(self) -> np.ndarray:
        padded = self.n_blocks * self.blocksize
        if self.codebook.bits in (4, 8):
            return unpack_codes(self.codes, self.codebook.bits, padded)
        return self.codes[:padded].copy()


def pack_codes(codes, k: int) -> np.ndarray:
    """blockquant.py:81-98: even index in the low nibble, odd tail -> 0."""
    if k not in (4, 8):
        raise ValueError(f"pack_codes supports k in {{4, 8}}, got {k}")
    codes = np.asarray(codes)
    if codes.size and (codes.min() < 0 or codes.max() >= 2 ** k):
        raise ValueError(f"codes out of range for k={k}")
    codes = codes.astype(np.uint8).ravel()
    if k == 8:
        return codes.copy()
    if codes.size % 2:
        codes = np.append(codes, np.uint8(0))
    return (codes[0::2] | (codes[1::2] << 4)).astype(np.uint8)


def unpack_codes(packed, k: int, count: int) -> np.ndarray:
    """blockquant.py:101-115."""
    if k not in (4, 8):
        raise ValueError(f"unpack_codes supports k in {{4, 8}}, got {k}")
    packed = np.asarray(packed, dtype=np.uint8)
    if (packed.size if k == 8 else packed.size * 2) < count:
        raise ValueError("packed buffer shorter than requested count")
    if k == 8:
        return packed[:count].copy()
    out = np.empty(packed.size * 2, dtype=np.uint8)
    out[0::2] = packed & 0x0F
    out[1::2] = packed >> 4
    return out[:count]


def nearest_codes(q: np.ndarray, cb: Codebook) -> np.ndarray:
    """blockquant.py:123-129: q >= 0 (incl. -0.0) -> #{mids <= q};
    q < 0 -> #{mids < q}  (ties away from zero)."""
    mids = cb.midpoints()
    return np.where(q >= 0, np.searchsorted(mids, q, "right"),
                    np.searchsorted(mids, q, "left")).astype(np.uint8)


def quantize(x, codebook: Codebook, blocksize: int = 64, double_quant: bool = False,
             blocksize2: int = 256, fp8_spec: Fp8Spec | None = None) -> BlockQuantized:
    """blockquant.py:132-195."""
    x = np.asarray(x)
    if x.size == 0:
        raise ValueError("cannot quantize an empty tensor")
    if blocksize < 1:
        raise ValueError(f"blocksize must be >= 1, got {blocksize}")
    flat = np.ascontiguousarray(x, dtype=np.float64).ravel()
    bad = np.flatnonzero(~np.isfinite(flat))
    if bad.size:
        raise ValueError(f"non-finite input at flat index {int(bad[0])}")
    nb = -(-flat.size // blocksize)
    blocks = np.zeros(nb * blocksize)
    blocks[: flat.size] = flat
    blocks = blocks.reshape(nb, blocksize)
    constants = np.abs(blocks).max(axis=1).astype(np.float32)   # :166
    scale = constants.astype(np.float64)
    live = scale > 0.0
    norm = np.zeros_like(blocks)
    np.divide(blocks, scale[:, None], out=norm, where=live[:, None])  # :167-170
    codes = nearest_codes(norm, codebook).reshape(-1)
    pad = codebook.pad_code()
    codes[flat.size:] = pad                                       # :177-178
    codes[~np.repeat(live, blocksize)] = pad                      # :179
    k = codebook.bits
    packed = pack_codes(codes, k) if k in (4, 8) else codes.copy()
    dq = dq_compress(constants, blocksize2, fp8_spec or Fp8Spec()) if double_quant else None
    return BlockQuantized(tuple(x.shape), blocksize, codebook, packed,
                          None if double_quant else constants, dq)


class CorruptDataError(Exception):
    """errors.py:35-37 (the oracle raises the same message text)."""


def dequantize(q: BlockQuantized) -> np.ndarray:
    """blockquant.py:198-213: float64, original shape."""
    codes = q.unpacked_codes()
    if codes.size and codes.max() >= q.codebook.values.size:
        raise CorruptDataError(f"code {int(codes.max())} out of range for k={q.codebook.bits}")
    c = q.block_constants().astype(np.float64)
    if c.shape != (q.n_blocks,):
        raise CorruptDataError(f"expected {q.n_blocks} block constants, got {c.shape}")
    out = q.codebook.values[codes].reshape(q.n_blocks, q.blocksize) * c[:, None]
    return out.reshape(-1)[: q.numel].reshape(q.shape)


# ---------------------------------------------------------------------------
# QLoRA linear (restates qlora.py:48-167), float64 "high" precision mode
# ---------------------------------------------------------------------------

@dataclass
class LoraAdapter:
    """qlora.py:48-60."""
    rank: int
    alpha: float
    l1: np.ndarray
    l2: np.ndarray
    dropout_p: float = 0.0

    @property
    def scaling(self) -> float:
        return self.alpha / self.rank


def qlinear_forward(w: np.ndarray, adapters, x: np.ndarray, masks=None, dtype=np.float64):
    """qlora.py:124-148 with the dense base ``w`` already at compute
    precision.  ``masks`` (optional, per adapter) replays dropout."""
    x = x.astype(dtype, copy=False)
    w = w.astype(dtype, copy=False)
    y = x @ w
    branches = []
    for i, ad in enumerate(adapters):
        mask = None if masks is None else masks[i]
        xa = x if mask is None else x * mask
        t = xa @ ad.l1.astype(dtype)
        y = y + dtype(ad.scaling) * (t @ ad.l2.astype(dtype))
        branches.append({"xa": xa, "t": t, "mask": mask})
    return y, {"x": x, "w": w, "branches": branches}


def qlinear_backward(adapters, d_y: np.ndarray, cache, dtype=np.float64):
    """qlora.py:150-167."""
    d_y = d_y.astype(dtype, copy=False)
    d_x = d_y @ cache["w"].T
    grads = {}
    for i, (ad, br) in enumerate(zip(adapters, cache["branches"])):
        s = dtype(ad.scaling)
        d_t = s * (d_y @ ad.l2.astype(dtype).T)
        grads[f"adapter{i}.l2"] = s * (br["t"].T @ d_y)
        grads[f"adapter{i}.l1"] = br["xa"].T @ d_t
        d_xa = d_t @ ad.l1.astype(dtype).T
        if br["mask"] is not None:
            d_xa = d_xa * br["mask"]
        d_x = d_x + d_xa
    return d_x, grads


# ---------------------------------------------------------------------------
# optimizer (restates training.py:62-90, 398-442)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class TrainConfig:
    """training.py:62-90 (defaults)."""
    learning_rate: float = 0.01
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    max_grad_norm: float = 0.3


def clip_global_norm(grads: dict, order: list, max_norm: float) -> float:
    """training.py:398-413: fp64 sum of squares, in-place scale."""
    total = 0.0
    for name in order:
        total += float(np.sum(np.square(grads[name], dtype=np.float64)))
    norm = math.sqrt(total)
    if norm > max_norm and norm > 0.0:
        scale = max_norm / norm
        for name in order:
            g = grads[name]
            g *= g.dtype.type(scale)
    return norm


@dataclass
class AdamState:
    t: int = 0
    moments: dict = field(default_factory=dict)


def adam_step(params: dict, grads: dict, cfg: TrainConfig, state: AdamState) -> None:
    """training.py:426-442.  For float32 params numpy 2 (NEP 50) rounds the
    Python-float constants to float32 first; the op order is kept."""
    state.t += 1
    bc1 = 1.0 - cfg.adam_beta1 ** state.t
    bc2 = 1.0 - cfg.adam_beta2 ** state.t
    for name, p in params.items():
        g = grads[name]
        if name not in state.moments:
            state.moments[name] = (np.zeros_like(p), np.zeros_like(p))
        m, v = state.moments[name]
        m *= cfg.adam_beta1
        m += (1.0 - cfg.adam_beta1) * g
        v *= cfg.adam_beta2
        v += (1.0 - cfg.adam_beta2) * (g * g)
        step = (m / bc1) / (np.sqrt(v / bc2) + cfg.adam_eps)
        p -= cfg.learning_rate * step
