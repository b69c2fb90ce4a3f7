"""The ``.qlrt`` container for GPU-resident quantized tensors (SURVEY.md §8(f)
rank 2), byte-compatible with the reference's format version 1
(pkg/docs/FORMAT.md; reference implementation pkg/src/qlrt/container.py:49-225).

``save`` takes a :class:`BlockQuantized` whose arrays live on the GPU (the
output of the sm_100a quantizer) and writes exactly the bytes the reference
would write for the same tensor; ``load`` reads any version-1 file (the
reference's or ours) straight into device tensors ready for ``dequantize`` /
``QLinear`` -- no re-quantization.  ``inspect_header`` reports the fields and
a ``crc_ok`` flag without raising on a corrupt payload.
"""

from __future__ import annotations

import struct
import zlib

import numpy as np
import torch

from .blockquant import BlockQuantized
from .codebooks import get_codebook
from .doublequant import DQConstants, Fp8Spec
from .errors import BadMagicError, ChecksumMismatchError, ContainerError, TruncatedFileError, UnsupportedVersionError

MAGIC = b"QLRT"
VERSION = 1
_PREFIX = struct.Struct("<4sIHBBI")      # magic, version, family, k, flags, ndim (16 bytes)
_DQ_SUB = struct.Struct("<fI4B")         # mu, blocksize2, exp, mant, bias, 0 (12 bytes)
_FAMILIES = ("nf", "fp4-e2m1", "fp4-e3m0", "int", "nf-eq")  # family id = index + 1
_F_DQ = 1


def _family_id(name: str) -> int:
    """Family of a codebook name (FORMAT.md 'Codebook family ids')."""
    for fam in ("fp4-e2m1", "fp4-e3m0", "nf-eq"):
        if name == fam or (fam == "nf-eq" and name.startswith("nf-eq")):
            return _FAMILIES.index(fam) + 1
    for fam in ("nf", "int"):
        if name.startswith(fam) and name[len(fam):].isdigit():
            return _FAMILIES.index(fam) + 1
    raise ValueError(f"codebook {name!r} has no container family id")


def _host(t: torch.Tensor, dtype) -> bytes:
    return np.ascontiguousarray(t.detach().cpu().numpy().astype(dtype, copy=False)).tobytes()


def save(q: BlockQuantized, path: str) -> int:
    """Serialize ``q`` (device arrays) to ``path``; returns the byte count."""
    cb = q.codebook
    fid = _family_id(cb.name)
    nb = q.n_blocks
    flags = _F_DQ if q.dq is not None else 0
    parts = [_PREFIX.pack(MAGIC, VERSION, fid, cb.bits, flags, len(q.shape)),
             b"".join(struct.pack("<Q", int(d)) for d in q.shape), struct.pack("<I", q.blocksize)]
    if q.dq is None:
        if q.constants is None or q.constants.numel() != nb:
            raise ValueError("plain container needs one float32 constant per block")
        parts.append(_host(q.constants, "<f4"))
    else:
        d = q.dq
        parts.append(_DQ_SUB.pack(float(np.float32(d.mu.reshape(-1)[0].item())), d.blocksize2,
                                  d.spec.exp_bits, d.spec.mant_bits, d.spec.bias, 0))
        parts.append(_host(d.c1, "<f4"))
        parts.append(_host(d.codes, "u1"))
    payload = _code_bytes(nb * q.blocksize, cb.bits)
    codes = _host(q.codes, "u1")
    if len(codes) != payload:
        raise ValueError(f"packed code buffer is {len(codes)} bytes, the container needs {payload}")
    parts.append(codes)
    body = b"".join(parts)
    data = body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)
    with open(path, "wb") as fh:
        fh.write(data)
    return len(data)


def _code_bytes(padded: int, k: int) -> int:
    """Packed code bytes of a container (container.py:180-181): two codes per
    byte for k = 4, one byte per code for every other k."""
    return (padded + 1) // 2 if k == 4 else padded


class _Cursor:
    def __init__(self, data: bytes):
        self.data, self.off = data, 0

    def take(self, n: int, what: str) -> bytes:
        if n < 0 or self.off + n > len(self.data):
            raise TruncatedFileError(f"file truncated in {what}: need {n} bytes at offset {self.off}, "
                                     f"{len(self.data) - self.off} remain")
        b = self.data[self.off: self.off + n]
        self.off += n
        return b


def _read(data: bytes, payload: bool, device) -> dict:
    cur = _Cursor(data)
    magic, version, fid, k, flags, ndim = _PREFIX.unpack(cur.take(_PREFIX.size, "header"))
    if magic != MAGIC:
        raise BadMagicError(f"expected magic {MAGIC!r}, found {magic!r}")
    if version != VERSION:
        raise UnsupportedVersionError(f"unsupported container version {version}")
    if not 1 <= fid <= len(_FAMILIES):
        raise ContainerError(f"unknown codebook family id {fid}")
    family = _FAMILIES[fid - 1]
    if ndim > 64:
        raise ContainerError(f"implausible ndim {ndim}")
    shape = struct.unpack(f"<{ndim}Q", cur.take(8 * ndim, "dims")) if ndim else ()
    (blocksize,) = struct.unpack("<I", cur.take(4, "blocksize"))
    if blocksize < 1:
        raise ContainerError("blocksize field must be >= 1")
    numel = int(np.prod(shape, dtype=np.int64)) if ndim else 1
    nb = -(-numel // blocksize)
    info = {"version": version, "codebook": family if family.startswith("fp4-") else f"{family}{k}", "k": k,
            "double_quant": bool(flags & _F_DQ), "shape": tuple(int(s) for s in shape), "blocksize": blocksize,
            "numel": numel, "n_blocks": nb}
    if flags & _F_DQ:
        mu, b2, eb, mb, bias, _ = _DQ_SUB.unpack(cur.take(_DQ_SUB.size, "dq subheader"))
        if b2 < 1:
            raise ContainerError("dq blocksize2 field must be >= 1")
        n2 = -(-nb // b2)
        c1 = cur.take(4 * n2, "dq scales")
        codes2 = cur.take(nb, "dq codes")
        info.update(blocksize2=b2, fp8=f"e{eb}m{mb}b{bias}")
        consts = (mu, b2, Fp8Spec(eb, mb, bias), c1, codes2)
    else:
        consts = cur.take(4 * nb, "constants")
    codes = cur.take(_code_bytes(nb * blocksize, k), "codes")
    (crc,) = struct.unpack("<I", cur.take(4, "crc32"))
    if cur.off != len(data):
        raise TruncatedFileError(f"{len(data) - cur.off} trailing bytes after the checksum")
    info["crc_ok"] = (zlib.crc32(data[: cur.off - 4]) & 0xFFFFFFFF) == crc
    if not payload:
        return info
    if not info["crc_ok"]:
        raise ChecksumMismatchError(f"crc32 mismatch: stored {crc:#010x}")
    cb = get_codebook(info["codebook"], bits=None if family.startswith("fp4-") else k)
    dev = torch.device(device)
    u8 = lambda b: torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)  # noqa: E731
    f32 = lambda b: torch.frombuffer(bytearray(b), dtype=torch.float32).to(dev)  # noqa: E731
    if flags & _F_DQ:
        mu, b2, spec, c1, codes2 = consts
        dq = DQConstants(mu=torch.tensor([mu], dtype=torch.float32, device=dev), blocksize2=b2, spec=spec,
                         c1=f32(c1), codes=u8(codes2))
        q = BlockQuantized(shape=info["shape"], blocksize=blocksize, codebook=cb, codes=u8(codes), constants=None,
                           dq=dq)
    else:
        q = BlockQuantized(shape=info["shape"], blocksize=blocksize, codebook=cb, codes=u8(codes),
                           constants=f32(consts), dq=None)
    info["quantized"] = q
    return info


def load(path: str, device="cuda") -> BlockQuantized:
    """Read a container into device tensors; raises the distinct error classes
    on bad magic, version mismatch, truncation and checksum failure."""
    with open(path, "rb") as fh:
        return _read(fh.read(), True, device)["quantized"]


def inspect_header(path: str) -> dict:
    """Header fields plus ``crc_ok`` and ``file_bytes``, without materializing the tensor."""
    with open(path, "rb") as fh:
        data = fh.read()
    info = _read(data, False, None)
    info["file_bytes"] = len(data)
    return info


__all__ = ["MAGIC", "VERSION", "save", "load", "inspect_header"]
