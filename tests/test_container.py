"""The .qlrt container (pkg/docs/FORMAT.md) on GPU tensors: reference-written
files (tests/golden/containers, made by make_golden_container.py) load and
dequantize bit-exactly, GPU-quantized tensors save to the reference's exact
bytes, and the failure taxonomy matches (pkg/tests/test_container.py)."""

from __future__ import annotations

import os
import struct
import zlib

import numpy as np
import pytest
import torch

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "containers")
CASES = {"golden_nf4_dq": ("nf4", 64, True), "nf4_plain_64x64": ("nf4", 64, False),
         "nf4_dq_ragged": ("nf4", 64, True), "int4_plain": ("int4", 64, False), "fp4_dq": ("fp4-e2m1", 64, True),
         "nfeq4_b16": ("nf-eq4", 16, False), "scalar": ("nf4", 64, False)}
# k != 4: one byte per code in the file (reference container.py:180-181)
K_CASES = {"nf3_plain": ("nf3", 64, False), "int8_dq": ("int8", 64, True), "int2_b32": ("int2", 32, False)}


def _bytes(name):
    with open(os.path.join(HERE, name + ".qlrt"), "rb") as fh:
        return fh.read()


# ---------------------------------------------------------------- host only
def test_inspect_reference_files():
    from paper_2305_14314_b200 import container
    for name, (cb, bs, dq) in {**CASES, **K_CASES}.items():
        info = container.inspect_header(os.path.join(HERE, name + ".qlrt"))
        assert info["codebook"] == cb and info["blocksize"] == bs and info["double_quant"] is dq
        assert info["crc_ok"] is True and info["file_bytes"] == len(_bytes(name))
        if dq:
            assert info["blocksize2"] == 256 and info["fp8"] == "e4m3b7"
    info = container.inspect_header(os.path.join(HERE, "golden_nf4_dq.qlrt"))
    assert info["shape"] == (8, 16) and info["numel"] == 128 and info["n_blocks"] == 2


def test_failure_taxonomy(tmp_path):
    from paper_2305_14314_b200 import container
    from paper_2305_14314_b200.errors import (BadMagicError, ChecksumMismatchError, ContainerError, QlrtError,
                                              TruncatedFileError, UnsupportedVersionError)
    good = _bytes("nf4_dq_ragged")
    p = tmp_path / "t.qlrt"

    def check(data, exc, fn=container.inspect_header):
        p.write_bytes(data)
        with pytest.raises(exc):
            fn(str(p))

    check(b"XXXX" + good[4:], BadMagicError)
    check(good[:4] + struct.pack("<I", 2) + good[8:], UnsupportedVersionError)
    check(good[:8] + struct.pack("<H", 9) + good[10:], ContainerError)
    blk = 16 + 8 * 2
    check(good[:blk] + struct.pack("<I", 0) + good[blk + 4:], ContainerError)
    for keep in (0, 3, 15, 20, len(good) - 1):
        check(good[:keep], TruncatedFileError)
    check(good + b"\0", TruncatedFileError)
    bad = bytearray(good)
    bad[-5] ^= 0xFF
    p.write_bytes(bytes(bad))
    assert container.inspect_header(str(p))["crc_ok"] is False
    assert issubclass(ChecksumMismatchError, ContainerError) and issubclass(ContainerError, QlrtError)
    assert issubclass(BadMagicError, ContainerError) and issubclass(TruncatedFileError, ContainerError)
    assert container.MAGIC == b"QLRT" and container.VERSION == 1


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_reference_files_load_and_resave_byte_identical(tmp_path, qb, cuda):
    from paper_2305_14314_b200 import container
    arr = np.load(os.path.join(HERE, "arrays.npz"))
    for name in CASES:
        q = container.load(os.path.join(HERE, name + ".qlrt"))
        assert q.codes.is_cuda
        assert np.array_equal(qb.dequantize(q).cpu().numpy().reshape(arr[name + "/deq"].shape), arr[name + "/deq"])
        out = tmp_path / (name + ".qlrt")
        n = container.save(q, str(out))
        assert out.read_bytes() == _bytes(name) and n == len(_bytes(name)), name
    for name, (cb, bs, dq) in K_CASES.items():  # byte round trip (the kernels quantize 4-bit only)
        q = container.load(os.path.join(HERE, name + ".qlrt"))
        assert q.codebook.bits == int(cb[-1]) and q.codes.numel() == q.n_blocks * bs
        out = tmp_path / (name + ".qlrt")
        assert container.save(q, str(out)) == len(_bytes(name)) and out.read_bytes() == _bytes(name), name


@pytest.mark.gpu
def test_gpu_quantized_tensors_save_to_reference_bytes(tmp_path, qb, cuda):
    from paper_2305_14314_b200 import container
    arr = np.load(os.path.join(HERE, "arrays.npz"))
    for name, (cb, bs, dq) in CASES.items():
        x = arr[name + "/x"]
        q = qb.quantize(torch.from_numpy(np.atleast_1d(x).reshape(x.shape) if x.shape else x.reshape(()).copy()),
                        qb.get_codebook(cb), bs, double_quant=dq)
        out = tmp_path / (name + ".qlrt")
        container.save(q, str(out))
        assert out.read_bytes() == _bytes(name), name
        body = out.read_bytes()
        assert struct.unpack("<I", body[-4:])[0] == zlib.crc32(body[:-4]) & 0xFFFFFFFF
