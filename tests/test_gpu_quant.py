"""GPU parity: quantize / double-quant / dequantize are bit-exact with the
reference (golden vectors from the real qlrt) and with the CPU oracle."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def h16(a) -> str:
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def test_golden_quant_cases(golden, golden_meta, qb, cuda):
    for c in golden_meta["quant_cases"]:
        tag = c["tag"]
        x = golden[f"q/{tag}/x"]
        q = qb.quantize(x, qb.get_codebook(c["codebook"]), c["blocksize"], c["double_quant"], c["blocksize2"])
        assert q.shape == tuple(c["shape"])
        assert np.array_equal(q.codes.cpu().numpy(), golden[f"q/{tag}/codes"]), tag
        if c["double_quant"]:
            assert np.array_equal(q.dq.codes.cpu().numpy(), golden[f"q/{tag}/dq_codes"]), tag
            assert np.array_equal(q.dq.c1.cpu().numpy(), golden[f"q/{tag}/dq_c1"]), tag
            assert q.dq.mu.cpu().numpy()[0] == golden[f"q/{tag}/dq_mu"][0], tag
            assert np.array_equal(q.block_constants().cpu().numpy(), golden[f"q/{tag}/absmax_dq"]), tag
        else:
            assert np.array_equal(q.constants.cpu().numpy(), golden[f"q/{tag}/constants"]), tag
        ref = golden[f"q/{tag}/deq"]
        assert np.array_equal(qb.dequantize(q).cpu().numpy(), ref), tag                       # float64, bit-exact
        assert np.array_equal(qb.dequantize(q, torch.float32).cpu().numpy(), ref.astype(np.float32)), tag
        bf = qb.dequantize(q, torch.bfloat16).cpu()
        assert torch.equal(bf, torch.from_numpy(ref.astype(np.float32)).to(torch.bfloat16)), tag


def test_config_c1_hashes(golden_meta, qb, cuda):
    """4096^2 Gaussian, NF4 / 64 / DQ 256 -- every field bit-exact."""
    meta = golden_meta["c1"]
    x = np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32)
    assert h16(x) == meta["x"]
    q = qb.quantize(torch.from_numpy(x).cuda(), qb.get_codebook("nf4"), 64, double_quant=True, blocksize2=256)
    assert h16(q.codes) == meta["codes"]
    assert h16(q.dq.codes) == meta["dq_codes"]
    assert h16(q.dq.c1) == meta["dq_c1"]
    assert float(q.dq.mu.item()).hex() == meta["mu_hex"]
    assert h16(q.block_constants()) == meta["absmax_dq"]
    assert h16(qb.dequantize(q, torch.float32)) == meta["deq_f32"]
    assert h16(qb.dequantize(q, torch.bfloat16).view(torch.int16)) == meta["deq_bf16"]
    plain = qb.quantize(torch.from_numpy(x).cuda(), qb.get_codebook("nf4"), 64)
    assert h16(plain.constants) == meta["plain_constants"]


def test_near_midpoint_fallback_and_subnormal_blocks(oracle, qb, cuda):
    """Values within a few ulp of every decision boundary (the fp64 re-check
    path) and blocks whose absmax is subnormal."""
    cb = oracle.get_codebook("nf4")
    mids = cb.midpoints()
    rng = np.random.default_rng(3)
    blocks = []
    for b in range(400):
        c = np.float32(rng.uniform(0.1, 10.0))
        vals = [c]
        while len(vals) < 64:
            m = mids[rng.integers(mids.size)]
            k = rng.integers(-4, 5)
            v = np.float32(m * float(c))
            v = np.nextafter(v, np.float32(np.inf) if k > 0 else np.float32(-np.inf)) if k else v
            for _ in range(abs(int(k)) - 1):
                v = np.nextafter(v, np.float32(np.inf) if k > 0 else np.float32(-np.inf))
            vals.append(np.float32(v))
        blocks.append(vals)
    x = np.array(blocks, dtype=np.float32).reshape(-1)
    x[:64] = (rng.standard_normal(64) * 1e-40).astype(np.float32)  # subnormal absmax
    x[64:128] = np.float32(1e-45) * rng.integers(-3, 4, size=64).astype(np.float32)
    ref = oracle.quantize(x.astype(np.float64), cb, 64, double_quant=True)
    q = qb.quantize(x, qb.get_codebook("nf4"), 64, double_quant=True)
    assert np.array_equal(q.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(q.dq.codes.cpu().numpy(), ref.dq.codes)
    assert np.array_equal(q.dq.c1.cpu().numpy(), ref.dq.c1)
    assert np.array_equal(qb.dequantize(q).cpu().numpy(), oracle.dequantize(ref))


@pytest.mark.parametrize("dtype", ["bf16", "f64"])
def test_input_dtypes_match_oracle(dtype, oracle, qb, cuda):
    rng = np.random.default_rng(9)
    x32 = (rng.standard_normal((96, 640)) * np.exp(rng.uniform(-5, 5, size=(96, 1)))).astype(np.float32)
    if dtype == "bf16":
        xt = torch.from_numpy(x32).to(torch.bfloat16)
        x64 = xt.float().numpy().astype(np.float64)
    else:
        x64 = x32.astype(np.float64) * (1 + 1e-9 * rng.standard_normal(x32.shape))
        xt = torch.from_numpy(x64)
    ref = oracle.quantize(x64, oracle.get_codebook("nf4"), 64, double_quant=True)
    q = qb.quantize(xt.cuda(), qb.get_codebook("nf4"), 64, double_quant=True)
    assert np.array_equal(q.codes.cpu().numpy(), ref.codes)
    assert np.array_equal(q.dq.codes.cpu().numpy(), ref.dq.codes)
    assert q.dq.mu.item() == ref.dq.mu
    assert np.array_equal(qb.dequantize(q).cpu().numpy(), oracle.dequantize(ref))


def test_large_shape_properties(qb, cuda):
    """65B-layer shape (22016 x 8192): round-trip properties that do not need
    the oracle -- idempotence, zeros preserved, error bound, bits/param."""
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(22016, 8192, device="cuda", generator=g) * 0.02
    x[0, :128] = 0.0
    cb = qb.get_codebook("nf4")
    q = qb.quantize(x, cb, 64, double_quant=True)
    deq = qb.dequantize(q, torch.float32)
    assert torch.all(deq[0, :128] == 0)
    q2 = qb.quantize(deq, cb, 64)
    assert torch.equal(q2.codes, q.codes)
    assert torch.equal(qb.dequantize(q2, torch.float32), deq)
    c = q.block_constants().repeat_interleave(64).view_as(x)
    plain = qb.quantize(x, cb, 64)
    c0 = plain.constants.repeat_interleave(64).view_as(x)
    bound = c0.double() * cb.max_gap / 2 + (c0.double() - c.double()).abs()
    assert bool(((x.double() - deq.double()).abs() <= bound * (1 + 1e-6) + 1e-12).all())
    nbytes = q.codes.numel() + q.dq.codes.numel() + 4 * q.dq.c1.numel()
    assert nbytes * 8 / x.numel() == qb.bits_per_param(4, 64, dq=(256, 8))


def test_errors_match_reference(qb, cuda):
    cb = qb.get_codebook("nf4")
    for dt in (torch.float32, torch.float64, torch.bfloat16):
        x = torch.ones(1000, dtype=dt)
        x[517] = float("inf")
        with pytest.raises(ValueError, match="flat index 517"):
            qb.quantize(x, cb)
        x[517] = 1.0
        x[700] = float("nan")
        x[999] = float("nan")
        with pytest.raises(ValueError, match="flat index 700"):
            qb.quantize(x, cb, blocksize=48)
    with pytest.raises(ValueError, match="empty"):
        qb.quantize(np.array([], dtype=np.float32), cb)
    with pytest.raises(ValueError, match="blocksize"):
        qb.quantize(np.ones(4), cb, blocksize=0)
    q = qb.quantize(np.random.default_rng(0).normal(size=128), cb, 64)
    q.constants = q.constants[:1]
    with pytest.raises(qb.CorruptDataError, match="constants"):
        qb.dequantize(q)


def test_fp8_grid_and_dq_cases(golden, golden_meta, qb, cuda):
    assert np.array_equal(qb.decode_fp8(np.arange(256, dtype=np.uint8)).cpu().numpy(), golden["fp8/decode"])
    assert np.array_equal(qb.encode_fp8(golden["fp8/probe"]).cpu().numpy(), golden["fp8/probe_codes"])
    for i, _n in enumerate(golden_meta["dq_cases"]):
        dq = qb.dq_compress(golden[f"dq/{i}/c"], 256)
        assert dq.mu.item() == golden[f"dq/{i}/mu"][0], i
        assert np.array_equal(dq.c1.cpu().numpy(), golden[f"dq/{i}/c1"]), i
        assert np.array_equal(dq.codes.cpu().numpy(), golden[f"dq/{i}/codes"]), i
        assert np.array_equal(qb.dq_decompress(dq).cpu().numpy(), golden[f"dq/{i}/rec"]), i
    e5m2 = qb.Fp8Spec(5, 2, 15)
    vals, _ = e5m2.grid()
    assert np.array_equal(qb.decode_fp8(qb.encode_fp8(vals, e5m2), e5m2).cpu().numpy(), vals)
    with pytest.raises(ValueError):
        qb.dq_compress(np.array([1.0, -0.5], dtype=np.float32))


def test_dq_mean_order_random(oracle, qb, cuda):
    """numpy-order fp64 mean on adversarial magnitudes, several chunk counts."""
    rng = np.random.default_rng(21)
    for n in (1, 7, 129, 1031, 5000, 8191, 8192, 8193, 3 * 8192 + 1000, 100_000):
        c = np.abs(rng.standard_normal(n) * np.exp(rng.uniform(-40, 40, size=n))).astype(np.float32)
        ref = oracle.dq_compress(c, 256)
        dq = qb.dq_compress(c, 256)
        assert dq.mu.item() == ref.mu, n
        assert np.array_equal(dq.codes.cpu().numpy(), ref.codes), n
        assert np.array_equal(dq.c1.cpu().numpy(), ref.c1), n


def test_pack_unpack(qb, cuda):
    assert qb.pack_codes(np.array([0xA, 0x3]), 4).cpu().tolist() == [0x3A]
    assert qb.pack_codes(np.array([1, 2, 3]), 4).cpu().tolist() == [0x21, 0x03]
    codes = np.random.default_rng(0).integers(0, 16, size=10001)
    packed = qb.pack_codes(codes, 4)
    assert packed.numel() == 5001
    assert np.array_equal(qb.unpack_codes(packed, 4, 10001).cpu().numpy(), codes)
    with pytest.raises(ValueError, match="out of range"):
        qb.pack_codes(np.array([16]), 4)
    with pytest.raises(ValueError, match="shorter"):
        qb.unpack_codes(np.array([0x21], dtype=np.uint8), 4, 3)


@pytest.mark.parametrize("dq", [False, True])
def test_dequant_bf16_ragged_and_misaligned(dq, oracle, qb, cuda):
    """bf16 dequant (the two-lanes-per-block STG.256 kernel, and the staged
    kernel it falls back to for a 16B- but not 32B-aligned output) equals
    bf16(f32(dequantize)) of the oracle at ragged sizes."""
    from paper_2305_14314_b200 import _native
    cb = qb.get_codebook("nf4")
    rng = np.random.default_rng(7)
    for n in (1, 31, 63, 64, 65, 1000, 64 * 17 + 5, 64 * 1000 + 33, 64 * 4099):
        x = (rng.standard_normal(n) * rng.uniform(0.01, 3)).astype(np.float32)
        q = qb.quantize(torch.from_numpy(x).cuda(), cb, 64, double_quant=dq)
        ref = oracle.dequantize(oracle.quantize(x, oracle.get_codebook("nf4"), 64, double_quant=dq))
        want = torch.from_numpy(ref.astype(np.float32)).to(torch.bfloat16)
        assert torch.equal(qb.dequantize(q, torch.bfloat16).cpu(), want), n
        # misaligned destination (offset 8 elements = 16 B): staged kernel
        buf = torch.empty(n + 8, dtype=torch.bfloat16, device="cuda")
        dst = buf[8:]
        d = q.dq
        spec = (d.spec if dq else qb.Fp8Spec()).to_c()
        rc = _native.lib().qlrt_dequantize4(
            _native.ptr(q.codes), n, 64, q.codebook.to_c(),
            None if dq else _native.ptr(q.constants),
            _native.ptr(d.codes) if dq else None, _native.ptr(d.c1) if dq else None,
            _native.ptr(d.mu) if dq else None, 256, spec, _native.ptr(dst), _native.BF16, _native.stream_ptr())
        assert rc == 0
        torch.cuda.synchronize()
        assert torch.equal(dst.cpu(), want), ("misaligned", n)


@pytest.mark.gpu
@pytest.mark.parametrize("spec_args", [(4, 3, 7), (5, 2, 15)])
def test_fp8_encode_midpoints_vs_oracle(spec_args, oracle, qb, cuda):
    """encode_fp8 on every grid midpoint and its +-1..2 ulp neighbours, the grid
    itself, the subnormal range and random magnitudes: bit-exact vs the oracle."""
    spec = qb.Fp8Spec(*spec_args)
    ospec = oracle.Fp8Spec(*spec_args)
    vals, _ = spec.grid()
    v = np.unique(np.abs(np.asarray(vals, dtype=np.float64)))
    mids = (v[1:] + v[:-1]) / 2
    probes = [v, mids]
    for k in (1, 2):
        probes += [np.nextafter(mids, np.inf) if k == 1 else np.nextafter(np.nextafter(mids, np.inf), np.inf),
                   np.nextafter(mids, -np.inf) if k == 1 else np.nextafter(np.nextafter(mids, -np.inf), -np.inf)]
    rng = np.random.default_rng(7)
    probes.append(np.exp(rng.uniform(np.log(v[1] / 4), np.log(v[-1] * 1.5), 20000)))
    x = np.concatenate(probes)
    x = np.concatenate([x, -x, [0.0, -0.0]])
    got = qb.encode_fp8(x, spec).cpu().numpy()
    assert np.array_equal(got, oracle.encode_fp8(x, ospec))


@pytest.mark.parametrize("name", ["nf4", "fp4-e2m1", "fp4-e3m0", "int4", "nf-eq4"])
def test_stream_quantize_all_4bit_codebooks(name, oracle, qb, cuda):
    """The streaming phase-A kernel (fp32, blocksize 64, whole blocks) with its
    single-lookup private bin table, for every 4-bit codebook: random values
    and values within a few ulp of every midpoint (the fp64 re-decision)
    match the oracle bit for bit; DQ over a partial 8192-chunk as well."""
    cbo = oracle.get_codebook(name)
    mids = cbo.midpoints()
    rng = np.random.default_rng(len(name))
    blocks = []
    for b in range(300):
        c = np.float32(rng.uniform(0.01, 20.0))
        vals = [c if b % 2 else -c]
        while len(vals) < 64:
            if rng.random() < 0.5:
                vals.append(np.float32(rng.uniform(-1, 1) * float(c)))
                continue
            m = mids[rng.integers(mids.size)]
            v = np.float32(m * float(c))
            for _ in range(int(rng.integers(0, 4))):
                v = np.nextafter(v, np.float32(np.inf) if rng.random() < 0.5 else np.float32(-np.inf))
            vals.append(np.float32(v))
        blocks.append(vals)
    x = np.concatenate([np.array(blocks, dtype=np.float32).reshape(-1),
                        rng.standard_normal(64 * 5000).astype(np.float32)])
    ref = oracle.quantize(x.astype(np.float64), cbo, 64, double_quant=True)
    q = qb.quantize(torch.from_numpy(x).cuda(), qb.get_codebook(name), 64, double_quant=True)
    assert np.array_equal(q.codes.cpu().numpy(), ref.codes)
    assert q.dq.mu.item() == ref.dq.mu
    assert np.array_equal(q.dq.codes.cpu().numpy(), ref.dq.codes)
    assert np.array_equal(q.dq.c1.cpu().numpy(), ref.dq.c1)
