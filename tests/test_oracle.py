"""Pin the CPU oracle against golden vectors made by the real reference."""

from __future__ import annotations

import numpy as np
import pytest


def test_codebooks_bitexact(golden, golden_meta, oracle):
    for name in ("nf4", "fp4-e2m1", "fp4-e3m0", "int4", "nf-eq4"):
        cb = oracle.get_codebook(name)
        assert np.array_equal(cb.values, golden[f"cb/{name}/values"]), name
        assert np.array_equal(cb.midpoints(), golden[f"cb/{name}/mids"]), name
        assert cb.n_emitted == golden_meta[f"cb/{name}"]["n_emitted"]
        assert cb.zero_code == golden_meta[f"cb/{name}"]["zero_code"]


def test_nf4_hex_appendix_a(golden_meta):
    # SURVEY.md Appendix A, first and a middle value
    hexes = golden_meta["cb/nf4"]["values_hex"]
    assert hexes[0] == "-0x1.0000000000000p+0"
    assert hexes[8] == "0x1.45f602226d8dbp-4"
    assert hexes[7] == "0x0.0p+0"


def test_nf4_vs_appendix_e_file(oracle):
    # the paper's fp32 table (pkg/tests/data/nf4_reference.txt) to <= 1e-6
    paper = np.array([-1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
                      -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
                      0.07958029955625534, 0.16093020141124725, 0.24611230194568634,
                      0.33791524171829224, 0.44070982933044434, 0.5626170039176941,
                      0.7229568362236023, 1.0])
    assert np.max(np.abs(oracle.get_codebook("nf4").values - paper)) <= 1e-6


def test_fp8_grid(golden, oracle):
    assert np.array_equal(oracle.decode_fp8(np.arange(256)), golden["fp8/decode"])
    assert np.array_equal(oracle.encode_fp8(golden["fp8/probe"]), golden["fp8/probe_codes"])
    vals, codes = oracle.fp8_grid()
    assert vals.size == 255 and vals[-1] == 480.0 and vals[vals > 0][0] == 2.0 ** -9


def _case_q(oracle, golden, c):
    tag = c["tag"]
    x = golden[f"q/{tag}/x"]
    return oracle.quantize(x, oracle.get_codebook(c["codebook"]), c["blocksize"],
                           c["double_quant"], c["blocksize2"])


def test_quantize_cases(golden, golden_meta, oracle):
    for c in golden_meta["quant_cases"]:
        tag = c["tag"]
        q = _case_q(oracle, golden, c)
        assert np.array_equal(q.codes, golden[f"q/{tag}/codes"]), tag
        if c["double_quant"]:
            assert np.array_equal(q.dq.codes, golden[f"q/{tag}/dq_codes"]), tag
            assert np.array_equal(q.dq.c1, golden[f"q/{tag}/dq_c1"]), tag
            assert q.dq.mu == golden[f"q/{tag}/dq_mu"][0], tag
        else:
            assert np.array_equal(q.constants, golden[f"q/{tag}/constants"]), tag
        assert np.array_equal(oracle.dequantize(q), golden[f"q/{tag}/deq"]), tag


def test_dq_mean_order_emulation(golden, golden_meta, oracle):
    """The explicit buffered-pairwise order reproduces numpy's mean."""
    for i, _n in enumerate(golden_meta["dq_cases"]):
        c = golden[f"dq/{i}/c"]
        assert oracle.numpy_order_sum_f64(c) == golden[f"dq/{i}/sum64"][0]
        for emulate in (False, True):
            dq = oracle.dq_compress(c, 256, emulate_order=emulate)
            assert dq.mu == golden[f"dq/{i}/mu"][0]
            assert np.array_equal(dq.c1, golden[f"dq/{i}/c1"])
            assert np.array_equal(dq.codes, golden[f"dq/{i}/codes"])
            assert np.array_equal(oracle.dq_decompress(dq), golden[f"dq/{i}/rec"])


def test_dq_mean_order_random_live(oracle):
    """Also against live numpy on fresh adversarial data (same numpy)."""
    r = np.random.default_rng(5)
    for n in (7, 8, 127, 128, 129, 4096, 8191, 8192, 8193, 24577, 50000):
        c = np.abs(r.standard_normal(n) * np.exp(r.uniform(-40, 40, size=n))).astype(np.float32)
        assert oracle.numpy_order_sum_f64(c) == c.sum(dtype=np.float64), n


def test_qlinear_cases(golden, golden_meta, oracle):
    for i, c in enumerate(golden_meta["qlinear_cases"]):
        g = lambda k: golden[f"ql/{i}/{k}"]  # noqa: E731
        q = oracle.quantize(g("w"), oracle.get_codebook("nf4"), 64, True)
        assert np.array_equal(q.codes, g("codes"))
        w = oracle.dequantize(q).astype(np.float32)
        # bf16 rounding of the dense base, as in the golden generator
        u = w.view(np.uint32).astype(np.uint64)
        w = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)
        ad = oracle.LoraAdapter(c["rank"], c["alpha"], g("l1"), g("l2"))
        y, cache = oracle.qlinear_forward(w.astype(np.float64), [ad], g("x"))
        dx, grads = oracle.qlinear_backward([ad], g("dy"), cache)
        assert np.array_equal(y, g("y"))
        assert np.array_equal(dx, g("dx"))
        assert np.array_equal(grads["adapter0.l1"], g("dl1"))
        assert np.array_equal(grads["adapter0.l2"], g("dl2"))


def test_adam_and_clip(golden, golden_meta, oracle):
    p = golden["adam/p0"].copy()
    st = oracle.AdamState()
    cfg = oracle.TrainConfig(learning_rate=0.01)
    for t in range(5):
        oracle.adam_step({"p": p}, {"p": golden[f"adam/g{t}"]}, cfg, st)
        assert np.array_equal(p, golden[f"adam/p{t + 1}"]), t
    grads = {"a": golden["clip/a"].copy(), "b": golden["clip/b"].copy()}
    norm = oracle.clip_global_norm(grads, ["a", "b"], 0.3)
    assert norm == golden_meta["clip_norm"]
    assert np.array_equal(grads["a"], golden["clip/a_out"])
    assert np.array_equal(grads["b"], golden["clip/b_out"])


def test_errors(oracle):
    cb = oracle.get_codebook("nf4")
    x = np.ones(10)
    x[5] = np.nan
    with pytest.raises(ValueError, match="flat index 5"):
        oracle.quantize(x, cb)
    with pytest.raises(ValueError, match="empty"):
        oracle.quantize(np.array([]), cb)
    with pytest.raises(ValueError, match="blocksize"):
        oracle.quantize(np.ones(4), cb, blocksize=0)


def test_bits_per_param(oracle):
    assert oracle.bits_per_param(4, 64) == 4.5
    assert oracle.bits_per_param(4, 64, dq=(256, 8)) == 4.126953125
