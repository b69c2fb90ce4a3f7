"""The torch custom-op layer (torch.ops.qlrt_b200.*, csrc/torch_ops.cpp) over
the C ABI: schemas registered, Meta (fake-tensor) implementations give the
shapes on CPU, and on the GPU every op equals the ctypes-bound product path
bit for bit (and passes torch.library.opcheck's schema / fake checks)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

OPS = ("quantize4", "dq_compress", "dequantize4", "nf4_linear_fwd", "nf4_linear_bwd", "nf4_gemv", "adam_step")


def _ops():
    from paper_2305_14314_b200._native import load_torch_ops
    return load_torch_ops()


def test_ops_registered_with_meta_shapes():
    ops = _ops()
    for name in OPS:
        assert hasattr(ops, name), name
    meta = torch.device("meta")
    x = torch.empty(300, 512, dtype=torch.bfloat16, device=meta)
    codes = torch.empty(512 * 768 // 2, dtype=torch.uint8, device=meta)
    dqc = torch.empty(512 * 768 // 64, dtype=torch.uint8, device=meta)
    c1 = torch.empty(24, device=meta)
    mu = torch.empty(1, device=meta)
    l1 = torch.empty(512, 64, dtype=torch.bfloat16, device=meta)
    l2 = torch.empty(64, 768, dtype=torch.bfloat16, device=meta)
    vals = [0.0] * 16
    y, ts, consts = ops.nf4_linear_fwd(x, codes, dqc, c1, mu, 512, 768, 256, [4, 3, 7], vals, l1, l2, 0.25)
    assert y.shape == (300, 768) and y.dtype == torch.bfloat16 and ts.shape == (300, 128)
    dy = torch.empty(300, 768, dtype=torch.bfloat16, device=meta)
    dx, dl1, dl2 = ops.nf4_linear_bwd(dy, x, ts, consts, codes, dqc, c1, mu, 512, 768, 256, [4, 3, 7], vals, l1, l2,
                                      0.25)
    assert dx.shape == (300, 512) and dl1.shape == (512, 64) and dl2.shape == (64, 768) and dl1.dtype == torch.float32
    cb = torch.empty(1, dtype=torch.uint8)  # meta impl ignores the codebook bytes
    q, a, bad = ops.quantize4(torch.empty(1000, device=meta), cb, 64)
    assert q.shape == (16 * 64 // 2,) and a.shape == (16,) and bad.dtype == torch.int64
    out = ops.dequantize4(q, 1000, 64, cb, dqc, c1, mu, 256, [4, 3, 7], torch.bfloat16)
    assert out.shape == (1000,) and out.dtype == torch.bfloat16


@pytest.mark.gpu
def test_ops_equal_ctypes_path(qb, cuda):
    from paper_2305_14314_b200._native import codebook_blob
    ops = _ops()
    rng = np.random.default_rng(4)
    k, n, m, r = 512, 768, 300, 64
    w = torch.from_numpy((0.02 * rng.standard_normal((k, n))).astype(np.float32)).cuda()
    cb = qb.get_codebook("nf4")
    q = qb.quantize(w, cb, 64, double_quant=True)
    blob = codebook_blob(cb)
    codes, absmax, bad = ops.quantize4(w, blob, 64)
    assert torch.equal(codes, q.codes) and int(bad.item()) >= k * n  # no non-finite element
    mu, c1, dqc = ops.dq_compress(absmax, 256, [4, 3, 7])
    assert torch.equal(mu, q.dq.mu.reshape(1)) and torch.equal(c1, q.dq.c1) and torch.equal(dqc, q.dq.codes)
    for dt in (torch.float32, torch.bfloat16):
        assert torch.equal(ops.dequantize4(codes, k * n, 64, blob, dqc, c1, mu, 256, [4, 3, 7], dt).view(k, n),
                           qb.dequantize(q, dt))
    l1 = torch.from_numpy(rng.standard_normal((k, r)).astype(np.float32) / 8).cuda()
    l2 = torch.from_numpy(0.02 * rng.standard_normal((r, n)).astype(np.float32)).cuda()
    lin = qb.QLinear(q, [qb.LoraAdapter(r, 16.0, l1, l2)])
    x = torch.randn(m, k, device="cuda").bfloat16()
    dy = torch.randn(m, n, device="cuda").bfloat16()
    y_ref, cache = lin.forward(x)
    dx_ref, g_ref = lin.backward(dy, cache)
    vals = [float(v) for v in cb.values]
    args = (codes, dqc, c1, mu, k, n, 256, [4, 3, 7], vals, l1.bfloat16(), l2.bfloat16(), 0.25)
    y, ts, consts = ops.nf4_linear_fwd(x, *args)
    dx, dl1, dl2 = ops.nf4_linear_bwd(dy, x, ts, consts, *args)
    assert torch.equal(y, y_ref) and torch.equal(dx, dx_ref)
    assert torch.equal(dl1, g_ref["adapter0.l1"]) and torch.equal(dl2, g_ref["adapter0.l2"])
    yv = ops.nf4_gemv(x[:1], *args)
    assert torch.equal(yv, lin.forward(x[:1])[0])
    p = torch.randn(1000, device="cuda")
    p2, g = p.clone(), torch.randn(1000, device="cuda")
    mm, vv = torch.zeros_like(p), torch.zeros_like(p)
    consts_adam = qb.AdamOptimizer({"p": p2}, qb.TrainConfig(), qb.PlainMomentStore())
    consts_adam.t = 1
    ops.adam_step(p, g, mm, vv, *consts_adam.constants())
    consts_adam.t = 0
    consts_adam.step({"p": g})
    assert torch.equal(p, p2)
    torch.library.opcheck(ops.nf4_linear_fwd.default, (x,) + args,
                          test_utils=("test_schema", "test_faketensor"))
