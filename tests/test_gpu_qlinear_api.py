"""QLinear API surface beyond the single-adapter fused path (qlora.py:91-167):
several adapters per layer, dropout with a fixed mask (pkg/tests/test_qlora.py:
225-268) at M > 1 and on the batch-1 GEMV, and the bf16 operand copies
following the fp32 masters when AdamOptimizer updates them (no caller-side
shadows).  Tolerances as tests/test_gpu_linear.py (north star)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MAX_REL, MEAN_REL = 1e-2, 1e-3


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def assert_tol(got, ref, what):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    d = np.abs(got - ref)
    mx, mn = d.max() / np.abs(ref).max(), d.mean() / np.abs(ref).mean()
    assert mx <= MAX_REL and mn <= MEAN_REL, f"{what}: max-rel {mx:.3e} mean-rel {mn:.3e}"


def _base(oracle, qb, k, n, seed):
    rng = np.random.default_rng(seed)
    w = (0.02 * rng.standard_normal((k, n))).astype(np.float32)
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    wd = bf16_round(qb.dequantize(q, torch.float32).cpu().numpy()).astype(np.float64)
    return rng, q, wd


def _adapters(rng, qb, oracle, k, n, specs):
    ads, oads = [], []
    for r, alpha, p in specs:
        l1 = bf16_round(rng.standard_normal((k, r)) / np.sqrt(r))
        l2 = bf16_round(0.02 * rng.standard_normal((r, n)))
        ads.append(qb.LoraAdapter(r, alpha, torch.from_numpy(l1).cuda(), torch.from_numpy(l2).cuda(), dropout_p=p))
        oads.append(oracle.LoraAdapter(r, alpha, l1.astype(np.float64), l2.astype(np.float64)))
    return ads, oads


@pytest.mark.parametrize("m", [300, 1])
def test_multi_adapter_vs_oracle(m, oracle, qb, cuda):
    """Three adapters of ranks 16 / 64 / 12 (12 padded to 16 on the GPU) with
    different scalings: one concatenated augmented segment in the fused GEMM."""
    k, n = 512, 768
    rng, q, wd = _base(oracle, qb, k, n, 11)
    ads, oads = _adapters(rng, qb, oracle, k, n, [(16, 32.0, 0.0), (64, 16.0, 0.0), (12, 6.0, 0.0)])
    lin = qb.QLinear(q, ads)
    x = bf16_round(rng.standard_normal((m, k)))
    dy = bf16_round(rng.standard_normal((m, n)))
    y, cache = lin.forward(torch.from_numpy(x))
    dx, grads = lin.backward(torch.from_numpy(dy), cache)
    torch.cuda.synchronize()
    yr, c = oracle.qlinear_forward(wd, oads, x.astype(np.float64))
    dxr, gr = oracle.qlinear_backward(oads, dy.astype(np.float64), c)
    assert_tol(y.float().cpu().numpy(), bf16_round(yr), "y")
    assert_tol(dx.float().cpu().numpy(), bf16_round(dxr), "dx")
    assert set(grads) == set(gr)
    for key in gr:
        assert tuple(grads[key].shape) == gr[key].shape
        assert_tol(grads[key].cpu().numpy(), gr[key], key)


@pytest.mark.parametrize("m", [300, 1])
def test_dropout_fixed_mask_vs_oracle(m, oracle, qb, cuda):
    """Train-mode dropout with a numpy rng draws the reference's mask
    (qlora.py:137-143); with that mask held fixed the forward and every
    gradient match the oracle (test_qlora.py:246-268)."""
    k, n = 512, 640
    rng, q, wd = _base(oracle, qb, k, n, 7)
    ads, oads = _adapters(rng, qb, oracle, k, n, [(16, 32.0, 0.5)])
    lin = qb.QLinear(q, ads)
    x = bf16_round(rng.standard_normal((m, k)))
    dy = bf16_round(rng.standard_normal((m, n)))
    y, cache = lin.forward(torch.from_numpy(x), train=True, rng=np.random.default_rng(3))
    mask = cache["masks"][0].cpu().numpy()
    ref_mask = (np.random.default_rng(3).random((m, k)) >= 0.5).astype(np.float32) / np.float32(0.5)
    assert np.array_equal(mask, ref_mask)
    assert set(np.unique(mask)) <= {0.0, 2.0}
    dx, grads = lin.backward(torch.from_numpy(dy), cache)
    torch.cuda.synchronize()
    yr, c = oracle.qlinear_forward(wd, oads, x.astype(np.float64), masks=[mask.astype(np.float64)])
    dxr, gr = oracle.qlinear_backward(oads, dy.astype(np.float64), c)
    assert_tol(y.float().cpu().numpy(), bf16_round(yr), "y")
    assert_tol(dx.float().cpu().numpy(), bf16_round(dxr), "dx")
    assert_tol(grads["adapter0.l1"].cpu().numpy(), gr["adapter0.l1"], "dl1")
    assert_tol(grads["adapter0.l2"].cpu().numpy(), gr["adapter0.l2"], "dl2")
    # eval mode ignores dropout (test_qlora.py:232-238)
    y_eval, _ = lin.forward(torch.from_numpy(x), train=False)
    y_plain, _ = qb.QLinear(q, [qb.LoraAdapter(16, 32.0, ads[0].l1, ads[0].l2)]).forward(torch.from_numpy(x))
    assert torch.equal(y_eval, y_plain)
    with pytest.raises(ValueError, match="rng"):
        lin.forward(torch.from_numpy(x), train=True)


def test_adam_updates_reach_the_kernels(qb, cuda):
    """lora_init leaves l2 = 0; AdamOptimizer over lin.trainable() (no
    shadows) must move the adapter seen by forward and backward: after each
    step the layer equals a fresh layer built from the current masters."""
    rng = np.random.default_rng(0)
    k, n, r = 256, 384, 8
    q = qb.quantize(0.02 * rng.standard_normal((k, n)), qb.get_codebook("nf4"), 64, double_quant=True)
    lin = qb.QLinear(q, [qb.lora_init(k, n, r, 16.0, rng)])
    opt = qb.AdamOptimizer(lin.trainable(), qb.TrainConfig(learning_rate=1e-2), qb.PlainMomentStore())
    x = torch.from_numpy(rng.standard_normal((64, k)).astype(np.float32))
    dy = torch.from_numpy(rng.standard_normal((64, n)).astype(np.float32))
    y0, _ = lin.forward(x)
    for step in range(3):
        y, cache = lin.forward(x)
        _, grads = lin.backward(dy, cache)
        opt.step(grads)
        fresh = qb.QLinear(q, [qb.LoraAdapter(r, 16.0, lin.adapters[0].l1.clone(), lin.adapters[0].l2.clone())])
        y_now, c_now = lin.forward(x)
        y_fresh, c_fresh = fresh.forward(x)
        assert torch.equal(y_now, y_fresh), step
        assert torch.equal(lin.backward(dy, c_now)[1]["adapter0.l1"], fresh.backward(dy, c_fresh)[1]["adapter0.l1"])
    assert not torch.equal(y_now, y0)
    assert float(lin.adapters[0].l2.abs().max()) > 0


@pytest.mark.parametrize("k,n", [(4096, 11008), (1024, 704)])
def test_deferred_backward_equals_joined(k, n, qb, cuda):
    """QLinear.backward(defer=[...]) leaves dl2 / dl1 on the side stream
    (QLRT_BWD_DEFER); after side_join every output is bit-identical to the
    joined backward, and the inputs the side work reads are handed back."""
    g = torch.Generator(device="cuda").manual_seed(7)
    m, r = 512, 64
    w = torch.randn(k, n, device="cuda", generator=g) * 0.02
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    l1 = (torch.randn(k, r, device="cuda", generator=g) / 8).bfloat16().float()
    l2 = (torch.randn(r, n, device="cuda", generator=g) * 0.01).bfloat16().float()
    lin = qb.QLinear(q, [qb.LoraAdapter(r, 16.0, l1, l2)])
    x = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    dy = torch.randn(m, n, device="cuda", generator=g).bfloat16()
    y, cache = lin.forward(x)
    dx0, g0 = lin.backward(dy, cache)
    g0 = {kk: v.clone() for kk, v in g0.items()}
    keep: list = []
    dx1, g1 = lin.backward(dy, cache, defer=keep)
    qb.side_join()
    torch.cuda.synchronize()
    assert len(keep) == 6
    assert torch.equal(dx0, dx1)
    for kk in g0:
        assert torch.equal(g0[kk], g1[kk]), kk


@pytest.mark.parametrize("g,k,ng,m", [(3, 1024, 512, 300), (2, 512, 768, 256), (1, 256, 256, 128)])
def test_group_linear_vs_torch_fp32(g, k, ng, m, qb, cuda):
    """QLinearGroup (q | k | v, gate | up as one call): per member the same
    math as QLinear with one adapter (qlora.py:124-167), against a plain
    PyTorch fp32 statement over the same bf16 operands; dX sums the members."""
    gen = torch.Generator(device="cuda").manual_seed(g * 100 + k)
    r, alpha = 64, 16.0
    s = alpha / r
    bases = [qb.quantize(torch.randn(k, ng, device="cuda", generator=gen) * 0.02, qb.get_codebook("nf4"), 64,
                         double_quant=True) for _ in range(g)]
    wds = [qb.dequantize(b, torch.bfloat16).float() for b in bases]
    l1 = (torch.randn(k, g * r, device="cuda", generator=gen) / 8).bfloat16().float()
    l2 = (torch.randn(r, g * ng, device="cuda", generator=gen) * 0.05).bfloat16().float()
    grp = qb.QLinearGroup(bases, l1, l2, r, alpha)
    x = torch.randn(m, k, device="cuda", generator=gen).bfloat16()
    dy = torch.randn(m, g * ng, device="cuda", generator=gen).bfloat16()
    y, cache = grp.forward(x)
    dl1 = torch.empty(k, g * r, device="cuda")
    dl2 = torch.empty(r, g * ng, device="cuda")
    dx = grp.backward(dy, cache, dl1, dl2)
    torch.cuda.synchronize()
    torch.backends.cuda.matmul.allow_tf32 = False
    xf, dyf = x.float(), dy.float()
    dx_ref = torch.zeros(m, k, device="cuda")
    for i in range(g):
        a1, a2 = l1[:, i * r:(i + 1) * r], l2[:, i * ng:(i + 1) * ng]
        dyi = dyf[:, i * ng:(i + 1) * ng]
        t = xf @ a1
        y_ref = xf @ wds[i] + s * t @ a2
        dt = s * dyi @ a2.t()
        dx_ref += dyi @ wds[i].t() + dt @ a1.t()
        for got, ref, what in ((y[:, i * ng:(i + 1) * ng].float(), y_ref.bfloat16().float(), "y"),
                               (dl2[:, i * ng:(i + 1) * ng], s * t.t() @ dyi, "dl2"),
                               (dl1[:, i * r:(i + 1) * r], xf.t() @ dt, "dl1")):
            d = (got - ref).abs()
            assert (d.max() / ref.abs().max()).item() <= MAX_REL, (what, i)
            assert (d.mean() / ref.abs().mean()).item() <= MEAN_REL, (what, i)
    d = (dx.float() - dx_ref.bfloat16().float()).abs()
    assert (d.max() / dx_ref.abs().max()).item() <= MAX_REL
    assert (d.mean() / dx_ref.abs().mean()).item() <= MEAN_REL
