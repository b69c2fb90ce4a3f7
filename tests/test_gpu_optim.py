"""GPU parity: bit-exact fp32 Adam, clip_global_norm, paged == plain."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_adam_bitexact_vs_reference(golden, qb, cuda):
    p = torch.from_numpy(golden["adam/p0"].copy()).cuda()
    shadow = torch.empty_like(p, dtype=torch.bfloat16)
    opt = qb.AdamOptimizer({"p": p}, qb.TrainConfig(learning_rate=0.01), qb.PlainMomentStore(), {"p": shadow})
    for t in range(5):
        opt.step({"p": torch.from_numpy(golden[f"adam/g{t}"]).cuda()})
        assert np.array_equal(p.cpu().numpy(), golden[f"adam/p{t + 1}"]), t
    assert torch.equal(shadow, p.bfloat16())


def test_adam_hand_computed(qb, cuda):
    w = torch.tensor([1.0], device="cuda")
    opt = qb.AdamOptimizer({"w": w}, qb.TrainConfig(learning_rate=0.1), qb.PlainMomentStore())
    opt.step({"w": torch.tensor([0.5], device="cuda")})
    assert w.item() == pytest.approx(1.0 - 0.1 * (0.5 / (0.5 + 1e-8)), abs=1e-6)


def test_clip_global_norm(golden, golden_meta, qb, cuda):
    grads = {"a": torch.from_numpy(golden["clip/a"].copy()).cuda(),
             "b": torch.from_numpy(golden["clip/b"].copy()).cuda()}
    norm = qb.clip_global_norm(grads, ["a", "b"], 0.3)
    assert norm == pytest.approx(golden_meta["clip_norm"], rel=1e-15)
    assert np.array_equal(grads["a"].cpu().numpy(), golden["clip/a_out"])
    assert np.array_equal(grads["b"].cpu().numpy(), golden["clip/b_out"])
    g = {"a": torch.tensor([0.1, -0.2], device="cuda")}
    assert qb.clip_global_norm(g, ["a"], 1.0) == pytest.approx(np.hypot(0.1, 0.2), rel=1e-7)
    assert torch.equal(g["a"], torch.tensor([0.1, -0.2], device="cuda"))


@pytest.mark.parametrize("budget_slabs", [1, 2, 16])
def test_paged_equals_plain(budget_slabs, qb, cuda):
    """The reference's transparency property (tests/test_training.py:325-350)."""
    rng = np.random.default_rng(1)
    shapes = {"l1": (4096, 64), "l2": (64, 11008), "s": (3,)}
    init = {k: rng.standard_normal(s).astype(np.float32) for k, s in shapes.items()}
    grads_seq = [{k: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).cuda() for k, s in shapes.items()}
                 for _ in range(4)]
    results = []
    for paged in (False, True):
        params = {k: torch.from_numpy(v.copy()).cuda() for k, v in init.items()}
        if paged:
            slab = 2 * max(int(np.prod(s)) for s in shapes.values()) * 4
            pb = 2 << 20
            pager = qb.pager_open(qb.PagerConfig(budget_bytes=budget_slabs * ((slab + pb - 1) // pb) * pb, page_bytes=pb))
            store = qb.PagedMomentStore(pager)
        else:
            store = qb.PlainMomentStore()
        opt = qb.AdamOptimizer(params, qb.TrainConfig(learning_rate=1e-3), store)
        for g in grads_seq:
            gg = {k: v.clone() for k, v in g.items()}
            qb.clip_global_norm(gg, list(gg), 0.3)
            opt.step(gg)
        torch.cuda.synchronize()
        results.append({k: v.cpu().numpy() for k, v in params.items()})
        if paged:
            assert pager.faults > 0
            assert pager.peak_resident_bytes <= pager.config.budget_bytes
            if budget_slabs == 1:
                assert pager.evictions > 0
            pager.close()
    for k in shapes:
        assert np.array_equal(results[0][k], results[1][k]), k


@pytest.mark.parametrize("shape", [(1,), (7,), (8,), (100,), (128,), (129,), (16, 4), (4096, 64), (64, 11008),
                                   (333, 37)])
def test_clip_norm_in_numpy_pairwise_order(shape, qb, cuda):
    """clip_global_norm's sum of squares follows numpy's pairwise order per
    tensor (training.py:404-406): the norm is bit-identical to the
    reference's for every size, so the f32 clip scale is too."""
    rng = np.random.default_rng(sum(shape))
    gs = {"a": (rng.standard_normal(shape) * 3).astype(np.float32),
          "b": (rng.standard_normal((5, 3)) * 1e-3).astype(np.float32)}
    want = 0.0
    for name in ("a", "b"):
        want += float(np.sum(np.square(gs[name], dtype=np.float64)))
    got = qb.training.pairwise_sumsq({k: torch.from_numpy(v).cuda() for k, v in gs.items()}, ["a", "b"])
    assert float(got.item()) == want
    dev = {k: torch.from_numpy(v.copy()).cuda() for k, v in gs.items()}
    norm = qb.clip_global_norm(dev, ["a", "b"], 0.3)
    assert norm == math.sqrt(want)
    scale = np.float32(0.3 / norm)
    for k in gs:
        assert np.array_equal(dev[k].cpu().numpy(), gs[k] * scale)


@pytest.mark.parametrize("n,off", [(1, 0), (7, 1), (4096, 0), (1_000_003, 3), (40_000_000, 2)])
def test_fixed_order_sumsq(n, off, qb, cuda):
    """qlrt_sumsq_f64 (the harness's clip norm): fp64 sum of squares of a
    float32 vector, also from an unaligned start; deterministic run to run."""
    from paper_2305_14314_b200.training import global_sumsq
    g = torch.Generator(device="cuda").manual_seed(n)
    base = torch.randn(n + off, device="cuda", generator=g)
    v = base[off:]
    got = float(global_sumsq({"v": v}, ["v"]).item())
    want = float((v.double() ** 2).sum().item())
    assert got == pytest.approx(want, rel=1e-12)
    assert got == float(global_sumsq({"v": v}, ["v"]).item())
