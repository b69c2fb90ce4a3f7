"""The LLaMA-shaped QLoRA harness (C3/C5 measurement vehicle): adapter
gradients through the fused NF4 kernels match a float32 PyTorch autograd
reference of the same decoder (W = bf16(dequantize)), the fused clip + Adam
step matches the reference update order, and a CUDA-graph replay of the
whole step equals eager execution."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

# a tiny decoder whose shapes take the grouped q|k|v / gate|up path
GROUPED_TINY = {"hidden": 512, "ffn": 1024, "rank": 64}


def _reference_grads(model, tokens, targets):
    """fp32 autograd through the same decoder; returns loss and d/d(l1, l2)."""
    import paper_2305_14314_b200 as qb
    from paper_2305_14314_b200.llama import PROJS, rope_reference
    cfg = model.cfg
    b, s = tokens.shape
    nh, d = cfg.n_heads, cfg.hidden // cfg.n_heads
    leaves = {n: t.detach().clone().float().requires_grad_(True) for n, t in model.params.items()}
    ws = {}
    for li, lay in enumerate(model.layers):
        for pj in PROJS:
            ws[(li, pj)] = qb.dequantize(lay[pj].base, torch.float32).to(torch.bfloat16).float()
    sc = cfg.alpha / cfg.rank

    def lin(x, li, pj):
        l1 = leaves[f"{li}.{pj}.l1"].to(torch.bfloat16).float()
        l2 = leaves[f"{li}.{pj}.l2"].to(torch.bfloat16).float()
        return x @ ws[(li, pj)] + sc * (x @ l1) @ l2

    def rms(x):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.rms_eps)

    x = F.embedding(tokens, model.embed.float())
    cs = model.cos_sin[:s]
    for li in range(cfg.n_layers):
        hn = rms(x)
        q = rope_reference(lin(hn, li, "q").view(b, s, nh, d), cs).transpose(1, 2)
        k = rope_reference(lin(hn, li, "k").view(b, s, nh, d), cs).transpose(1, 2)
        v = lin(hn, li, "v").view(b, s, nh, d).transpose(1, 2)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(b, s, cfg.hidden)
        x = x + lin(a, li, "o")
        hn = rms(x)
        x = x + lin(F.silu(lin(hn, li, "gate")) * lin(hn, li, "up"), li, "down")
    logits = rms(x).reshape(b * s, -1) @ model.lm_head.float()
    loss = F.cross_entropy(logits, targets.reshape(-1))
    loss.backward()
    return loss.item(), {n: t.grad for n, t in leaves.items()}


def test_glue_kernels_match_torch(cuda):
    """Fused RMSNorm / SwiGLU / RoPE forward and backward vs PyTorch fp32."""
    from paper_2305_14314_b200.llama import _RMSNormFn, _RoPEFn, _SwiGLUFn, rope_reference
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(6, 5, 256, device="cuda", generator=g).bfloat16().requires_grad_(True)
    y = _RMSNormFn.apply(x, 1e-6)
    xr = x.detach().float().requires_grad_(True)
    yr = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-6)
    dy = torch.randn(y.shape, device="cuda", generator=g).bfloat16()
    y.backward(dy)
    yr.backward(dy.float())
    assert (y.float() - yr).abs().max() <= 2e-2 * yr.abs().max()
    assert (x.grad.float() - xr.grad).abs().max() <= 2e-2 * xr.grad.abs().max()
    a = torch.randn(1000, 64, device="cuda", generator=g).bfloat16().requires_grad_(True)
    b = torch.randn(1000, 64, device="cuda", generator=g).bfloat16().requires_grad_(True)
    o = _SwiGLUFn.apply(a, b)
    ar, br = a.detach().float().requires_grad_(True), b.detach().float().requires_grad_(True)
    orf = F.silu(ar) * br
    do = torch.randn(o.shape, device="cuda", generator=g).bfloat16()
    o.backward(do)
    orf.backward(do.float())
    assert (o.float() - orf).abs().max() <= 2e-2 * orf.abs().max()
    assert (a.grad.float() - ar.grad).abs().max() <= 2e-2 * ar.grad.abs().max()
    assert (b.grad.float() - br.grad).abs().max() <= 2e-2 * br.grad.abs().max()
    t = torch.randn(2, 16, 4, 64, device="cuda", generator=g).bfloat16().requires_grad_(True)
    ang = torch.outer(torch.arange(16, device="cuda").float(), 1.0 / (10000 ** (torch.arange(0, 64, 2, device="cuda").float() / 64)))
    cs = torch.stack((torch.cos(ang), torch.sin(ang)), dim=-1).contiguous()
    r = _RoPEFn.apply(t, cs)
    tr = t.detach().float().requires_grad_(True)
    rr = rope_reference(tr, cs)
    dr = torch.randn(r.shape, device="cuda", generator=g).bfloat16()
    r.backward(dr)
    rr.backward(dr.float())
    assert (r.float() - rr).abs().max() <= 2e-2 * rr.abs().max()
    assert (t.grad.float() - tr.grad).abs().max() <= 2e-2 * tr.grad.abs().max()
    # the grouped-projection glue: RoPE / copy over concatenated q | k | v
    # rows, SwiGLU over concatenated gate | up rows (forward and backward)
    from paper_2305_14314_b200._native import lib, ptr, stream_ptr
    b_, s_, nh, d = 2, 16, 4, 64
    h = nh * d
    ycat = torch.randn(b_ * s_, 3 * h, device="cuda", generator=g).bfloat16()
    q, k, v = (torch.empty(b_, s_, nh, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    assert lib().qlrt_rope_qkv_fwd(ptr(ycat), ptr(q), ptr(k), ptr(v), ptr(cs), b_ * s_, nh, d, s_, stream_ptr()) == 0
    yv = ycat.float().view(b_, s_, 3, nh, d)
    for got, want in ((q, rope_reference(yv[:, :, 0], cs)), (k, rope_reference(yv[:, :, 1], cs)), (v, yv[:, :, 2])):
        assert (got.float() - want).abs().max() <= 2e-2 * want.abs().max()
    dq, dk, dv = (torch.randn(b_, s_, nh, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    dycat = torch.empty(b_ * s_, 3 * h, device="cuda", dtype=torch.bfloat16)
    assert lib().qlrt_rope_qkv_bwd(ptr(dq), ptr(dk), ptr(dv), ptr(dycat), ptr(cs), b_ * s_, nh, d, s_,
                                   stream_ptr()) == 0
    inv = torch.stack((cs[..., 0], -cs[..., 1]), dim=-1)  # the inverse rotation
    dv_ = dycat.float().view(b_, s_, 3, nh, d)
    for got, want in ((dv_[:, :, 0], rope_reference(dq.float(), inv)), (dv_[:, :, 1], rope_reference(dk.float(), inv)),
                      (dv_[:, :, 2], dv.float())):
        assert (got - want).abs().max() <= 2e-2 * want.abs().max()
    gu = torch.randn(300, 2 * 64, device="cuda", generator=g).bfloat16()
    out = torch.empty(300, 64, device="cuda", dtype=torch.bfloat16)
    assert lib().qlrt_swiglu_cat_fwd(ptr(gu), ptr(out), 300, 64, stream_ptr()) == 0
    gr_, ur_ = gu.float()[:, :64].requires_grad_(True), gu.float()[:, 64:].requires_grad_(True)
    orf = F.silu(gr_) * ur_
    assert (out.float() - orf).abs().max() <= 2e-2 * orf.abs().max()
    do = torch.randn(300, 64, device="cuda", generator=g).bfloat16()
    dgu = torch.empty_like(gu)
    assert lib().qlrt_swiglu_cat_bwd(ptr(gu), ptr(do), ptr(dgu), 300, 64, stream_ptr()) == 0
    orf.backward(do.float())
    assert (dgu.float()[:, :64] - gr_.grad).abs().max() <= 2e-2 * gr_.grad.abs().max()
    assert (dgu.float()[:, 64:] - ur_.grad).abs().max() <= 2e-2 * ur_.grad.abs().max()
    # residual add fused into the norm, forward and backward (both inputs)
    from paper_2305_14314_b200.llama import _AddRMSNormFn
    xa = torch.randn(7, 256, device="cuda", generator=g).bfloat16().requires_grad_(True)
    da = torch.randn(7, 256, device="cuda", generator=g).bfloat16().requires_grad_(True)
    sa, ya = _AddRMSNormFn.apply(xa, da, 1e-6)
    xr_, dr_ = xa.detach().float().requires_grad_(True), da.detach().float().requires_grad_(True)
    sr_ = xr_ + dr_
    yr_ = sr_ * torch.rsqrt(sr_.pow(2).mean(-1, keepdim=True) + 1e-6)
    gs, gy = (torch.randn(7, 256, device="cuda", generator=g).bfloat16() for _ in range(2))
    torch.autograd.backward([sa, ya], [gs, gy])
    torch.autograd.backward([sr_, yr_], [gs.float(), gy.float()])
    assert (ya.float() - yr_).abs().max() <= 2e-2 * yr_.abs().max()
    assert torch.equal(sa, (xa.detach() + da.detach()))
    for got, want in ((xa.grad, xr_.grad), (da.grad, dr_.grad)):
        assert (got.float() - want).abs().max() <= 2e-2 * want.abs().max()
    # cross entropy straight from bf16 logits vs torch's fp32 cross entropy
    from paper_2305_14314_b200.llama import _XentFn
    lg = (torch.randn(300, 1000, device="cuda", generator=g) * 3).bfloat16().requires_grad_(True)
    tg = torch.randint(0, 1000, (300,), device="cuda", generator=g)
    lo = _XentFn.apply(lg, tg)
    lr = lg.detach().float().requires_grad_(True)
    lor = F.cross_entropy(lr, tg)
    (2.5 * lo).backward()
    (2.5 * lor).backward()
    assert abs(lo.item() - lor.item()) <= 1e-5 * abs(lor.item())
    assert (lg.grad.float() - lr.grad).abs().max() <= 1e-2 * lr.grad.abs().max()


def _tiny(seed=0, cfg_kw=None, **model_kw):
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    cfg = LlamaConfig.tiny(**(cfg_kw or {}))
    m = LlamaQLoRA(cfg, seed=seed, **model_kw)
    # make the adapters live (lora_init leaves l2 = 0): nonzero l2, shadows refreshed
    g = torch.Generator(device="cuda").manual_seed(seed + 1)
    for n, p in m.params.items():
        if n.endswith(".l2"):
            p.copy_(torch.randn(p.shape, device="cuda", generator=g) * 0.05)
    m.shadow_flat.copy_(m.params_flat)
    tok = torch.randint(0, cfg.vocab, (2, cfg.seq), device="cuda", generator=g)
    tgt = torch.randint(0, cfg.vocab, (2, cfg.seq), device="cuda", generator=g)
    return m, tok, tgt


@pytest.mark.parametrize("grouped", [False, True])
def test_adapter_grads_match_fp32_reference(grouped, cuda):
    """Adapter gradients of the harness (per projection, or q | k | v and
    gate | up as grouped calls) against fp32 autograd of the same decoder."""
    kw = {} if not grouped else {"hidden": 512, "ffn": 1024, "rank": 64}
    m, tok, tgt = _tiny(cfg_kw=kw)
    assert m.grouped == grouped
    loss = m.loss(tok, tgt)
    loss.backward()
    torch.cuda.synchronize()
    ref_loss, ref = _reference_grads(m, tok, tgt)
    assert abs(loss.item() - ref_loss) <= 2e-2 * abs(ref_loss)
    got = torch.cat([m.gviews[n].flatten() for n in m.names]).double()
    want = torch.cat([ref[n].flatten() for n in m.names]).double()
    d = (got - want).abs()
    assert d.max() / want.abs().max() <= 5e-2, float(d.max() / want.abs().max())
    assert d.mean() / want.abs().mean() <= 2e-2, float(d.mean() / want.abs().mean())


def test_step_matches_reference_update_and_graph_replay(cuda):
    from paper_2305_14314_b200.training import global_sumsq
    m, tok, tgt = _tiny(3)
    p0 = m.params_flat.clone()
    m.set_step_constants()
    loss = m.train_step(tok, tgt)
    torch.cuda.synchronize()
    # reference: clip (fp64 norm, f32 scale) then Adam in the reference op order, float32
    g = m.bucket.flat.clone()
    norm = math.sqrt(float(global_sumsq({"g": g}, ["g"]).item()))
    c = m.train_cfg
    f = np.float32
    if norm > c.max_grad_norm:
        g = g * torch.tensor(float(f(c.max_grad_norm / norm)), device="cuda")
    full = lambda v: torch.full_like(g, float(f(v)))  # noqa: E731  (true IEEE division, not x * (1/s))
    mm = full(1 - c.adam_beta1) * g
    vv = full(1 - c.adam_beta2) * (g * g)
    step = (mm / full(1 - c.adam_beta1)) / (torch.sqrt(vv / full(1 - c.adam_beta2)) + full(c.adam_eps))
    want = p0 - full(c.learning_rate) * step
    assert torch.equal(m.params_flat, want)
    assert torch.equal(m.shadow_flat, m.params_flat.to(torch.bfloat16))
    assert torch.isfinite(loss)
    # whole-step CUDA graph: replaying it equals running it eagerly
    m2, tok2, tgt2 = _tiny(3)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        m2.set_step_constants()
        m2.train_step(tok2, tgt2)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        gl = m2.train_step(tok2, tgt2)
    m3, tok3, tgt3 = _tiny(3)
    m3.set_step_constants()
    m3.train_step(tok3, tgt3)
    for _ in range(2):
        m2.set_step_constants()
        graph.replay()
        m3.set_step_constants()
        el = m3.train_step(tok3, tgt3)
    torch.cuda.synchronize()
    assert torch.equal(m2.params_flat, m3.params_flat)
    assert torch.equal(gl, el)


@pytest.mark.parametrize("lag", [None, 1, 2])
def test_grad_groups_launch_as_backward_reaches_them(lag, cuda):
    """The overlapped reducer launches each layer group's all-reduce from
    inside the backward, last group first (before the backward returns); with
    deferred adapter gradients a layer's group launches once the backward is
    ``lag`` layers further, the rest when the backward lands."""
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    m = LlamaQLoRA(LlamaConfig.tiny(n_layers=4), seed=0, bucket_layers=1, defer_lag=lag)
    g = torch.Generator(device="cuda").manual_seed(0)
    tok = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    m._pending = [7] * 4
    m.reducer.reset()
    m.loss(tok, tok).backward()
    assert m.reducer.launched == [3, 2, 1, 0][: 4 - (lag or 0)]
    m._land_all()
    assert m.reducer.launched == [3, 2, 1, 0]


@pytest.mark.parametrize("lag", [1, 3])
def test_deferred_adapter_grads_equal_joined(lag, cuda):
    """QLRT_BWD_DEFER moves only the completion point of dl2 / dl1 (side
    stream, waited for ``lag`` layers later): loss and every adapter gradient
    bit-identical to joining inside each projection's backward."""
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    cfg = LlamaConfig.tiny(n_layers=4, hidden=512, ffn=1024, rank=64)
    a = LlamaQLoRA(cfg, seed=3, defer_lag=None)
    b = LlamaQLoRA(cfg, seed=3, defer_lag=lag)
    for mdl in (a, b):
        for n, p in mdl.params.items():
            if n.endswith(".l2"):
                p.copy_(torch.randn(p.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)) * 0.05)
        mdl.shadow_flat.copy_(mdl.params_flat)
    g = torch.Generator(device="cuda").manual_seed(1)
    tok = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    la = a.forward_backward(tok, tok)
    lb = b.forward_backward(tok, tok)
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    assert torch.equal(a.bucket.flat, b.bucket.flat)
    assert b._inflight == {} and b._ready_q == []


def _paged_pair(budget_layers, page_bytes, cfg_kw=None):
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    cfg = LlamaConfig.tiny(n_layers=4, **(cfg_kw or {}))
    plain = LlamaQLoRA(cfg, seed=5)
    span = plain.layer_spans[0][1]
    slab_pages = (2 * span * 4 + page_bytes - 1) // page_bytes
    paged = LlamaQLoRA(cfg, seed=5, optimizer="paged", pager_budget_bytes=budget_layers * slab_pages * page_bytes,
                       page_bytes=page_bytes)
    return plain, paged


@pytest.mark.parametrize("budget_layers,page_bytes,cfg_kw", [(1, 64 << 10, None), (2, 64 << 10, None),
                                                            (4, 2 << 20, None), (1, 1 << 20, GROUPED_TINY)])
def test_paged_adamw_equals_plain(budget_layers, page_bytes, cfg_kw, cuda):
    """PagedMomentStore transparency on the training path (pkg/tests/
    test_training.py:325-350): the paged harness -- moments in unified-memory
    pages under a budget below the total state, elevator order, look-ahead
    prefetch -- produces bit-identical parameters and moments to the plain one."""
    plain, paged = _paged_pair(budget_layers, page_bytes, cfg_kw)
    g = torch.Generator(device="cuda").manual_seed(2)
    tok = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    tgt = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    for _ in range(4):
        for mdl in (plain, paged):
            mdl.set_step_constants()
            mdl.train_step(tok, tgt)
    torch.cuda.synchronize()
    assert torch.equal(plain.params_flat, paged.params_flat)
    assert torch.equal(plain.shadow_flat, paged.shadow_flat)
    pm, pv = paged.moments()
    assert torch.equal(plain.m_flat, pm) and torch.equal(plain.v_flat, pv)
    pg = paged.pager
    assert pg.faults > 0 and pg.peak_resident_bytes <= pg.config.budget_bytes
    if budget_layers < 4:
        assert pg.evictions > 0 and pg.bytes_read > 0
    paged.close()


@pytest.mark.parametrize("cfg_kw", [{}, GROUPED_TINY], ids=["per-projection", "grouped"])
def test_checkpointed_layers_match(cfg_kw, cuda):
    """Gradient checkpointing recomputes each layer in the backward: same loss
    and adapter gradients as keeping the activations."""
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    cfg = LlamaConfig.tiny(n_layers=3, **cfg_kw)
    a = LlamaQLoRA(cfg, seed=9)
    b = LlamaQLoRA(cfg, seed=9, checkpoint=True)
    g = torch.Generator(device="cuda").manual_seed(1)
    for mdl in (a, b):
        for n, p in mdl.params.items():
            if n.endswith(".l2"):
                p.copy_(torch.randn(p.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)) * 0.05)
        mdl.shadow_flat.copy_(mdl.params_flat)
    tok = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    la = a.forward_backward(tok, tok)
    lb = b.forward_backward(tok, tok)
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    d = (a.bucket.flat - b.bucket.flat).abs().max() / a.bucket.flat.abs().max()
    assert float(d) <= 1e-6, float(d)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("grouped", ["0", "1"])
def test_dp_two_ranks_equal_one_rank_over_concatenated_batch(grouped, cuda, tmp_path):
    """Two data-parallel ranks (gloo, both on cuda:0), each on half of the
    batch: the all-reduced adapter gradients and the loss equal one rank's
    over the whole batch (tolerance: bf16 GEMMs see different M tilings)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    helper = os.path.join(os.path.dirname(__file__), "helpers", "dp_llama_worker.py")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   OUT=str(tmp_path / f"r{r}.pt"), GROUPED=grouped)
        procs.append(subprocess.Popen([sys.executable, helper], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    for p in procs:
        out, err = p.communicate(timeout=280)
        assert p.returncode == 0, err[-3000:]
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", OUT=str(tmp_path / "single.pt"), GROUPED=grouped)
    env.pop("MASTER_PORT", None)
    single = subprocess.run([sys.executable, helper], env=env, capture_output=True, text=True, timeout=280)
    assert single.returncode == 0, single.stderr[-3000:]
    r0, r1, one = (torch.load(tmp_path / f, weights_only=True) for f in ("r0.pt", "r1.pt", "single.pt"))
    assert torch.equal(r0["grads"], r1["grads"]) and torch.equal(r0["params"], r1["params"])
    loss_dp = (r0["loss"] + r1["loss"]) / 2
    assert abs(float(loss_dp - one["loss"])) <= 1e-3 * abs(float(one["loss"]))
    d = (r0["grads"] - one["grads"]).abs()
    assert float(d.max() / one["grads"].abs().max()) <= 2e-2
    assert float(d.mean() / one["grads"].abs().mean()) <= 1e-2
    assert json.loads(r0["launched"]) == [1, 0]


@pytest.mark.parametrize("lag", [None, 1])
def test_grouped_projections_match_separate(lag, cuda):
    """q | k | v and gate | up as grouped calls (QLinearGroup: shared-input
    adapter GEMMs, one fused grid per group, in-place RoPE / SwiGLU on the
    concatenated outputs) against the same model run projection by
    projection: same loss and adapter gradients within the bf16 tolerance."""
    kw = {"hidden": 512, "ffn": 1024, "rank": 64}
    a, tok, tgt = _tiny(4, cfg_kw=kw, grouped=False, defer_lag=lag)
    b, _, _ = _tiny(4, cfg_kw=kw, grouped=True, defer_lag=lag)
    assert b.grouped and not a.grouped
    la = a.forward_backward(tok, tgt)
    lb = b.forward_backward(tok, tgt)
    torch.cuda.synchronize()
    assert abs(la.item() - lb.item()) <= 1e-3 * abs(la.item())
    ga = torch.cat([a.gviews[n].flatten() for n in a.names]).double()
    gb = torch.cat([b.gviews[n].flatten() for n in b.names]).double()
    d = (ga - gb).abs()
    # (two bf16 pipelines through two layers; each also meets the fp32 bound
    # of test_adapter_grads_match_fp32_reference)
    assert d.max() / ga.abs().max() <= 5e-2, float(d.max() / ga.abs().max())
    assert d.mean() / ga.abs().mean() <= 2e-2, float(d.mean() / ga.abs().mean())


def test_paged_resident_step_captures_whole(cuda):
    """Paged moments under a budget that holds them: once resident the
    optimizer issues no migration (optimizer_resident()), so the whole train
    step -- paged Adam included -- replays from one CUDA graph, bit-identical
    to eager steps."""
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    cfg = LlamaConfig.tiny(n_layers=2)
    a = LlamaQLoRA(cfg, seed=6, optimizer="paged")
    b = LlamaQLoRA(cfg, seed=6, optimizer="paged")
    assert not a.optimizer_resident()  # nothing faulted in yet
    g = torch.Generator(device="cuda").manual_seed(3)
    tok = torch.randint(0, 512, (2, 64), device="cuda", generator=g)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        a.set_step_constants()
        a.train_step(tok, tok)
    torch.cuda.current_stream().wait_stream(s)
    b.set_step_constants()
    b.train_step(tok, tok)
    torch.cuda.synchronize()
    assert a.optimizer_resident()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        a.train_step(tok, tok)
    for _ in range(2):
        a.set_step_constants()
        graph.replay()
        b.set_step_constants()
        b.train_step(tok, tok)
    torch.cuda.synchronize()
    assert torch.equal(a.params_flat, b.params_flat)
    ma, va = a.moments()
    mb, vb = b.moments()
    assert torch.equal(ma, mb) and torch.equal(va, vb)
