"""Benchmark of the B200-native QLoRA hot path.

Headline (BASELINE.json metric "... QLoRA tokens/sec at 1/2/4/8 B200"):
config C3, the LLaMA-7B-shape QLoRA finetune step -- 32 layers, every linear
(q, k, v, o, gate, up, down) a frozen NF4 + DQ base with a LoRA adapter
r = 64 through the fused tcgen05 kernels, seq 512 x 4 sequences = 2048
tokens per GPU per step (weak scaling), forward + backward + adapter-gradient
all-reduce (NCCL, overlapped with the backward) + fused clip + bit-exact
AdamW, the whole step one CUDA graph.  value = whole-job tokens/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` with N > 1 and no torchrun environment re-launches itself under
``torch.distributed.run`` (one rank per GPU, NCCL); under torchrun it runs as
the rank it is.  Rank 0 prints one JSON line.  Besides the headline, rank 0
reports (N = 1) the other BASELINE configs as named extras: C1 (NF4 + DQ
quantize / dequantize GB/s), C2 (one linear fwd+bwd TFLOP/s), C4 (LLaMA-65B
layer sweep: fused fwd/bwd + LoRA TFLOP/s and batch-1 GEMV GB/s), C3 with the
paged AdamW, and at every N C5 (LLaMA-33B shapes, paged AdamW) tokens/s.

``--impl reference`` times the reference's own CPU implementation (qlrt,
installed offline into baseline/_ref; the oracle port if that is absent) on
the host cores: the C3 metric as a linear-only extrapolation, one linear
shape of the layer sampled per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NF4 dequant GB/s vs HBM peak; fused 4-bit GEMM TFLOPS; QLoRA tokens/sec at 1/2/4/8 B200"
C3_LAYERS, C3_H, C3_FFN, C3_TOKENS = 32, 4096, 11008, 2048
C3_SHAPES = (("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
             ("gate", 4096, 11008), ("up", 4096, 11008), ("down", 11008, 4096))
M_TOK, K_IN, N_OUT, RANK, ALPHA = 2048, 4096, 11008, 64, 16.0


def flops_fwd(m=M_TOK, k=K_IN, n=N_OUT, r=RANK):
    return 2 * m * k * n + 2 * m * k * r + 2 * m * r * n


def flops_bwd(m=M_TOK, k=K_IN, n=N_OUT, r=RANK):
    return 2 * m * n * k + 2 * m * n * r + 2 * r * m * n + 2 * k * m * r + 2 * m * r * k


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def traffic_of(key):
    """DRAM bytes per launch of a kernel from the committed ncu capture
    (profiles/roofline_traffic.json, dram__bytes_read.sum + write.sum)."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            return json.load(fh)[key]["dram_bytes"]
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks sampler (NVML during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle reasons sampled in-process through NVML every ~2 ms
    while the timed region runs."""

    REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.err = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def _run(self):
        nv, h = self.nv, self.h
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(get_r(h))))
            except Exception as e:  # pragma: no cover
                self.err = repr(e)
                return
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if hasattr(self, "t"):
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "error": self.err}
        reasons = set()
        for _, bits in self.samples:
            for bit, name in self.REASONS.items():
                if bits & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
# the reference's CPU implementation (reference arm + cpu_baseline legs)
# ---------------------------------------------------------------------------
class CpuReference:
    """qlrt's own QLinear / quantize / dequantize (pip-installed offline into
    baseline/_ref, kind "reference"), else the oracle port (kind "port"),
    float32 as the reference's low-precision mode, numpy's default BLAS
    threads (all host cores)."""

    def __init__(self):
        ref = os.path.join(ROOT, "baseline", "_ref")
        self.kind = "port"
        if os.path.isdir(os.path.join(ref, "qlrt")):
            sys.path.insert(0, ref)
            try:
                import qlrt.blockquant as bq
                import qlrt.codebooks as cbs
                import qlrt.qlora as ql
                self.bq, self.cbs, self.ql = bq, cbs, ql
                self.kind = "reference"
            except Exception:  # pragma: no cover
                self.kind = "port"
        if self.kind == "port":
            from oracle import qlrt_oracle as orc
            self.orc = orc
        self.cores = os.cpu_count()

    def quantize(self, w):
        if self.kind == "reference":
            return self.bq.quantize(w, self.cbs.get_codebook("nf4"), 64, double_quant=True)
        return self.orc.quantize(w, self.orc.get_codebook("nf4"), 64, double_quant=True)

    def dequantize(self, q):
        return (self.bq if self.kind == "reference" else self.orc).dequantize(q)

    def layer(self, q, l1, l2):
        if self.kind == "reference":
            return self.ql.QLinear(q, [self.ql.LoraAdapter(l1.shape[1], ALPHA, l1, l2)], dtype=np.float32)
        return (q, self.orc.LoraAdapter(l1.shape[1], ALPHA, l1, l2))

    def fwd_bwd(self, lin, x, dy):
        """One QLinear forward + backward (qlora.py:124-167): the base is
        dequantized inside every call, as the reference does."""
        if self.kind == "reference":
            y, cache = lin.forward(x)
            return lin.backward(dy, cache)
        q, ad = lin
        wd = self.orc.dequantize(q).astype(np.float32)
        y, cache = self.orc.qlinear_forward(wd, [ad], x, dtype=np.float32)
        return self.orc.qlinear_backward([ad], dy, cache, dtype=np.float32)


def _cpu_c3_layers(ref: CpuReference, tokens: int = C3_TOKENS):
    """The 7 linear shapes of one C3 layer as reference QLinear layers (NF4 +
    DQ base of N(0, 0.02) weights, LoRA r = 64 with live l2) and inputs."""
    rng = np.random.default_rng(0)
    out = []
    for name, k, n in C3_SHAPES:
        w = (0.02 * rng.standard_normal((k, n))).astype(np.float32)
        l1 = (rng.standard_normal((k, RANK)) / 8).astype(np.float32)
        l2 = (0.01 * rng.standard_normal((RANK, n))).astype(np.float32)
        x = rng.standard_normal((tokens, k)).astype(np.float32)
        dy = rng.standard_normal((tokens, n)).astype(np.float32)
        out.append((name, k, n, ref.layer(ref.quantize(w), l1, l2), x, dy))
    return out


def _c3_extrapolate(times: dict) -> float:
    """tokens/s of the C3 step from per-shape fwd+bwd seconds: 32 layers x the
    7 linears of a layer (linear-only: attention, norms and the optimizer are
    not counted, so this upper-bounds the CPU's tokens/s)."""
    return C3_TOKENS / (C3_LAYERS * sum(times.values()))


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    t_all = time.perf_counter()
    ref = CpuReference()
    layers = _cpu_c3_layers(ref)
    last: dict = {}
    vals = []
    # at least one full cycle of the 7 shapes: the extrapolation needs every one
    n_steps = max(args.warmup + args.steps, len(layers))
    for i in range(n_steps):
        name, k, n, lin, x, dy = layers[i % len(layers)]
        t0 = time.perf_counter()
        ref.fwd_bwd(lin, x, dy)
        last[name] = time.perf_counter() - t0
        if len(last) == len(layers) and i >= args.warmup:
            vals.append(_c3_extrapolate(last))
    value = statistics.median(vals) if vals else _c3_extrapolate(last)
    sample = (f"{ref.kind} QLinear fwd+bwd fp32 (NF4+DQ base dequantized per call, LoRA r=64), one of the 7 "
              f"linear shapes of a LLaMA-7B layer per step at the full 2048 tokens, tokens/s = 2048 / (32 layers x "
              f"sum of the latest per-shape times): linear-only extrapolation of the C3 step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": C3_TOKENS / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": c3_config(args.gpus),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": ref.cores, "kind": ref.kind,
                             "sample": sample},
            "per_shape_s": last,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


def c3_config(world: int) -> dict:
    return {"workload": "C3: LLaMA-7B-shape QLoRA finetune step (32 layers, h 4096, ffn 11008, 32 heads, vocab "
                        "32000; q,k,v,o,gate,up,down NF4+DQ frozen with LoRA r=64 alpha 16), seq 512 x 4 "
                        "sequences per GPU, data-parallel adapter-gradient all-reduce, fused clip + paged AdamW (moments in "
                        "unified-memory pages)",
            "tokens_per_gpu": C3_TOKENS, "seq_len": 512, "global_batch": 4 * world,
            "parallelism": f"dp{world}",
            "l2": "inputs larger than L2: every step streams 3.3 GB of NF4 weights (126 MB L2)"}


# ---------------------------------------------------------------------------
# the LLaMA QLoRA step (C3 / C5): our arm
# ---------------------------------------------------------------------------
def llama_step_bench(torch, dist, name, cfg, world, dev, steps, warmup, optimizer="plain", budget=None,
                     e2e_steps=0, count_launches=False, graph=True):
    """Build the model (random N(0, 0.02) weights quantized NF4 + DQ on the
    GPU), warm up eagerly, capture one step in a CUDA graph (the NCCL
    all-reduces of the overlapped reducer included), time ``steps`` replays
    with CUDA events on the launching stream; max over ranks."""
    from paper_2305_14314_b200.llama import LlamaQLoRA
    t0 = time.time()
    m = LlamaQLoRA(cfg, device=dev, seed=0, optimizer=optimizer, pager_budget_bytes=budget)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    rank = dist.get_rank() if world > 1 else 0
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    batch = C3_TOKENS // cfg.seq
    tok = torch.randint(0, cfg.vocab, (batch, cfg.seq), device=dev, generator=g)
    tgt = torch.randint(0, cfg.vocab, (batch, cfg.seq), device=dev, generator=g)
    paged = optimizer == "paged"
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            m.set_step_constants()
            m.train_step(tok, tgt)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    captured = False
    if graph and world > 1 and dist.get_backend() == "gloo":
        graph = False  # (gloo collectives are not capturable: the shared-GPU launcher check runs eager)
    # paged moments that all stay resident (the budget holds them): the
    # optimizer issues no migration, so it joins the captured step too
    opt_in_graph = m.optimizer_resident()
    if graph:
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                loss_g = m.train_step(tok, tgt) if opt_in_graph else m.forward_backward(tok, tgt)
            captured = True
        except Exception as e:  # pragma: no cover - reported, eager steps instead
            graph_err = repr(e)[:200]
            torch.cuda.synchronize()

    def one_step():
        m.set_step_constants()
        if captured:
            gr.replay()
            if not opt_in_graph:
                m.optimizer_step()
            return loss_g
        return m.train_step(tok, tgt)

    one_step()
    torch.cuda.synchronize()
    launches = None
    if count_launches and not os.environ.get("QLRT_NO_TORCH_PROFILER"):
        try:
            from torch.profiler import ProfilerActivity, profile
            # one eager step (the same launches the captured graph replays)
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                m.set_step_constants()
                m.train_step(tok, tgt)
                torch.cuda.synchronize()
            names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
            launches = sum(1 for n in names if "qlrt" in n)
        except Exception:
            launches = None
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(dev.index if dev.index is not None else 0) as clk:
        ev[0].record(stream)
        for _ in range(steps):
            loss = one_step()
        ev[1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([ev[0].elapsed_time(ev[1]) / steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    out = {"model": name, "layers": cfg.n_layers, "tokens_per_step_per_gpu": batch * cfg.seq,
           "ms_per_step": ms, "tokens_per_s": world * batch * cfg.seq / (ms / 1e3),
           "tflops_per_gpu": cfg.flops_per_token() * batch * cfg.seq / (ms / 1e3) / 1e12,
           "flops_per_token": cfg.flops_per_token(), "linear_params": cfg.linear_params,
           "lora_params": cfg.lora_params, "optimizer": optimizer, "build_s": build_s, "cuda_graph": captured,
           "optimizer_in_graph": captured and opt_in_graph,
           "max_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9, "loss": float(loss.item()),
           "clocks": clk.summary()}
    if graph and not captured:
        out["graph_error"] = graph_err
    if paged:
        pg = m.pager
        out["pager"] = {"budget_bytes": pg.config.budget_bytes, "state_bytes": sum(8 * n for _, n in m.layer_spans),
                        "page_bytes": pg.config.page_bytes, "faults": pg.faults, "evictions": pg.evictions,
                        "bytes_read": pg.bytes_read, "bytes_written": pg.bytes_written,
                        "peak_resident_bytes": pg.peak_resident_bytes}
    if launches is not None:
        out["gpu_launches_per_step"] = launches
    if e2e_steps:
        # through the public API (LlamaQLoRA.train_step, captured): each step's
        # tokens and targets copied in from pinned host memory, its loss read
        # back to pinned host memory, all inside the timed region
        tok_h = tok.cpu().pin_memory()
        tgt_h = tgt.cpu().pin_memory()
        loss_h = torch.empty(e2e_steps, dtype=torch.float32).pin_memory()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for i in range(e2e_steps):
            tok.copy_(tok_h, non_blocking=True)
            tgt.copy_(tgt_h, non_blocking=True)
            lo = one_step()
            loss_h[i: i + 1].copy_(lo.reshape(1), non_blocking=True)
        ev[1].record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([ev[0].elapsed_time(ev[1]) / e2e_steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        out["e2e"] = {"value": world * batch * cfg.seq / (e_ms / 1e3), "unit": "tokens/s",
                      "h2d_bytes_per_step": tok_h.numel() * 8 + tgt_h.numel() * 8, "d2h_bytes_per_step": 4,
                      "steps": e2e_steps, "ms_per_step": e_ms,
                      "note": "LlamaQLoRA.train_step (CUDA-graph captured) with tokens/targets copied from pinned "
                              "host memory and the loss read back every step"}
    m.close()
    del m
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# named extras (rank 0, N = 1): C1, C2, C4
# ---------------------------------------------------------------------------
def _timed(torch, stream, flush, fns, n=20):
    """CUDA graph of the launches replayed after an L2 flush; mean ms."""
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    g.replay()
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / n


def c2_linear(qb, torch, dev, flush, stream, world, dist, steps, warmup):
    """C2: one frozen NF4 linear 4096 -> 11008, LoRA r = 64, bf16 fwd + bwd on
    2048 tokens; device time per graph-captured step after an L2 flush, and e2e
    through QLinear.forward/backward with pinned host X, dY in and dX, dl1,
    dl2 out (copies double-buffered on side streams)."""
    g = torch.Generator(device=dev).manual_seed(1234)
    w = torch.randn(K_IN, N_OUT, device=dev, generator=torch.Generator(device=dev).manual_seed(0)) * 0.02
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    del w
    l1 = torch.randn(K_IN, RANK, device=dev, generator=g) / 8
    l2 = torch.randn(RANK, N_OUT, device=dev, generator=g) * 0.01
    lin = qb.QLinear(q, [qb.LoraAdapter(RANK, ALPHA, l1, l2)])
    x = torch.randn(M_TOK, K_IN, device=dev, generator=g).bfloat16()
    dy = torch.randn(M_TOK, N_OUT, device=dev, generator=g).bfloat16()
    for _ in range(warmup):
        c = lin.forward(x)[1]
        lin.backward(dy, c)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y_g, c_g = lin.forward(x)
        dx_g, grads_g = lin.backward(dy, c_g)
    graph.replay()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        starts[i].record(stream)
        graph.replay()
        ends[i].record(stream)
    torch.cuda.synchronize()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / steps
    step_flops = flops_fwd() + flops_bwd()
    out = {"tflops": step_flops / (ms / 1e3) / 1e12, "ms_per_step": ms, "flops_per_step": step_flops,
           "workload": "C2: frozen NF4 linear 4096->11008, LoRA r=64, bf16 fwd+bwd, 4x512 tokens",
           "l2": "flushed (256 MiB write) before every timed step"}
    # e2e with pinned host buffers
    xh, dyh = x.cpu().pin_memory(), dy.cpu().pin_memory()
    dxh = torch.empty(M_TOK, K_IN, dtype=torch.bfloat16).pin_memory()
    g1h, g2h = torch.empty(K_IN, RANK).pin_memory(), torch.empty(RANK, N_OUT).pin_memory()
    e_steps = max(4, steps // 2)
    xin, dyin = [x.clone() for _ in range(2)], [dy.clone() for _ in range(2)]
    e_graphs = []
    for j in range(2):
        gj = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gj):
            _, cj = lin.forward(xin[j])
            dxj, grj = lin.backward(dyin[j], cj)
        e_graphs.append((gj, dxj, grj))
    torch.cuda.synchronize()
    cstream, ostream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    out_ready = torch.cuda.Event()
    out_read = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        j = i % 2
        with torch.cuda.stream(cstream):
            cstream.wait_event(used[j])
            xin[j].copy_(xh, non_blocking=True)
            dyin[j].copy_(dyh, non_blocking=True)
            h2d_done[j].record(cstream)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    cstream.wait_event(ev0)
    h2d(0)
    for i in range(e_steps):
        if i + 1 < e_steps:
            h2d(i + 1)
        j = i % 2
        stream.wait_event(h2d_done[j])
        gj, dxo, gro = e_graphs[j]
        stream.wait_event(out_read[j])
        gj.replay()
        used[j].record(stream)
        out_ready.record(stream)
        with torch.cuda.stream(ostream):
            ostream.wait_event(out_ready)
            dxh.copy_(dxo, non_blocking=True)
            g1h.copy_(gro["adapter0.l1"], non_blocking=True)
            g2h.copy_(gro["adapter0.l2"], non_blocking=True)
            out_read[j].record(ostream)
    stream.wait_stream(cstream)
    stream.wait_stream(ostream)
    ev1.record(stream)
    torch.cuda.synchronize()
    e_ms = ev0.elapsed_time(ev1) / e_steps
    out["e2e"] = {"tflops": step_flops / (e_ms / 1e3) / 1e12, "ms_per_step": e_ms,
                  "h2d_bytes_per_step": xh.numel() * 2 + dyh.numel() * 2,
                  "d2h_bytes_per_step": dxh.numel() * 2 + g1h.numel() * 4 + g2h.numel() * 4,
                  "note": "QLinear.forward/backward from pinned host X, dY; dX, dl1, dl2 back to pinned host"}
    return out, q, x


def roofline_fused(qb, torch, dev, flush, stream, q, x, tf_burst, peak_kind):
    """The dominant kernel of the C3 step: the fused NF4 dequant-GEMM forward
    of the grouped gate | up projection (2048 x 4096 -> 2 x 11008: two NF4 +
    DQ weights, codes concatenated, QLinearGroup), launched alone through the
    C ABI with a pre-built block-constant cache (no adapter segment), CUDA
    events on its stream.  The C2-shape kernel (one 4096 -> 11008 weight) is
    reported beside it (``c2_kernel``)."""
    from paper_2305_14314_b200._native import lib as _lib, ptr as _ptr, stream_ptr as _sp
    g = torch.Generator(device=dev).manual_seed(11)
    q2 = qb.quantize(torch.randn(K_IN, N_OUT, device=dev, generator=g) * 0.02, qb.get_codebook("nf4"), 64,
                     double_quant=True)
    r = RANK
    grp = qb.QLinearGroup([q, q2], torch.zeros(K_IN, 2 * r, device=dev), torch.zeros(r, 2 * N_OUT, device=dev), r,
                          ALPHA)
    consts = grp._constants()
    desc = grp._desc(consts)
    y = torch.empty(M_TOK, 2 * N_OUT, dtype=torch.bfloat16, device=dev)
    ws = grp._workspace(M_TOK)
    lin0 = qb.QLinear(q, [])
    consts0 = lin0._constants()
    y0 = torch.empty(M_TOK, N_OUT, dtype=torch.bfloat16, device=dev)
    desc0 = lin0.weight_desc(consts0)

    def fused_fwd():
        rc = _lib().qlrt_nf4_linear_fwd(desc, _ptr(x), None, M_TOK, None, None, 0, 0.0, None, _ptr(y), _ptr(ws),
                                        _sp())
        assert rc == 0, rc

    def fused_fwd_c2():
        rc = _lib().qlrt_nf4_linear_fwd(desc0, _ptr(x), None, M_TOK, None, None, 0, 0.0, None, _ptr(y0), _ptr(ws),
                                        _sp())
        assert rc == 0, rc

    k_ms = _timed(torch, stream, flush, [fused_fwd], n=10)
    k_flops = 2 * M_TOK * K_IN * 2 * N_OUT
    achieved = k_flops / (k_ms / 1e3) / 1e12
    c2_ms = _timed(torch, stream, flush, [fused_fwd_c2], n=10)
    c2_flops = 2 * M_TOK * K_IN * N_OUT
    return {"bound": "tensor", "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
            "frac": achieved / tf_burst, "traffic": traffic_of("fused_fwd_gu"),
            "kernel": "gemm_kernel<512,NF4,pair> (fused NF4 dequant + tcgen05 GEMM, 256x512 2-CTA tiles), fwd "
                      "2048x4096x(2x11008): the grouped gate|up projection of the C3 step, alone",
            "kernel_ms": k_ms, "peak_kind": f"{peak_kind} burst bf16 (cuBLAS)",
            "algorithmic_flops_per_launch": k_flops,
            "c2_kernel": {"shape": "2048x4096x11008 (C2, one weight)", "kernel_ms": c2_ms,
                          "achieved": c2_flops / (c2_ms / 1e3) / 1e12,
                          "frac": c2_flops / (c2_ms / 1e3) / 1e12 / tf_burst, "traffic": traffic_of("fused_fwd_c2")}}


def c4_sweep(qb, torch, dev, flush, stream, tf_burst, hbm):
    """C4: LLaMA-65B layer shapes at M = 2048 -- QLinear forward and backward
    with LoRA r = 64 (each one CUDA graph, L2 flushed before each replay) as
    TFLOP/s vs the measured bf16 peak -- and the batch-1 GEMV (M = 1) in GB/s."""
    out = {}
    cb = qb.get_codebook("nf4")
    m = 2048
    for k, n in ((8192, 8192), (8192, 22016), (22016, 8192)):
        g = torch.Generator(device=dev).manual_seed(k + n)
        q = qb.quantize(torch.randn(k, n, device=dev, generator=g) * 0.02, cb, 64, double_quant=True)
        ad = qb.LoraAdapter(RANK, ALPHA, torch.randn(k, RANK, device=dev, generator=g) / 8,
                            torch.randn(RANK, n, device=dev, generator=g) * 0.01)
        lin = qb.QLinear(q, [ad])
        x = torch.randn(m, k, device=dev, generator=g).bfloat16()
        dy = torch.randn(m, n, device=dev, generator=g).bfloat16()
        holder = {}

        def fwd():
            holder["c"] = lin.forward(x)[1]

        fwd()
        cache = holder["c"]
        t_f = _timed(torch, stream, flush, [fwd], n=10)
        t_b = _timed(torch, stream, flush, [lambda: lin.backward(dy, cache)], n=10)
        ff, fb = flops_fwd(m, k, n), flops_bwd(m, k, n)
        out[f"c4_fused_{k}x{n}"] = {
            "m": m, "fwd_ms": t_f, "bwd_ms": t_b, "fwd_tflops": ff / (t_f / 1e3) / 1e12,
            "bwd_tflops": fb / (t_b / 1e3) / 1e12, "fwd_frac": ff / (t_f / 1e3) / 1e12 / tf_burst,
            "bwd_frac": fb / (t_b / 1e3) / 1e12 / tf_burst,
            "note": "QLinear.forward / .backward with LoRA r=64 (all launches: constants, adapter products, "
                    "fused NF4 GEMM), FLOPs incl. the adapter terms"}
        del lin, x, dy, cache, holder
        # batch-1 GEMV: one launch after an L2 flush, and the decode regime --
        # distinct weights of this shape back to back (> 2x L2, like the
        # layers of a model), per launch
        gb = k * n // 2 + k * n // 64 + 4 * (k * n // 64 // 256) + 2 * k + 2 * n
        reps = max(2, -(-(256 << 20) // gb))
        lins = [qb.QLinear(q, [])] + [
            qb.QLinear(qb.quantize(torch.randn(k, n, device=dev, generator=g) * 0.02, cb, 64, double_quant=True), [])
            for _ in range(reps - 1)]
        xv = torch.randn(1, k, device=dev, generator=g).bfloat16()
        t = _timed(torch, stream, flush, [lambda: lins[0].forward(xv)])
        ts = _timed(torch, stream, flush, [(lambda li: (lambda: li.forward(xv)))(li) for li in lins]) / reps
        out[f"c4_gemv_{k}x{n}"] = {"gbs": gb / (t / 1e3) / 1e9, "ms": t, "bytes": gb,
                                   "stream_ms": ts, "stream_gbs": gb / (ts / 1e3) / 1e9,
                                   "frac_hbm": gb / (ts / 1e3) / 1e9 / hbm,
                                   "note": f"ms: one launch after an L2 flush; stream: {reps} distinct weights back "
                                           "to back (> L2), per launch"}
        del q, lins
    torch.cuda.empty_cache()
    return out


def c1_kernels(qb, torch, dev, flush, stream, hbm):
    """C1: NF4 + DQ quantize (fp32 in) and dequantize (bf16 out) GB/s of
    algorithmic bytes; single launch after a flush and a
    stream of distinct tensors (> L2) back to back."""
    from paper_2305_14314_b200._native import BF16, lib, ptr, stream_ptr
    from paper_2305_14314_b200.blockquant import quantize_async
    out = {}
    cb = qb.get_codebook("nf4")

    def deq_launch(q, o):
        d = q.dq
        return lambda: lib().qlrt_dequantize4(ptr(q.codes), q.numel, 64, q.codebook.to_c(), None, ptr(d.codes),
                                              ptr(d.c1), ptr(d.mu), d.blocksize2, d.spec.to_c(), ptr(o), BF16,
                                              stream_ptr())

    for name, shape, reps in (("c1_dequant_bf16", (4096, 4096), 8), ("c4_dequant_bf16_8192x22016", (8192, 22016), 2)):
        n = shape[0] * shape[1]
        qs = [qb.quantize(torch.randn(*shape, device=dev), cb, 64, double_quant=True) for _ in range(reps)]
        outs = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(reps)]
        nb = n // 64
        by = n // 2 + nb + 4 * (nb // 256) + 4 + 2 * n
        t1 = _timed(torch, stream, flush, [deq_launch(qs[0], outs[0])])
        tr = _timed(torch, stream, flush, [deq_launch(q, o) for q, o in zip(qs, outs)]) / reps
        out[name] = {"bytes": by, "single_ms": t1, "single_gbs": by / t1 / 1e6, "stream_ms": tr,
                     "stream_gbs": by / tr / 1e6, "frac_hbm": by / tr / 1e6 / hbm,
                     "note": f"stream = {reps} distinct tensors back to back (> L2), per launch"}
        del qs, outs
    x = torch.randn(4096, 4096, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    n = x.numel()
    nb = n // 64
    q_bytes = 4 * n + n // 2 + nb + 4 * (nb // 256) + 4
    t = _timed(torch, stream, flush, [lambda: quantize_async(x, cb, 64, double_quant=True)])
    xs = [torch.randn(4096, 4096, device=dev) for _ in range(4)]
    ts = _timed(torch, stream, flush, [lambda xx=xx: quantize_async(xx, cb, 64, double_quant=True) for xx in xs]) / 4
    out["c1_quantize_dq_f32"] = {"gbs": q_bytes / (t / 1e3) / 1e9, "ms": t, "stream_ms": ts,
                                 "stream_gbs": q_bytes / (ts / 1e3) / 1e9, "bytes": q_bytes,
                                 "frac_hbm": q_bytes / (ts / 1e3) / 1e9 / hbm,
                                 "note": "quantize + DQ kernels (the non-finite check's host read excluded); "
                                         "stream = 4 distinct inputs back to back, per call"}
    return out


def cpu_baselines(ref: CpuReference):
    """The reference on the host cores: C3 linear-only extrapolation (median
    of 2 fwd+bwd per shape after a warm-up, full 2048 tokens), C2 (the gate /
    up shape of the same sample), C1 quantize + dequantize."""
    layers = _cpu_c3_layers(ref)
    times = {}
    for name, k, n, lin, x, dy in layers:
        ref.fwd_bwd(lin, x, dy)
        ts = []
        for _ in range(2):
            t0 = time.perf_counter()
            ref.fwd_bwd(lin, x, dy)
            ts.append(time.perf_counter() - t0)
        times[name] = statistics.median(ts)
    tok_s = _c3_extrapolate(times)
    c2_t = times["gate"]
    x1 = np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32)
    t0 = time.perf_counter()
    q1 = ref.quantize(x1)
    tq = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref.dequantize(q1)
    td = time.perf_counter() - t0
    n = x1.size
    nb = n // 64
    return ({"value": tok_s, "unit": "tokens/s", "cores": ref.cores, "kind": ref.kind,
             "sample": f"{ref.kind} QLinear fwd+bwd fp32 at each of the 7 LLaMA-7B linear shapes, 2048 tokens, "
                       "median of 2 after a warm-up, x 32 layers (linear-only extrapolation of the C3 step)",
             "per_shape_s": times},
            {"c2_cpu_baseline": {"value": (flops_fwd() + flops_bwd()) / c2_t / 1e12, "unit": "TFLOP/s",
                                 "s_per_step": c2_t, "cores": ref.cores, "kind": ref.kind, "same_config": True,
                                 "sample": "QLinear 4096->11008 r=64 fwd+bwd fp32 on all 2048 tokens"},
             "c1_cpu_baseline": {"quantize_s": tq, "dequantize_s": td,
                                 "quantize_gbs": (4 * n + n // 2 + nb + 4 * (nb // 256) + 4) / tq / 1e9,
                                 "dequantize_gbs": (n // 2 + nb + 4 * (nb // 256) + 4 + 8 * n) / td / 1e9,
                                 "cores": ref.cores, "kind": ref.kind,
                                 "sample": "quantize(4096^2 N(0,1) f32, nf4, 64, double_quant) + dequantize "
                                           "(float64 out), one run each"}})


# ---------------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------------
def spawn(args) -> int:
    """--gpus N > 1 outside torchrun: one rank per GPU under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    # QLRT_BENCH_SHARE_GPU=1 (launcher check only, not a scaling number): every
    # rank on cuda:0 with gloo -- exercises the spawn / rank / reduction path
    # on a one-GPU box
    share = os.environ.get("QLRT_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2305_14314_b200 as qb
    from paper_2305_14314_b200.llama import LlamaConfig

    hbm, tf_burst, tf_sus, peak_kind = load_peaks()
    stream = torch.cuda.current_stream()
    t_wall = time.perf_counter()

    # ---- headline: C3 LLaMA-7B QLoRA step, tokens/s (weak scaling over ranks)
    # (paged AdamW as SURVEY.md §8(d) C3 names it: the moments in unified-memory
    # pages under a budget that holds them; the whole step one CUDA graph)
    c3 = llama_step_bench(torch, dist, "llama-7b shapes", LlamaConfig.llama7b(), world, dev, args.steps, args.warmup,
                          optimizer="paged", e2e_steps=max(4, args.steps // 2), count_launches=True)
    c3["roofline_tokens_per_s"] = world * tf_burst * 1e12 / c3["flops_per_token"]
    c3["roofline_frac"] = c3["tokens_per_s"] / c3["roofline_tokens_per_s"]
    value = c3["tokens_per_s"]

    # ---- C5: LLaMA-33B shapes with paged AdamW (budget = half the moments), every N
    extras = {}
    if not args.no_extras:
        try:
            cfg33 = LlamaConfig.llama33b()
            c5 = llama_step_bench(torch, dist, "llama-33b shapes", cfg33, world, dev, max(3, args.steps // 4), 3,
                                  optimizer="paged")
            c5["roofline_tokens_per_s"] = world * tf_burst * 1e12 / c5["flops_per_token"]
            c5["note"] = ("60 layers h6656 ffn17920 52 heads, seq 512 x 4 per GPU, weak scaling; paged AdamW: "
                          "moments in unified-memory pages under a budget that holds all of them (the normal "
                          "regime: pages fault in once, no eviction)")
            extras["c5_llama33b_paged"] = c5
        except Exception as e:  # pragma: no cover
            extras["c5_llama33b_paged"] = {"error": repr(e)[:300]}

    # ---- C2 single linear (its gate/up fused GEMM is also the roofline kernel)
    c2, q2, x2 = c2_linear(qb, torch, dev, torch.empty(256 << 20, dtype=torch.uint8, device=dev), stream, world,
                           dist, args.steps, args.warmup)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    roofline = roofline_fused(qb, torch, dev, flush, stream, q2, x2, tf_burst, peak_kind)
    extras["c2_linear"] = c2
    del q2, x2

    if rank == 0 and world == 1 and not args.no_extras:
        for fn in (lambda: c1_kernels(qb, torch, dev, flush, stream, hbm),
                   lambda: c4_sweep(qb, torch, dev, flush, stream, tf_burst, hbm)):
            try:
                extras.update(fn())
            except Exception as e:  # pragma: no cover
                extras.setdefault("errors", []).append(repr(e)[:300])
        for label, opt, budget_frac in (("c3_llama7b_plain_adamw", "plain", None),
                                        ("c3_llama7b_paged_budget50", "paged", 0.5)):
            try:
                cfg7 = LlamaConfig.llama7b()
                budget = None if budget_frac is None else int(8 * cfg7.lora_params * budget_frac)
                r = llama_step_bench(torch, dist, "llama-7b shapes", cfg7, world, dev, max(4, args.steps // 2), 3,
                                     optimizer=opt, budget=budget)
                r["vs_plain_ms"] = c3["ms_per_step"]
                extras[label] = r
            except Exception as e:  # pragma: no cover
                extras[label] = {"error": repr(e)[:300]}

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": c3["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens; random-init N(0,0.02) weights quantized NF4+DQ (no checkpoints offline)",
            "config": c3_config(world),
            "e2e": c3.pop("e2e"),
            "roofline": roofline,
            "roofline_tokens_per_s": c3["roofline_tokens_per_s"],
            "gpu_launches": (c3["gpu_launches_per_step"] * args.steps) if c3.get("gpu_launches_per_step") else None,
            "gpu_launches_per_step": c3.get("gpu_launches_per_step"),
            "clocks": c3.pop("clocks"), "c3_llama7b_qlora_step": c3}
    line.update(extras)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb_line, cb_extras = cpu_baselines(CpuReference())
            line["cpu_baseline"] = cb_line
            line.update(cb_extras)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(e)[:300]}
    line["wall_s"] = time.perf_counter() - t_wall
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
