"""Benchmark of the B200-native QLoRA hot path.

Default workload (BASELINE.json configs[1], "C2"): one frozen NF4 linear
4096 -> 11008 with a LoRA adapter r = 64 (alpha 16), bf16 forward + backward
over 4 x 512 tokens per GPU.  A step = forward (Ts = s X l1 and the fused NF4
dequant-GEMM with the LoRA term in the same TMEM accumulator) + backward (dT,
fused dX GEMM, dl1, dl2) [+ on N > 1 GPUs the NCCL all-reduce of the adapter
gradients, weak scaling].  value = whole-job TFLOP/s of the fwd+bwd FLOPs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

``--impl reference`` times the CPU oracle (numpy restatement of qlrt, the
reference's algorithm) on this host's cores on a bounded token sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NF4 dequant GB/s vs HBM peak; fused 4-bit GEMM TFLOPS; QLoRA tokens/sec at 1/2/4/8 B200"
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
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle reasons sampled in-process through NVML every ~2 ms
    while the timed region runs (the region is only milliseconds long)."""

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
# reference arm / cpu baseline: the oracle (numpy restatement of qlrt)
# ---------------------------------------------------------------------------
def cpu_reference(m_sample: int, reps: int, seed: int = 0):
    """QLinear fwd + bwd of the CPU oracle at config C2's layer, float32 (the
    reference's "low" precision mode), on ``m_sample`` tokens; dequantization
    of the full 4096 x 11008 weight every call as the reference does."""
    from oracle import qlrt_oracle as orc
    rng = np.random.default_rng(seed)
    w = (0.02 * rng.standard_normal((K_IN, N_OUT))).astype(np.float32)
    q = orc.quantize(w, orc.get_codebook("nf4"), 64, double_quant=True)
    ad = orc.LoraAdapter(RANK, ALPHA, (rng.standard_normal((K_IN, RANK)) / 8).astype(np.float32),
                         (0.01 * rng.standard_normal((RANK, N_OUT))).astype(np.float32))
    x = rng.standard_normal((m_sample, K_IN)).astype(np.float32)
    dy = rng.standard_normal((m_sample, N_OUT)).astype(np.float32)
    times = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        wd = orc.dequantize(q).astype(np.float32)          # qlora.py:117-122 (per call)
        y, cache = orc.qlinear_forward(wd, [ad], x, dtype=np.float32)
        dx, grads = orc.qlinear_backward([ad], dy, cache, dtype=np.float32)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times[1:])
    fl = flops_fwd(m_sample) + flops_bwd(m_sample)
    return fl / t / 1e12, t, os.cpu_count()


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    m_sample = 256
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.warmup):
        cpu_reference(m_sample, 1)
    for _ in range(args.steps):
        v, _, cores = cpu_reference(m_sample, 1)
        vals.append(v)
    value = statistics.median(vals)
    sample = f"oracle QLinear fwd+bwd fp32, {m_sample} of {M_TOK} tokens, full 4096x11008 dequant per call"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2 single NF4 linear 4096->11008 LoRA r=64 fwd+bwd (token sample)",
                       "tokens_per_step": m_sample},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
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

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2305_14314_b200 as qb
    from paper_2305_14314_b200.parallel import GradBucket

    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    w = torch.randn(K_IN, N_OUT, device=dev, generator=torch.Generator(device=dev).manual_seed(0)) * 0.02
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    del w
    l1 = torch.randn(K_IN, RANK, device=dev, generator=g) / 8
    l2 = torch.randn(RANK, N_OUT, device=dev, generator=g) * 0.01
    lin = qb.QLinear(q, [qb.LoraAdapter(RANK, ALPHA, l1, l2)])
    x = torch.randn(M_TOK, K_IN, device=dev, generator=g).bfloat16()
    dy = torch.randn(M_TOK, N_OUT, device=dev, generator=g).bfloat16()
    bucket = GradBucket({"adapter0.l1": (K_IN, RANK), "adapter0.l2": (RANK, N_OUT)}, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(xx, dd):
        y, cache = lin.forward(xx)
        dx, grads = lin.backward(dd, cache)
        if world > 1:
            bucket.load(grads)
            bucket.start()
            grads = bucket.finish()
        return y, dx, grads

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step(x, dy)
    torch.cuda.synchronize()
    # the fwd+bwd launches captured once into a CUDA graph (no tracing compiler:
    # the same ctypes launches, replayed without per-kernel host overhead)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y_g, c_g = lin.forward(x)
        dx_g, grads_g = lin.backward(dy, c_g)
    graph.replay()
    torch.cuda.synchronize()

    def step_graph():
        graph.replay()
        if world > 1:
            bucket.load(grads_g)
            bucket.start()
            bucket.finish()

    # count our kernel launches per step (profiler pass outside the timed region)
    launches_per_step = None
    try:
        if os.environ.get("QLRT_NO_TORCH_PROFILER"):
            raise RuntimeError("disabled (running under ncu)")
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(x, dy)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        launches_per_step = sum(1 for n in names if "qlrt" in n)
    except Exception:
        pass

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step_graph()
            ends[i].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    step_flops = flops_fwd() + flops_bwd()
    value = world * step_flops * args.steps / (ms / 1e3) / 1e12

    # ---- e2e through the public API with pinned host buffers: every step copies
    # its X, dY in (pinned -> device) and dX, dl1, dl2 out (device -> pinned).
    # Copies run on a side stream, double-buffered, so step i+1's inputs cross
    # PCIe while step i computes (the compute stream waits on per-buffer events).
    xh = x.cpu().pin_memory()
    dyh = dy.cpu().pin_memory()
    dxh = torch.empty(M_TOK, K_IN, dtype=torch.bfloat16).pin_memory()
    g1h = torch.empty(K_IN, RANK).pin_memory()
    g2h = torch.empty(RANK, N_OUT).pin_memory()
    e_steps = max(4, args.steps // 2)
    xin = [x.clone() for _ in range(2)]
    dyin = [dy.clone() for _ in range(2)]
    # the public-API calls (QLinear.forward / backward) on each input buffer,
    # captured once into a CUDA graph so the host does not pace the GPU
    e_graphs = []
    for j in range(2):
        gj = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gj):
            _, cj = lin.forward(xin[j])
            dxj, grj = lin.backward(dyin[j], cj)
        e_graphs.append((gj, dxj, grj))
    torch.cuda.synchronize()
    cstream = torch.cuda.Stream(dev)
    ostream = torch.cuda.Stream(dev)  # D2H on its own stream: both PCIe directions at once
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    out_ready = torch.cuda.Event()
    out_read = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        j = i % 2
        with torch.cuda.stream(cstream):
            cstream.wait_event(used[j])  # the compute of step i-2 is done with buffer j
            xin[j].copy_(xh, non_blocking=True)
            dyin[j].copy_(dyh, non_blocking=True)
            h2d_done[j].record(cstream)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    cstream.wait_event(ev0)
    h2d(0)
    for i in range(e_steps):
        if i + 1 < e_steps:
            h2d(i + 1)
        j = i % 2
        stream.wait_event(h2d_done[j])
        gj, dx, grads = e_graphs[j]
        stream.wait_event(out_read[j])
        gj.replay()
        if world > 1:
            bucket.load(grads)
            bucket.start()
            grads = bucket.finish()
        used[j].record(stream)
        out_ready.record(stream)
        with torch.cuda.stream(ostream):
            ostream.wait_event(out_ready)
            dxh.copy_(dx, non_blocking=True)
            g1h.copy_(grads["adapter0.l1"], non_blocking=True)
            g2h.copy_(grads["adapter0.l2"], non_blocking=True)
            out_read[j].record(ostream)  # graph j's outputs are read; its next replay (step i+2) waits
    stream.wait_stream(cstream)
    stream.wait_stream(ostream)
    ev1.record(stream)
    torch.cuda.synchronize()
    e_ms = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e = world * step_flops * e_steps / (float(e_ms.item()) / 1e3) / 1e12
    h2d_bytes = xh.numel() * 2 + dyh.numel() * 2
    d2h = dxh.numel() * 2 + g1h.numel() * 4 + g2h.numel() * 4
    # pinned H2D bandwidth of this box (context for e2e)
    ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ta.record(stream)
    for _ in range(3):
        dyin[0].copy_(dyh, non_blocking=True)
    tb.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = 3 * dyh.numel() * 2 / (ta.elapsed_time(tb) / 1e3) / 1e9

    # ---- roofline of the dominant kernel: the fused NF4 dequant-GEMM (forward
    # main GEMM, 2*M*K*N FLOPs per launch), launched alone through the C ABI
    # with a pre-built block-constant cache (so the graph holds only that kernel)
    hbm, tf_burst, tf_sus, peak_kind = load_peaks()
    from paper_2305_14314_b200._native import lib as _lib, ptr as _ptr, stream_ptr as _sp
    lin0 = qb.QLinear(q, [])
    consts0 = lin0._constants()
    y0 = torch.empty(M_TOK, N_OUT, dtype=torch.bfloat16, device=dev)
    ws0 = lin0._workspace(M_TOK)
    desc0 = lin0.weight_desc(consts0)

    def fused_fwd():
        rc = _lib().qlrt_nf4_linear_fwd(desc0, _ptr(x), None, M_TOK, None, None, 0, 0.0, None, _ptr(y0), _ptr(ws0),
                                        _sp())
        assert rc == 0, rc

    for _ in range(3):
        fused_fwd()
    torch.cuda.synchronize()
    g0 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g0):
        fused_fwd()
    g0.replay()
    n_k = 10
    ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_ms = 0.0
    for _ in range(n_k):
        flush.zero_()
        ka.record(stream)
        g0.replay()
        kb.record(stream)
        torch.cuda.synchronize()
        k_ms += ka.elapsed_time(kb)
    k_ms /= n_k
    k_flops = 2 * M_TOK * K_IN * N_OUT
    achieved = k_flops / (k_ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
                "frac": achieved / tf_burst, "traffic": traffic_of("fused_fwd_c2"),
                "kernel": "gemm_kernel<512,NF4,pair> (fused NF4 dequant + tcgen05 GEMM, 256x512 2-CTA tiles), fwd 2048x4096x11008, alone",
                "kernel_ms": k_ms, "peak_kind": f"{peak_kind} burst bf16 (cuBLAS)",
                "algorithmic_flops_per_launch": k_flops}

    extras = {}
    if not args.no_extras:
        extras = secondary(qb, torch, dev, flush, stream, hbm)
        # C3: LLaMA-7B-shape QLoRA finetune step on this GPU (tokens/s), whole step in one CUDA graph
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from bench_c3 import run as run_c3
            c3 = run_c3("7b", batch=4, steps=10)
            c3["roofline_tokens_per_s"] = tf_burst * 1e12 / c3["flops_per_token"]
            c3["note"] = ("32 layers h4096 ffn11008 vocab32000, seq 512 x 4, all 7 linears NF4+DQ with LoRA r=64; "
                          "random-init weights, synthetic tokens; fwd+bwd+grad all-reduce+clip+Adam per step")
            extras["c3_llama7b_qlora_step"] = c3
        except Exception as e:  # pragma: no cover
            extras["c3_llama7b_qlora_step"] = {"error": repr(e)}

    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random N(0,0.02) weight quantized NF4+DQ)",
            "config": {"workload": "C2: single frozen NF4 linear 4096->11008, LoRA r=64 alpha=16, bf16 fwd+bwd, "
                                   "4x512 tokens per GPU" + (", adapter-grad NCCL all-reduce" if world > 1 else ""),
                       "tokens_per_gpu": M_TOK, "flops_per_step_per_gpu": step_flops,
                       "parallelism": f"dp{world}", "l2": "flushed (256 MiB write) before every timed step"},
            "tokens_per_s": world * M_TOK * args.steps / (ms / 1e3),
            "e2e": {"value": e2e, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h,
                    "steps": e_steps, "pinned_h2d_gbs": h2d_gbs,
                    "note": "QLinear.forward/backward (CUDA-graph captured) from pinned host X, dY; dX, dl1, "
                            "dl2 back to pinned host; copies double-buffered on a side stream"},
            "roofline": roofline,
            "gpu_launches": (launches_per_step * args.steps) if launches_per_step else None,
            "gpu_launches_per_step": launches_per_step,
            "clocks": clk.summary(), "wall_s": t_wall}
    line.update(extras)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, t, cores = cpu_reference(256, 2)
        line["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                                "sample": "oracle QLinear fwd+bwd fp32 on 256 of 2048 tokens (full-weight dequant "
                                          f"per call), median of 2 after 1 warm-up: {t:.2f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def secondary(qb, torch, dev, flush, stream, hbm):
    """HBM-bound kernels (C1 dequant / quantize, 65B-shape dequant and GEMV)
    and the plain-bf16 engine ceiling, each timed alone: a CUDA graph of the
    launches replayed after an L2 flush (single = one launch; stream = R
    launches over R distinct tensors, > L2 in total, per launch)."""
    out = {}

    def timed(fns, n=20):
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

    from paper_2305_14314_b200._native import BF16, lib, ptr, stream_ptr
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
        t1 = timed([deq_launch(qs[0], outs[0])])
        tr = timed([deq_launch(q, o) for q, o in zip(qs, outs)]) / reps
        out[name] = {"bytes": by, "single_ms": t1, "single_gbs": by / t1 / 1e6, "stream_ms": tr,
                     "stream_gbs": by / tr / 1e6, "frac_hbm": by / tr / 1e6 / hbm,
                     "note": f"stream = {reps} distinct tensors back to back (> L2), per launch"}
        del qs, outs
    x = torch.randn(4096, 4096, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    n = x.numel()
    nb = n // 64
    q_bytes = 4 * n + n // 2 + nb + 4 * (nb // 256) + 4
    from paper_2305_14314_b200.blockquant import quantize_async
    t = timed([lambda: quantize_async(x, cb, 64, double_quant=True)])
    out["c1_quantize_dq_f32"] = {"gbs": q_bytes / (t / 1e3) / 1e9, "ms": t, "bytes": q_bytes,
                                 "frac_hbm": q_bytes / (t / 1e3) / 1e9 / hbm,
                                 "note": "quantize + DQ kernels; the non-finite check's host read excluded"}
    # the same tcgen05 engine without the dequant producer (TMA-fed dense bf16 W), C2 shape
    wb = (torch.randn(4096, 11008, device=dev) * 0.02).bfloat16()
    xb = torch.randn(2048, 4096, device=dev).bfloat16()
    ob = torch.empty(2048, 11008, device=dev, dtype=torch.bfloat16)
    t = timed([lambda: qb.gemm_bf16(xb, wb, out=ob)])
    out["engine_bf16_gemm_2048x4096x11008"] = {"tflops": 2 * 2048 * 4096 * 11008 / (t / 1e3) / 1e12, "ms": t}
    del wb, xb, ob
    for k, nn in ((8192, 8192), (8192, 22016), (22016, 8192)):
        lin = qb.QLinear(qb.quantize(torch.randn(k, nn, device=dev) * 0.02, cb, 64, double_quant=True), [])
        xv = torch.randn(1, k, device=dev).bfloat16()
        t = timed([lambda: lin.forward(xv)])
        nw = k * nn
        gb = nw // 2 + nw // 64 + 4 * (nw // 64 // 256) + 2 * k + 2 * nn
        out[f"c4_gemv_{k}x{nn}"] = {"gbs": gb / (t / 1e3) / 1e9, "ms": t, "bytes": gb,
                                    "frac_hbm": gb / (t / 1e3) / 1e9 / hbm}
        del lin
    return out


if __name__ == "__main__":
    main()
