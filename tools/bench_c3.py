"""Config C3 / C5: LLaMA-shaped QLoRA finetune step, tokens/s (one CUDA graph per step).
usage: python tools/bench_c3.py [7b|33b|tiny] [--layers L] [--batch B] [--steps K]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA  # noqa: E402


def run(model_name="7b", layers=None, batch=4, steps=10, warmup=3, graph=True, lag=1):
    mk = {"7b": LlamaConfig.llama7b, "33b": LlamaConfig.llama33b, "tiny": LlamaConfig.tiny}[model_name]
    cfg = mk(**({"n_layers": layers} if layers else {}))
    t0 = time.time()
    m = LlamaQLoRA(cfg, seed=0, defer_lag=lag)
    build_s = time.time() - t0
    g = torch.Generator(device="cuda").manual_seed(0)
    tok = torch.randint(0, cfg.vocab, (batch, cfg.seq), device="cuda", generator=g)
    tgt = torch.randint(0, cfg.vocab, (batch, cfg.seq), device="cuda", generator=g)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warmup):
            m.set_step_constants()
            m.train_step(tok, tgt)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    step = lambda: m.train_step(tok, tgt)  # noqa: E731
    if graph:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            loss_g = m.train_step(tok, tgt)
        step = gr.replay
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(steps):
        m.set_step_constants()
        step()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    tokens = batch * cfg.seq
    fl = cfg.flops_per_token() * tokens
    return {"model": f"llama-{model_name} shapes" + (f" ({layers} layers)" if layers else ""),
            "layers": cfg.n_layers, "tokens_per_step": tokens, "ms_per_step": ms,
            "tokens_per_s": tokens / (ms / 1e3), "tflops": fl / (ms / 1e3) / 1e12,
            "flops_per_token": cfg.flops_per_token(), "linear_params": cfg.linear_params,
            "lora_params": cfg.lora_params, "build_s": build_s, "cuda_graph": graph,
            "max_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
            "loss": float((loss_g if graph else m.train_step(tok, tgt)).item())}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("model", nargs="?", default="7b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--lag", default="1", help="deferred adapter-gradient lag in layers, or 'none'")
    a = ap.parse_args()
    print(json.dumps(run(a.model, a.layers, a.batch, a.steps, graph=not a.no_graph,
                          lag=None if a.lag == "none" else int(a.lag))))
