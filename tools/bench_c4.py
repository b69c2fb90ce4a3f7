"""Config C4: LLaMA-65B layer shapes, fused NF4 dequant-GEMM + LoRA fwd / bwd at M tokens.

Per shape: fused forward (Y = X W + LoRA), fused backward (dX, dl1, dl2), the
main fused GEMM alone (no adapter), and cuBLAS bf16 on a dense W for context.
TFLOP/s use the SURVEY §8(d) FLOP counts; each op timed alone (graph replay
between L2 flushes, CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402


def main():
    m = int(os.environ.get("C4_M", "2048"))
    r = 64
    shapes = [(8192, 8192), (8192, 22016), (22016, 8192)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
    res = {}
    cb = qb.get_codebook("nf4")
    for k, n in shapes:
        g = torch.Generator(device="cuda").manual_seed(k + n)
        w = torch.randn(k, n, device="cuda", generator=g) * 0.02
        q = qb.quantize(w, cb, 64, double_quant=True)
        wb = w.bfloat16()
        del w
        x = torch.randn(m, k, device="cuda", generator=g).bfloat16()
        dy = torch.randn(m, n, device="cuda", generator=g).bfloat16()
        ad = qb.LoraAdapter(r, 16.0, torch.randn(k, r, device="cuda", generator=g) / 8,
                            torch.randn(r, n, device="cuda", generator=g) * 0.01)
        lin = qb.QLinear(q, [ad])
        lin0 = qb.QLinear(q, [])
        f_fwd = 2 * m * k * n + 2 * m * k * r + 2 * m * r * n
        f_bwd = 2 * m * n * k + 2 * m * n * r + 2 * r * m * n + 2 * k * m * r + 2 * m * r * k
        f_main = 2 * m * k * n
        t_fwd = timed([lambda: lin.forward(x)], n=10)
        _, c = lin.forward(x)
        t_bwd = timed([lambda: lin.backward(dy, c)], n=10)
        t_main = timed([lambda: lin0.forward(x)], n=10)
        _, c0 = lin0.forward(x)
        t_main_b = timed([lambda: lin0.backward(dy, c0)], n=10)
        o = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        t_cub = timed([lambda: torch.matmul(x, wb, out=o)], n=10)
        res[f"{k}x{n}"] = {
            "M": m,
            "fwd_lora_tflops": f_fwd / t_fwd / 1e9, "fwd_lora_us": t_fwd * 1e3,
            "bwd_lora_tflops": f_bwd / t_bwd / 1e9, "bwd_lora_us": t_bwd * 1e3,
            "fused_main_fwd_tflops": f_main / t_main / 1e9,
            "fused_main_bwd_tflops": f_main / t_main_b / 1e9,
            "cublas_dense_bf16_tflops": f_main / t_cub / 1e9,
        }
        del q, wb, x, dy, lin, lin0, c, c0, o
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
