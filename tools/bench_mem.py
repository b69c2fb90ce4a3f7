"""Time the HBM-bound kernels alone: dequant -> bf16, quantize+DQ, GEMV.

single = one launch after an L2 flush (graph replay, CUDA events);
stream = R launches on R distinct tensors (> L2 in total) in one graph, per launch.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from paper_2305_14314_b200.blockquant import quantize_async  # noqa: E402

FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
FLUSH_R = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def flush_l2():
    """Write 256 MiB (> 126 MB L2), then read another 256 MiB so the timed
    kernel does not pay for writing back the flush's own dirty lines."""
    FLUSH.zero_()
    return FLUSH_R.view(torch.int64).sum()


def timed(fns, n=20):
    """Average device time of one replay of a graph that runs fns in order."""
    for _ in range(2):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(n):
        flush_l2()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / n


def main():
    cb = qb.get_codebook("nf4")
    res = {}
    only = sys.argv[1:] or ["dequant", "quantize", "gemv"]
    if "dequant" in only:
        for shape, reps in (((4096, 4096), 8), ((8192, 22016), 2)):
            n = shape[0] * shape[1]
            xs = [torch.randn(*shape, device="cuda") for _ in range(reps)]
            qs = [qb.quantize(x, cb, 64, double_quant=True) for x in xs]
            del xs
            outs = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(reps)]
            nb = n // 64
            by = n // 2 + nb + 4 * (nb // 256) + 4 + 2 * n

            def one(i):
                q = qs[i]
                from paper_2305_14314_b200._native import BF16, lib, ptr, stream_ptr
                d = q.dq
                return lambda: lib().qlrt_dequantize4(ptr(q.codes), n, 64, q.codebook.to_c(), None, ptr(d.codes),
                                                      ptr(d.c1), ptr(d.mu), 256, d.spec.to_c(), ptr(outs[i]), BF16,
                                                      stream_ptr())
            t1 = timed([one(0)])
            tr = timed([one(i) for i in range(reps)]) / reps
            res[f"dequant_bf16_{shape[0]}x{shape[1]}"] = {"bytes": by, "single_us": t1 * 1e3,
                                                         "single_gbs": by / t1 / 1e6, "stream_us": tr * 1e3,
                                                         "stream_gbs": by / tr / 1e6}
            del qs, outs
    if "quantize" in only:
        x = torch.randn(4096, 4096, device="cuda")
        n = x.numel()
        nb = n // 64
        by = 4 * n + n // 2 + nb + 4 * (nb // 256) + 4
        t = timed([lambda: quantize_async(x, cb, 64, double_quant=True)])
        xs = [torch.randn(4096, 4096, device="cuda") for _ in range(4)]
        ts = timed([(lambda xx: (lambda: quantize_async(xx, cb, 64, double_quant=True)))(xx) for xx in xs]) / 4
        # phase A alone (codes + absmax), through the C ABI
        from paper_2305_14314_b200._native import F32, lib, ptr, stream_ptr
        codes = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
        am = torch.empty(nb, dtype=torch.float32, device="cuda")
        fb = torch.empty(1, dtype=torch.int64, device="cuda")
        cbc = cb.to_c()
        ta = timed([(lambda xx: (lambda: lib().qlrt_quantize4(ptr(xx), F32, n, 64, cbc, ptr(codes), ptr(am), ptr(fb),
                                                              stream_ptr())))(xx) for xx in xs]) / 4
        by_a = 4 * n + n // 2 + 4 * nb
        res["quantize_dq_f32_4096x4096"] = {"bytes": by, "single_us": t * 1e3, "single_gbs": by / t / 1e6,
                                            "stream_us": ts * 1e3, "stream_gbs": by / ts / 1e6,
                                            "phase_a_stream_us": ta * 1e3, "phase_a_gbs": by_a / ta / 1e6}
    if "gemv" in only:
        for k, nn in ((8192, 8192), (8192, 22016), (22016, 8192)):
            w = torch.randn(k, nn, device="cuda") * 0.02
            lin = qb.QLinear(qb.quantize(w, cb, 64, double_quant=True), [])
            del w
            xv = torch.randn(1, k, device="cuda").bfloat16()
            nw = k * nn
            by = nw // 2 + nw // 64 + 4 * (nw // 64 // 256) + 2 * k + 2 * nn
            t = timed([lambda: lin.forward(xv)])
            res[f"gemv_{k}x{nn}"] = {"bytes": by, "single_us": t * 1e3, "single_gbs": by / t / 1e6}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
