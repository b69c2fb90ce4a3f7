"""Small drivers for ncu captures: one op family per invocation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402


def main(which: str) -> None:
    dev = torch.device("cuda", 0)
    cb = qb.get_codebook("nf4")
    if which in ("gemm_fwd", "gemm_bwd", "linear"):
        w = torch.randn(4096, 11008, device=dev) * 0.02
        q = qb.quantize(w, cb, 64, double_quant=True)
        x = torch.randn(2048, 4096, device=dev).bfloat16()
        dy = torch.randn(2048, 11008, device=dev).bfloat16()
        ad = qb.LoraAdapter(64, 16.0, torch.randn(4096, 64, device=dev) / 8, torch.randn(64, 11008, device=dev) * .01)
        lin = qb.QLinear(q, [ad] if which == "linear" else [])
        for _ in range(4):
            y, c = lin.forward(x)
            if which != "gemm_fwd":
                lin.backward(dy, c)
    elif which == "gemm_gu":  # the grouped gate | up fused forward of the C3 step (no adapter segment)
        from paper_2305_14314_b200._native import lib, ptr, stream_ptr
        qs = [qb.quantize(torch.randn(4096, 11008, device=dev) * 0.02, cb, 64, double_quant=True) for _ in range(2)]
        grp = qb.QLinearGroup(qs, torch.zeros(4096, 128, device=dev), torch.zeros(64, 22016, device=dev), 64, 16.0)
        consts = grp._constants()
        desc = grp._desc(consts)
        x = torch.randn(2048, 4096, device=dev).bfloat16()
        y = torch.empty(2048, 22016, dtype=torch.bfloat16, device=dev)
        ws = grp._workspace(2048)
        for _ in range(4):
            assert lib().qlrt_nf4_linear_fwd(desc, ptr(x), None, 2048, None, None, 0, 0.0, None, ptr(y), ptr(ws),
                                             stream_ptr()) == 0
    elif which in ("group_bwd", "group_fwd"):  # the grouped gate | up linear of the C3 step with LoRA r = 64
        qs = [qb.quantize(torch.randn(4096, 11008, device=dev) * 0.02, cb, 64, double_quant=True) for _ in range(2)]
        grp = qb.QLinearGroup(qs, torch.randn(4096, 128, device=dev) / 8, torch.randn(64, 22016, device=dev) * .01,
                              64, 16.0)
        x = torch.randn(2048, 4096, device=dev).bfloat16()
        dy = torch.randn(2048, 22016, device=dev).bfloat16()
        dl1 = torch.empty(4096, 128, device=dev)
        dl2 = torch.empty(64, 22016, device=dev)
        for _ in range(4):
            y, c = grp.forward(x)
            if which == "group_bwd":
                grp.backward(dy, c, dl1, dl2)
    elif which == "dequant":
        x = torch.randn(4096, 4096, device=dev)
        q = qb.quantize(x, cb, 64, double_quant=True)
        for _ in range(4):
            qb.dequantize(q, torch.bfloat16)
    elif which == "quantize":
        x = torch.randn(4096, 4096, device=dev)
        for _ in range(4):
            qb.quantize(x, cb, 64, double_quant=True)
    elif which == "gemv":
        w = torch.randn(8192, 22016, device=dev) * 0.02
        lin = qb.QLinear(qb.quantize(w, cb, 64, double_quant=True), [])
        xv = torch.randn(1, 8192, device=dev).bfloat16()
        for _ in range(4):
            lin.forward(xv)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1])
