import torch, sys
sys.path.insert(0, '.')
import paper_2305_14314_b200 as qb
from torch.profiler import profile, ProfilerActivity
k, n, m = 4096, 11008, 2048
w = torch.randn(k, n, device="cuda") * 0.02
q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
for ads in ([], [qb.LoraAdapter(64, 16.0, torch.randn(k, 64, device="cuda") / 8, torch.randn(64, n, device="cuda") * .01)]):
    lin = qb.QLinear(q, ads)
    for _ in range(3):
        y, c = lin.forward(x); lin.backward(dy, c)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            y, c = lin.forward(x); lin.backward(dy, c)
        torch.cuda.synchronize()
    print("adapters", len(ads))
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=70))
