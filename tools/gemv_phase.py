import sys, torch
sys.path.insert(0, '.')
import paper_2305_14314_b200 as qb
k, n = (int(v) for v in sys.argv[1].split("x"))
q = qb.quantize(torch.randn(k, n, device="cuda") * 0.02, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(1, k, device="cuda").bfloat16()
lin = qb.QLinear(q, [])
for _ in range(3): lin.forward(x)
torch.cuda.synchronize()
print("----", flush=True)
lin.forward(x); torch.cuda.synchronize()
