import sys, time, json
sys.path.insert(0, ".")
import torch
import bench
import torch.distributed as dist
from paper_2305_14314_b200.llama import LlamaConfig
dev = torch.device("cuda", 0)
for opt in ("plain", "paged"):
    r = bench.llama_step_bench(torch, dist, "33b", LlamaConfig.llama33b(), 1, dev, 4, 3, optimizer=opt)
    print(opt, round(r["ms_per_step"], 2), round(r["tokens_per_s"], 1), flush=True)
