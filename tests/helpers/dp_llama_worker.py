"""One rank of the GPU data-parallel LLaMA-harness test: WORLD_SIZE ranks
(gloo) share cuda:0, each trains on its slice of one fixed batch; WORLD_SIZE=1
trains on the whole batch.  Saves loss, the all-reduced gradient bucket and
the updated parameters to $OUT."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA
    kw = {"hidden": 512, "ffn": 1024, "rank": 64} if os.environ.get("GROUPED") == "1" else {}
    cfg = LlamaConfig.tiny(n_layers=2, **kw)
    m = LlamaQLoRA(cfg, seed=0, bucket_layers=1)
    g = torch.Generator(device="cuda").manual_seed(7)
    for n, p in m.params.items():
        if n.endswith(".l2"):
            p.copy_(torch.randn(p.shape, device="cuda", generator=g) * 0.05)
    m.shadow_flat.copy_(m.params_flat)
    tok = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
    tgt = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
    per = 4 // world
    sl = slice(rank * per, (rank + 1) * per)
    m.set_step_constants()
    loss = m.train_step(tok[sl], tgt[sl])
    torch.cuda.synchronize()
    torch.save({"loss": loss.cpu(), "grads": m.bucket.flat.cpu(), "params": m.params_flat.cpu(),
                "launched": json.dumps(m.reducer.launched)}, os.environ["OUT"])
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
