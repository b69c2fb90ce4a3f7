"""One rank of the gloo data-parallel test (launched as a plain script)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> None:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_14314_b200.parallel import GradBucket, LayerReducer, allreduce_mean, shard_rows
        g = {"adapter0.l1": torch.full((8, 4), float(rank + 1)),
             "adapter0.l2": torch.arange(12, dtype=torch.float32).view(4, 3) * (rank + 1)}
        out = allreduce_mean(g)
        b = GradBucket({"a": (3,), "b": (2, 2)}, "cpu")
        b.load({"a": torch.ones(3) * rank, "b": torch.ones(2, 2) * (10 + rank)})
        b.start()
        avg = b.finish()
        sl = shard_rows(10, rank, world)
        # overlapped layer-group reducer: 5 layers of 3 values, groups of 2
        # layers; layers become ready last-first as in a backward
        red = {}
        for wire in (torch.float32, torch.bfloat16):
            flat = torch.arange(15, dtype=torch.float32) * (rank + 1)
            r = LayerReducer(flat, [(3 * i, 3) for i in range(5)], group_layers=2, wire_dtype=wire)
            r.reset()
            early = []
            for li in (4, 3, 2):
                r.layer_ready(li)
                early.append(list(r.launched))
            r.finish()
            red[str(wire)] = {"flat": flat.tolist(), "early": early, "launched": r.launched}
        print(json.dumps({"reducer": red, "rank": rank, "l1": out["adapter0.l1"].tolist(), "l2": out["adapter0.l2"].tolist(),
                          "a": avg["a"].tolist(), "b": avg["b"].tolist(), "shard": [sl.start, sl.stop]}))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
