"""Counter traces of the reference pager (pkg/src/qlrt/paging.py) for the
page-table parity test: random touch / with_slab traffic at several budgets,
with the counters after every operation.  Run in the build container, where
the reference imports:
    python tests/golden/make_golden_pager.py"""
import json
import os
import sys
import tempfile

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from qlrt.paging import PagerConfig, pager_open  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pager_traces.json")
traces = []
for seed, budget_pages, page_bytes, sizes in ((0, 3, 64, [16, 48, 64, 72, 100, 128, 150, 192]),
                                             (1, 2, 64, [48] * 6),
                                             (2, 5, 4096, [5000, 12000, 4096, 1, 30000 // 3])):
    rng = np.random.default_rng(seed)
    with tempfile.TemporaryDirectory() as d:
        cfg = PagerConfig(budget_bytes=budget_pages * page_bytes, backing_path=os.path.join(d, "s.bin"),
                          page_bytes=page_bytes)
        with pager_open(cfg) as p:
            slabs = [p.alloc(n) for n in sizes]
            ops, counters = [], []
            for _ in range(300):
                if rng.random() < 0.3:
                    pid = int(rng.integers(0, p.n_pages + 3))
                    p.touch(pid)
                    ops.append(["touch", pid])
                else:
                    i = int(rng.integers(len(slabs)))
                    p.with_slab(slabs[i], lambda v: None)
                    ops.append(["slab", i])
                counters.append([p.faults, p.evictions, p.bytes_read, p.bytes_written, p.peak_resident_bytes,
                                 p.resident_bytes])
            p.flush()
            final_flush = p.bytes_written
    traces.append({"budget_bytes": budget_pages * page_bytes, "page_bytes": page_bytes, "sizes": sizes,
                   "slabs": [[s.offset, s.nbytes] for s in slabs], "ops": ops, "counters": counters,
                   "bytes_written_after_flush": final_flush})
with open(OUT, "w") as fh:
    json.dump(traces, fh)
print("wrote", OUT)
