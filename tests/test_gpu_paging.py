"""The unified-memory pager against the reference pager's behaviour
(pkg/tests/test_paging.py): zero-filled first touch, contents surviving
eviction, multi-page slabs, a random shadow trace, budgets, lifecycle -- with
real migrations (cudaMemPrefetchAsync) under the page table."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pager(qb, budget_pages=4, page_bytes=4096):
    return qb.pager_open(qb.PagerConfig(budget_bytes=budget_pages * page_bytes, page_bytes=page_bytes))


def _fill(value):
    return lambda v: v.fill_(value)


def _read(sink):
    return lambda v: sink.append(v.cpu().numpy().tobytes())


def test_first_touch_zero_fills_and_write_back_survives(qb, cuda):
    with _pager(qb, budget_pages=1) as p:
        s = p.alloc(100)
        sink = []
        p.with_slab(s, _read(sink))
        assert sink[0] == bytes(100) and p.bytes_read == 0
        p.with_slab(s, _fill(0xAB))
        for pid in range(5, 9):  # force the dirty page out
            p.touch(pid)
        assert p.bytes_written >= 4096
        sink = []
        p.with_slab(s, _read(sink))
        assert sink[0] == bytes([0xAB]) * 100 and p.bytes_read >= 4096


def test_multi_page_slab_survives_eviction(qb, cuda):
    with _pager(qb, budget_pages=3) as p:
        s = p.alloc(3 * 4096)
        pattern = torch.arange(3 * 4096, device="cuda").to(torch.uint8)
        p.with_slab(s, lambda v: v.copy_(pattern))
        other = p.alloc(4096)
        p.with_slab(other, _fill(1))  # evicts part of s
        assert p.evictions >= 1
        sink = []
        p.with_slab(s, _read(sink))
        assert sink[0] == pattern.cpu().numpy().tobytes()
        wide = p.alloc(4 * 4096)
        with pytest.raises(ValueError, match="exceeding the budget"):
            p.with_slab(wide, _fill(0))


def test_random_trace_matches_shadow(qb, cuda):
    rng = np.random.default_rng(0)
    with _pager(qb, budget_pages=3) as p:
        sizes = [16, 48, 4096, 5000, 100, 8192, 150, 12000]
        slabs = [p.alloc(n) for n in sizes]
        shadow = {i: bytes(n) for i, n in enumerate(sizes)}
        for step in range(200):
            i = int(rng.integers(len(slabs)))
            if rng.random() < 0.5:
                payload = rng.integers(0, 256, size=sizes[i], dtype=np.uint8)
                t = torch.from_numpy(payload).cuda()
                p.with_slab(slabs[i], lambda v, t=t: v.copy_(t))
                shadow[i] = payload.tobytes()
            else:
                sink = []
                p.with_slab(slabs[i], _read(sink))
                assert sink[0] == shadow[i], f"step {step}, slab {i}"
            assert p.resident_bytes <= p.config.budget_bytes
        assert p.peak_resident_bytes <= p.config.budget_bytes and p.evictions > 0


def test_lookahead_prefetch_then_acquire(qb, cuda):
    """prefetch() faults a slab in without blocking the compute stream;
    acquire() then finds it resident (no second fault)."""
    with _pager(qb, budget_pages=2, page_bytes=2 << 20) as p:
        a, b = p.alloc(2 << 20), p.alloc(2 << 20)
        p.with_slab(a, _fill(3))
        p.prefetch(b)
        f = p.faults
        v = p.acquire(b)
        v.fill_(4)
        p.release(b)
        assert p.faults == f
        sink = []
        p.with_slab(a, _read(sink))
        assert set(sink[0]) == {3}


def test_lifecycle(qb, cuda):
    p = _pager(qb)
    p.touch(0)
    p.close()
    p.close()
    with pytest.raises(ValueError, match="closed"):
        p.touch(0)
