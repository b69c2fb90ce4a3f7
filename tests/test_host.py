"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side logic (codebook tables, fast-path brackets, accounting)."""

from __future__ import annotations

import re

import numpy as np
import pytest

import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _declared_symbols():
    text = (ROOT / "include" / "qlrt_b200.h").read_text()
    return sorted(set(re.findall(r"\b(qlrt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2305_14314_b200 import _native
    lib = _native.load_library()  # no kernels launched: works without a GPU
    declared = _declared_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTS)
    assert lib.qlrt_build_info() == b"qlrt_b200 sm_100a"


def test_workspace_queries_are_host_only():
    from paper_2305_14314_b200 import _native
    lib = _native.load_library()
    assert lib.qlrt_dq_workspace_bytes(262144) == 32 * 8 + 16  # chunk sums + mu ticket
    assert lib.qlrt_linear_workspace_bytes(2048, 4096, 11008, 64) >= 16 * 2048 * 64 * 4


def test_product_codebooks_match_reference_golden(golden, golden_meta):
    from paper_2305_14314_b200 import codebooks
    for name in ("nf4", "fp4-e2m1", "fp4-e3m0", "int4", "nf-eq4"):
        cb = codebooks.get_codebook(name)
        assert np.array_equal(cb.values, golden[f"cb/{name}/values"]), name
        assert np.array_equal(cb.midpoints(), golden[f"cb/{name}/mids"]), name
        assert cb.zero_code == golden_meta[f"cb/{name}"]["zero_code"]


def test_fast_path_brackets_are_sound():
    from paper_2305_14314_b200 import codebooks
    for name in ("nf4", "fp4-e2m1", "int4", "nf-eq4"):
        cb = codebooks.get_codebook(name)
        c = cb.to_c()
        mids = cb.midpoints()
        assert c.n_mids == mids.size
        for i, m in enumerate(mids):
            assert c.lo[i] < m < c.hi[i], (name, i)
            if i:
                assert c.hi[i - 1] < c.lo[i]
        for i in range(mids.size, 16):
            assert c.lo[i] == np.inf
        assert c.pad_code == (cb.zero_code if cb.zero_code is not None
                              else int(np.searchsorted(mids, 0.0, side="right")))


def test_pad_code_for_zero_free_codebook(golden):
    from paper_2305_14314_b200 import codebooks
    cb = codebooks.get_codebook("nf-eq4")
    assert cb.zero_code is None
    # the reference pads with nearest_codes(0) == searchsorted(mids, 0, 'right')
    assert cb.pad_code == int(np.searchsorted(golden["cb/nf-eq4/mids"], 0.0, side="right"))


def test_bits_per_param_and_fp8_spec():
    from paper_2305_14314_b200 import Fp8Spec, bits_per_param
    assert bits_per_param(4, 64) == 4.5
    assert bits_per_param(4, 64, dq=(256, 8)) == 4.126953125
    assert bits_per_param(4, 64) - bits_per_param(4, 64, dq=(256, 8)) == 0.373046875
    assert Fp8Spec().max_value == 480.0
    assert Fp8Spec(5, 2, 15).max_value == 1.75 * 2.0 ** 16
    vals, codes = Fp8Spec().grid()
    assert vals.size == 255 and vals[0] == -480.0
    with pytest.raises(ValueError):
        Fp8Spec(4, 4)
    with pytest.raises(ValueError):
        bits_per_param(4, 64, dq=(0, 8))


def test_gpu_calls_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2305_14314_b200 import get_codebook, quantize
    with pytest.raises(RuntimeError, match="CUDA"):
        quantize(np.ones(64, dtype=np.float32), get_codebook("nf4"))


def test_adam_constants_follow_nep50():
    from paper_2305_14314_b200.training import AdamOptimizer, PlainMomentStore, TrainConfig
    opt = AdamOptimizer({}, TrainConfig(), PlainMomentStore())
    opt.t = 2
    b1, omb1, b2, omb2, bc1, bc2, eps, lr = opt.constants()
    assert omb1 == float(np.float32(1.0 - 0.9))
    assert bc2 == float(np.float32(1.0 - 0.999 ** 2))
    assert lr == float(np.float32(0.01))


def test_page_table_replays_reference_pager_traces():
    """paging.PageTable (the GPU pager's replacement policy and counters) vs
    the reference Pager's counters after every operation of random traces
    (tests/golden/make_golden_pager.py; pkg/src/qlrt/paging.py:116-187)."""
    import json
    from paper_2305_14314_b200.paging import PagerConfig, PageTable, Slab
    traces = json.loads((ROOT / "tests" / "golden" / "pager_traces.json").read_text())
    for tr in traces:
        pb = tr["page_bytes"]
        t = PageTable(PagerConfig(budget_bytes=tr["budget_bytes"], page_bytes=pb))
        slabs = [Slab(offset=o, nbytes=n) for o, n in tr["slabs"]]
        for (op, arg), want in zip(tr["ops"], tr["counters"]):
            if op == "touch":
                t.touch(arg)
            else:
                pages = list(slabs[arg].pages(pb))
                for pid in pages:
                    t.touch(pid)
                t.mark_dirty(pages)
            got = [t.faults, t.evictions, t.bytes_read, t.bytes_written, t.peak_resident_bytes, t.resident_bytes]
            assert got == want, (op, arg, got, want)
        t.flush()
        assert t.bytes_written == tr["bytes_written_after_flush"]


def test_page_table_lru_order_and_slab_pages():
    """pkg/tests/test_paging.py:42-47, 63-86 restated on the page table."""
    from paper_2305_14314_b200.paging import PagerConfig, PageTable, Slab
    assert list(Slab(offset=0, nbytes=64).pages(64)) == [0]
    assert list(Slab(offset=64, nbytes=65).pages(64)) == [1, 2]
    assert list(Slab(offset=128, nbytes=200).pages(64)) == [2, 3, 4, 5]
    t = PageTable(PagerConfig(budget_bytes=128, page_bytes=64))
    for pid in (0, 1, 0, 2, 0, 1):
        t.touch(pid)
    assert (t.faults, t.evictions) == (4, 2)
    with pytest.raises(ValueError, match="at least one page"):
        PagerConfig(budget_bytes=63, page_bytes=64).validate()
    with pytest.raises(ValueError, match="page_bytes"):
        PagerConfig(budget_bytes=64, page_bytes=0).validate()
