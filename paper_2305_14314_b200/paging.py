"""Paged optimizer state in CUDA unified memory -- the B200-native form of the
reference's file-backed LRU pager (pkg/src/qlrt/paging.py:25-202).

The reference simulates demand paging with a budget of resident bytes, LRU
eviction, dirty write-back and counters, and is value-transparent.  Here the
backing store is host memory reached through ``cudaMallocManaged`` and the
"page cache" is the device: a slab touched by the optimizer is prefetched to
the GPU with ``cudaMemPrefetchAsync`` on a side stream (a *fault* in the
reference's vocabulary), least-recently-used slabs are pushed back to the
host when the resident budget would be exceeded (an *eviction*).  Kernels
read and write the same bytes wherever they live, so the arithmetic -- and
therefore every result -- is identical to the plain store (the transparency
property of pkg/tests/test_training.py:325-350).
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass

import torch

from ._native import check, lib

_cudart = None


def _rt():
    """libcudart for cudaMallocManaged / cudaFree (same runtime torch uses)."""
    global _cudart
    if _cudart is None:
        lib()  # fail loudly without CUDA
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                _cudart = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _cudart is None:
            import glob
            import os
            import nvidia.cuda_runtime as _cr  # torch's bundled runtime
            cands = glob.glob(os.path.join(os.path.dirname(_cr.__file__), "lib", "libcudart.so*"))
            _cudart = ctypes.CDLL(cands[0])
        _cudart.cudaMallocManaged.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
        _cudart.cudaFree.argtypes = [ctypes.c_void_p]
    return _cudart


class _ManagedBuffer:
    """A managed allocation exposed to torch through __cuda_array_interface__."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        rc = _rt().cudaMallocManaged(ctypes.byref(p), ctypes.c_size_t(nbytes), 1)  # cudaMemAttachGlobal
        if rc != 0:
            raise RuntimeError(f"cudaMallocManaged({nbytes}) failed with {rc}")
        self.ptr = p.value
        self.nbytes = nbytes
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 3, "strides": None, "stream": None}
        self.tensor = torch.as_tensor(self, device="cuda")

    def free(self) -> None:
        if self.ptr:
            torch.cuda.synchronize()
            _rt().cudaFree(ctypes.c_void_p(self.ptr))
            self.ptr = 0


@dataclass(frozen=True)
class PagerConfig:
    """Budget of device-resident bytes (paging.py:25-39).  ``backing_path`` is
    accepted for API parity and unused: the backing store is host memory."""

    budget_bytes: int
    backing_path: str | None = None
    page_bytes: int = 2 << 20  # the GPU's unified-memory page granularity

    def validate(self) -> None:
        if self.page_bytes < 1:
            raise ValueError("page_bytes must be >= 1")
        if self.budget_bytes < self.page_bytes:
            raise ValueError(f"budget ({self.budget_bytes}) must hold at least one page ({self.page_bytes})")


@dataclass(frozen=True)
class Slab:
    """A page-aligned byte range owned by one state tensor (paging.py:48-58)."""

    index: int
    offset: int
    nbytes: int


class Pager:
    """LRU residency manager over managed memory.  Not thread-safe, like the reference."""

    def __init__(self, config: PagerConfig):
        config.validate()
        self.config = config
        self._slabs: list[tuple[Slab, _ManagedBuffer]] = []
        self._resident: OrderedDict[int, int] = OrderedDict()  # slab index -> bytes
        self.faults = 0
        self.evictions = 0
        self.bytes_read = 0        # host -> device migrations
        self.bytes_written = 0     # device -> host migrations
        self.peak_resident_bytes = 0
        self._closed = False
        self._side = torch.cuda.Stream()

    def alloc(self, nbytes: int) -> Slab:
        if nbytes < 1:
            raise ValueError("cannot allocate an empty slab")
        pb = self.config.page_bytes
        size = (nbytes + pb - 1) // pb * pb
        buf = _ManagedBuffer(size)
        buf.tensor.zero_()
        slab = Slab(index=len(self._slabs), offset=sum(b.nbytes for _, b in self._slabs), nbytes=nbytes)
        self._slabs.append((slab, buf))
        return slab

    @property
    def resident_bytes(self) -> int:
        return sum(self._resident.values())

    def view(self, slab: Slab) -> torch.Tensor:
        return self._slabs[slab.index][1].tensor[: slab.nbytes]

    def _evict_one(self) -> None:
        idx, nbytes = self._resident.popitem(last=False)
        buf = self._slabs[idx][1]
        with torch.cuda.stream(self._side):
            check(lib().qlrt_prefetch(buf.ptr, buf.nbytes, -1, self._side.cuda_stream), "pager evict")
        self.evictions += 1
        self.bytes_written += buf.nbytes

    def touch(self, slab: Slab) -> None:
        """Make a slab device-resident and most recently used (prefetch on the
        side stream; the current stream waits on it)."""
        if self._closed:
            raise ValueError("pager is closed")
        if slab.index in self._resident:
            self._resident.move_to_end(slab.index)
            return
        buf = self._slabs[slab.index][1]
        if buf.nbytes > self.config.budget_bytes:
            raise ValueError(f"slab of {slab.nbytes} bytes exceeds the budget of {self.config.budget_bytes} bytes")
        while self._resident and self.resident_bytes + buf.nbytes > self.config.budget_bytes:
            self._evict_one()
        cur = torch.cuda.current_stream()
        self._side.wait_stream(cur)
        with torch.cuda.stream(self._side):
            check(lib().qlrt_prefetch(buf.ptr, buf.nbytes, torch.cuda.current_device(), self._side.cuda_stream),
                  "pager prefetch")
        cur.wait_stream(self._side)
        self._resident[slab.index] = buf.nbytes
        self.faults += 1
        self.bytes_read += buf.nbytes
        self.peak_resident_bytes = max(self.peak_resident_bytes, self.resident_bytes)

    def with_slab(self, slab: Slab, fn) -> None:
        """Run ``fn(byte_tensor)`` over the slab's bytes once resident (paging.py:162-187)."""
        self.touch(slab)
        fn(self.view(slab))

    def flush(self) -> None:
        torch.cuda.current_stream().wait_stream(self._side)

    def close(self) -> None:
        if self._closed:
            return
        self.flush()
        for _, buf in self._slabs:
            buf.free()
        self._closed = True

    def __enter__(self) -> "Pager":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def pager_open(config: PagerConfig) -> Pager:
    return Pager(config)


__all__ = ["PagerConfig", "Slab", "Pager", "pager_open"]
