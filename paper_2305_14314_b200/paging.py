"""Paged optimizer state in CUDA unified memory -- the B200-native form of the
reference's file-backed LRU pager (pkg/src/qlrt/paging.py:25-202).

The reference simulates demand paging: state lives in fixed-size pages, at
most ``budget_bytes`` of them are resident, touching a non-resident page is a
*fault* (read back from the backing file, or zero-filled on first touch),
least-recently-used pages are *evicted* (dirty ones written back), and
counters expose the traffic.  It is value-transparent.

Here the backing store is host memory reached through ``cudaMallocManaged``
and the "page cache" is the device:

* :class:`PageTable` is the reference's replacement policy and counters,
  page for page (LRU over page ids, faults / evictions / bytes read / bytes
  written / peak residency with the reference's definitions).  It is pure
  bookkeeping, so the CPU tests pin it to the reference's own traces.
* :class:`Pager` binds the table to memory: a fault is a
  ``cudaMemPrefetchAsync`` of the page run to the GPU on an H2D side stream,
  an eviction a prefetch back to the host (``cudaCpuDeviceId``) on a D2H side
  stream -- both PCIe directions move at once, beside the compute stream.
  An eviction waits only for the last kernel that used the page (a per-page
  "last use" event recorded by :meth:`Pager.release`), and a re-fault of a
  page waits for its pending eviction, so the migrations never race the
  kernels and the budget is real residency, not just accounting.
* :meth:`Pager.prefetch` is the look-ahead: it faults a slab's pages early
  without making the compute stream wait; :meth:`Pager.acquire` then waits
  on that prefetch's event only, at the point of use.

Kernels read and write the same bytes wherever they live, so the arithmetic
-- and therefore every result -- is identical to the plain store (the
transparency property of pkg/tests/test_training.py:325-350).
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass

import torch

from ._native import check, lib

_cudart = None
_CPU_DEVICE = -1  # cudaCpuDeviceId


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
    """A managed allocation exposed to torch through __cuda_array_interface__.
    Zero-filled by the CPU, so its pages start host-resident (not resident in
    the pager's sense) -- the reference's "first touch zero-fills"."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        rc = _rt().cudaMallocManaged(ctypes.byref(p), ctypes.c_size_t(nbytes), 1)  # cudaMemAttachGlobal
        if rc != 0:
            raise RuntimeError(f"cudaMallocManaged({nbytes}) failed with {rc}")
        self.ptr = p.value
        self.nbytes = nbytes
        ctypes.memset(self.ptr, 0, nbytes)
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
    accepted for API parity and unused: the backing store is host memory.
    The default page is the reference's 4 KiB; large optimizer states use
    the GPU's 2 MiB unified-memory migration unit (the LLaMA harness)."""

    budget_bytes: int
    backing_path: str | None = None
    page_bytes: int = 4096

    def validate(self) -> None:
        if self.page_bytes < 1:
            raise ValueError("page_bytes must be >= 1")
        if self.budget_bytes < self.page_bytes:
            raise ValueError(f"budget ({self.budget_bytes}) must hold at least one page ({self.page_bytes})")


@dataclass(frozen=True)
class Slab:
    """A page-aligned byte range owned by one state tensor (paging.py:48-58)."""

    offset: int
    nbytes: int
    index: int = 0

    def pages(self, page_bytes: int) -> range:
        first = self.offset // page_bytes
        last = (self.offset + max(self.nbytes, 1) - 1) // page_bytes
        return range(first, last + 1)


class PageTable:
    """The reference pager's replacement policy and counters without the
    bytes (paging.py:116-158): LRU over page ids, ``touch`` returns the page
    ids it faulted in and evicted so the caller can move memory."""

    def __init__(self, config: PagerConfig):
        config.validate()
        self.config = config
        self._resident: OrderedDict[int, bool] = OrderedDict()  # page id -> dirty
        self._backed: set[int] = set()  # pages written back at least once ("on disk")
        self.faults = 0
        self.evictions = 0
        self.bytes_read = 0
        self.bytes_written = 0
        self.peak_resident_bytes = 0

    @property
    def resident_bytes(self) -> int:
        return len(self._resident) * self.config.page_bytes

    def is_resident(self, page_id: int) -> bool:
        return page_id in self._resident

    def resident_pages(self) -> list[int]:
        """Resident page ids, least recently used first."""
        return list(self._resident)

    def _evict_one(self, evicted: list) -> None:
        pid, dirty = self._resident.popitem(last=False)
        if dirty:
            self._backed.add(pid)
            self.bytes_written += self.config.page_bytes
        self.evictions += 1
        evicted.append(pid)

    def touch(self, page_id: int, faulted: list | None = None, evicted: list | None = None) -> bool:
        """Make a page resident and most recently used; True on a fault."""
        faulted = [] if faulted is None else faulted
        evicted = [] if evicted is None else evicted
        if page_id in self._resident:
            self._resident.move_to_end(page_id)
            return False
        pb = self.config.page_bytes
        while self.resident_bytes + pb > self.config.budget_bytes:
            self._evict_one(evicted)
        self.faults += 1
        if page_id in self._backed:
            self.bytes_read += pb
        self._resident[page_id] = False
        faulted.append(page_id)
        self.peak_resident_bytes = max(self.peak_resident_bytes, self.resident_bytes)
        return True

    def mark_dirty(self, page_ids) -> None:
        for pid in page_ids:
            if pid in self._resident:
                self._resident[pid] = True

    def flush(self) -> int:
        """Write every dirty resident page back (does not evict); returns pages written."""
        n = 0
        for pid, dirty in self._resident.items():
            if dirty:
                self._backed.add(pid)
                self.bytes_written += self.config.page_bytes
                self._resident[pid] = False
                n += 1
        return n


def _runs(pages: list[int]) -> list[tuple[int, int]]:
    """Sorted page ids -> (first, count) runs of consecutive pages."""
    out: list[tuple[int, int]] = []
    for p in sorted(pages):
        if out and out[-1][0] + out[-1][1] == p:
            out[-1] = (out[-1][0], out[-1][1] + 1)
        else:
            out.append((p, 1))
    return out


class Pager:
    """LRU page cache of device residency over managed memory.  Not
    thread-safe, like the reference (paging.py:61-63)."""

    def __init__(self, config: PagerConfig):
        self.table = PageTable(config)
        self.config = config
        self._bufs: list[tuple[int, _ManagedBuffer]] = []  # (first page id, buffer)
        self._slabs: list[Slab] = []
        self._next_offset = 0
        self._last_use: dict[int, torch.cuda.Event] = {}   # page -> event after its last kernel
        self._evict_evt: dict[int, torch.cuda.Event] = {}  # page -> event after its pending eviction
        self._ready: dict[int, torch.cuda.Event] = {}      # slab index -> event after its prefetch
        self._closed = False
        lib()
        self._h2d = torch.cuda.Stream()
        self._d2h = torch.cuda.Stream()
        self._dev = torch.cuda.current_device()

    # -- counters (the reference's names) ---------------------------------
    faults = property(lambda self: self.table.faults)
    evictions = property(lambda self: self.table.evictions)
    bytes_read = property(lambda self: self.table.bytes_read)
    bytes_written = property(lambda self: self.table.bytes_written)
    peak_resident_bytes = property(lambda self: self.table.peak_resident_bytes)
    resident_bytes = property(lambda self: self.table.resident_bytes)

    @property
    def n_pages(self) -> int:
        return self._next_offset // self.config.page_bytes

    # -- allocation ---------------------------------------------------------
    def alloc(self, nbytes: int) -> Slab:
        """A page-aligned slab of ``nbytes`` backed by managed memory, zeroed,
        host-resident until first touched (paging.py:97-104)."""
        if nbytes < 1:
            raise ValueError("cannot allocate an empty slab")
        pb = self.config.page_bytes
        n_pages = (nbytes + pb - 1) // pb
        slab = Slab(offset=self._next_offset, nbytes=nbytes, index=len(self._slabs))
        self._bufs.append((self._next_offset // pb, _ManagedBuffer(n_pages * pb)))
        self._slabs.append(slab)
        self._next_offset += n_pages * pb
        return slab

    def view(self, slab: Slab) -> torch.Tensor:
        """The slab's bytes as a uint8 CUDA tensor (valid wherever the pages live)."""
        first, buf = self._bufs[slab.index]
        start = slab.offset - first * self.config.page_bytes
        return buf.tensor[start: start + slab.nbytes]

    def _locate(self, page_id: int):
        """(buffer, byte offset) of an allocated page; None for a page id
        outside every slab (bookkeeping-only, as ``touch`` allows)."""
        pb = self.config.page_bytes
        lo, hi = 0, len(self._bufs) - 1
        while lo <= hi:
            mid = (lo + hi) // 2
            first, buf = self._bufs[mid]
            if page_id < first:
                hi = mid - 1
            elif page_id >= first + buf.nbytes // pb:
                lo = mid + 1
            else:
                return buf, (page_id - first) * pb
        return None

    # -- migration --------------------------------------------------------
    def _migrate(self, pages: list[int], to_device: bool) -> torch.cuda.Event | None:
        """Prefetch runs of pages to the GPU (H2D stream) or back to the host
        (D2H stream); returns the event recorded after the last one."""
        if not pages:
            return None
        pb = self.config.page_bytes
        s = self._h2d if to_device else self._d2h
        issued = False
        for first, count in _runs(pages):
            # split runs at buffer boundaries
            p = first
            while p < first + count:
                loc = self._locate(p)
                if loc is None:
                    p += 1
                    continue
                buf, off = loc
                n = min(first + count - p, (buf.nbytes - off) // pb)
                for q in range(p, p + n):
                    if to_device:
                        ev = self._evict_evt.pop(q, None)
                        if ev is not None:
                            s.wait_event(ev)
                    else:
                        ev = self._last_use.pop(q, None)
                        if ev is not None:
                            s.wait_event(ev)
                check(lib().qlrt_prefetch(buf.ptr + off, n * pb, self._dev if to_device else _CPU_DEVICE,
                                          s.cuda_stream), "pager prefetch" if to_device else "pager evict")
                issued = True
                p += n
        if not issued:
            return None
        ev = torch.cuda.Event()
        ev.record(s)
        if not to_device:
            for p in pages:
                self._evict_evt[p] = ev
        return ev

    def _fault_slab(self, slab: Slab) -> torch.cuda.Event | None:
        if self._closed:
            raise ValueError("pager is closed")
        pb = self.config.page_bytes
        page_ids = list(slab.pages(pb))
        if len(page_ids) * pb > self.config.budget_bytes:
            raise ValueError(f"slab of {slab.nbytes} bytes spans {len(page_ids)} pages, "
                             f"exceeding the budget of {self.config.budget_bytes} bytes")
        faulted: list[int] = []
        evicted: list[int] = []
        for pid in page_ids:
            self.table.touch(pid, faulted, evicted)
        self._migrate(evicted, to_device=False)
        return self._migrate(faulted, to_device=True)

    # -- the reference's API ------------------------------------------------
    def touch(self, page_id: int) -> None:
        """Make one page resident and most recently used (paging.py:148-158)."""
        if self._closed:
            raise ValueError("pager is closed")
        faulted: list[int] = []
        evicted: list[int] = []
        self.table.touch(page_id, faulted, evicted)
        self._migrate(evicted, to_device=False)
        ev = self._migrate(faulted, to_device=True)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def prefetch(self, slab: Slab) -> None:
        """Look-ahead: fault the slab's pages in on the H2D stream now; the
        compute stream waits for them only in :meth:`acquire`."""
        ev = self._fault_slab(slab)
        if ev is not None:
            self._ready[slab.index] = ev

    def acquire(self, slab: Slab) -> torch.Tensor:
        """Make the slab resident (faulting what is missing) and order the
        current stream after its migration; returns the byte view."""
        ev = self._fault_slab(slab)
        cur = torch.cuda.current_stream()
        pending = self._ready.pop(slab.index, None)
        for e in (pending, ev):
            if e is not None:
                cur.wait_event(e)
        self.table.mark_dirty(slab.pages(self.config.page_bytes))
        return self.view(slab)

    def release(self, slab: Slab) -> None:
        """Record the current stream's position as the last use of the slab's
        pages: a later eviction of them waits for exactly this."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        for pid in slab.pages(self.config.page_bytes):
            self._last_use[pid] = ev

    def with_slab(self, slab: Slab, fn) -> None:
        """Run ``fn(byte_tensor)`` over the slab's bytes once resident; its
        pages become dirty (paging.py:162-187)."""
        view = self.acquire(slab)
        fn(view)
        self.release(slab)

    def flush(self) -> None:
        """The reference writes dirty pages back; unified memory has one copy,
        so this only counts them and joins the side streams."""
        self.table.flush()
        cur = torch.cuda.current_stream()
        cur.wait_stream(self._h2d)
        cur.wait_stream(self._d2h)

    def close(self) -> None:
        if self._closed:
            return
        self.flush()
        for _, buf in self._bufs:
            buf.free()
        self._closed = True

    def __enter__(self) -> "Pager":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def pager_open(config: PagerConfig) -> Pager:
    return Pager(config)


def with_page(pager: Pager, page_id: int, fn) -> None:
    """Run ``fn`` over one whole page, marking it dirty (paging.py:196-202)."""
    pager.touch(page_id)
    loc = pager._locate(page_id)
    if loc is not None:
        buf, off = loc
        fn(buf.tensor[off: off + pager.config.page_bytes])
    pager.table.mark_dirty([page_id])


__all__ = ["PagerConfig", "Slab", "PageTable", "Pager", "pager_open", "with_page"]
