"""Host <-> device copies for the drop-in per-layer API (host NumPy in, `bytes`
/ NumPy out, as the reference's codec.py:116-197 and precision.py:25-28).

A pageable `torch.from_numpy(x).cuda()` runs at ~11 GB/s and `.cpu().numpy()
.tobytes()` at ~1-2 GB/s on the B200 boxes: the latter pays the DMA through a
driver bounce buffer plus a single-threaded copy into freshly allocated
(page-faulting) memory. Large transfers here go through a reused pinned
staging buffer, in chunks: DMA at PCIe speed, and the host-side copy into or
out of the caller's memory split over worker threads (NumPy and ctypes copies
release the GIL, and page faults of a fresh output are taken in parallel).
The results are the same objects the reference returns: a new `bytes`, a new
writable float32 array.
"""

from __future__ import annotations

import ctypes
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

SMALL = 1 << 20            # below this, plain torch copies
CHUNK = 64 << 20           # staging chunk (bytes)
THREADS = 16               # host copy threads per chunk (>= 4 MiB each)
_init_lock = threading.Lock()   # lazy creation of the pool; the free lists of staging sets
_staging: dict = {}        # device index -> free staging sets (each: two pinned CHUNK buffers + events)
_pool = None

_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_AsString = ctypes.pythonapi.PyBytes_AsString
_PyBytes_AsString.restype = ctypes.c_void_p
_PyBytes_AsString.argtypes = [ctypes.py_object]


try:                                   # fresh outputs: ask for transparent huge pages
    _madvise = ctypes.CDLL(None, use_errno=True).madvise
    _madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
except (OSError, AttributeError):
    _madvise = None
_HUGE = 2 << 20
_MADV_HUGEPAGE = 14


def _advise_huge(ptr: int, nbytes: int) -> None:
    """First-touch page faults bound the copy into a freshly allocated output
    (~8 GB/s at 4 KiB pages on the B200 hosts, whose THP mode is "madvise");
    2 MiB pages take it to ~14 GB/s (profiles/r01_hostlink.md). Advisory only."""
    lo, hi = (ptr + _HUGE - 1) & ~(_HUGE - 1), (ptr + nbytes) & ~(_HUGE - 1)
    if _madvise is not None and hi > lo:
        _madvise(lo, hi - lo, _MADV_HUGEPAGE)


def _workers() -> ThreadPoolExecutor:
    global _pool
    if _pool is None:
        with _init_lock:
            if _pool is None:
                _pool = ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)))
    return _pool


class _Stage:
    """A staging set (two pinned CHUNK-byte buffers + their events, double
    buffering) checked out of the per-device free list for one copy: threads
    copying at the same time each get their own set (a new one is created
    when none is free), so host copies never serialise on a shared buffer."""

    def __init__(self, device: torch.device):
        self.idx = device.index if device.index is not None else torch.cuda.current_device()
        self.bufs = None

    def __enter__(self) -> list:
        with _init_lock:
            free = _staging.setdefault(self.idx, [])
            self.bufs = free.pop() if free else None
        if self.bufs is None:
            self.bufs = [(torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
                         for _ in range(2)]
        return self.bufs

    def __exit__(self, *exc):
        with _init_lock:
            _staging[self.idx].append(self.bufs)


class _SmallStage:
    """Per (thread, device) pinned + device scratch for one small call (< SMALL
    bytes each way): the host bytes are copied into pinned memory, the H2D,
    the kernels and the D2H are queued back to back on the current stream,
    and ONE stream sync ends the call — instead of a synchronous pageable
    H2D, the launch, and a second synchronous pageable D2H."""

    _local = threading.local()

    def __init__(self, device: torch.device):
        self.h_in = torch.empty(SMALL, dtype=torch.uint8, pin_memory=True)
        self.h_out = torch.empty(SMALL, dtype=torch.uint8, pin_memory=True)
        self.d_in = torch.empty(SMALL, dtype=torch.uint8, device=device)
        self.d_out = torch.empty(SMALL, dtype=torch.uint8, device=device)
        self.h_in_np, self.h_out_np = self.h_in.numpy(), self.h_out.numpy()

    @classmethod
    def get(cls, device: torch.device) -> "_SmallStage":
        stages = getattr(cls._local, "stages", None)
        if stages is None:
            stages = cls._local.stages = {}
        idx = device.index if device.index is not None else torch.cuda.current_device()
        st = stages.get(idx)
        if st is None:
            st = stages[idx] = _SmallStage(torch.device("cuda", idx))
        return st


def small_call(host_in: np.ndarray, out_nbytes: int, fn, device: torch.device | str = "cuda") -> np.ndarray:
    """One small host -> device -> host call: host_in (contiguous, < SMALL
    bytes) lands in a device uint8 buffer `d_in`, fn(d_in, d_out) queues the
    device work on the current stream writing d_out[:out_nbytes] (< SMALL),
    and the result comes back as a view of a reused pinned buffer — valid
    until this thread's next small call (callers copy it out)."""
    dev = torch.device(device)
    src = np.ascontiguousarray(host_in).reshape(-1).view(np.uint8)
    n = src.size
    if n > SMALL or out_nbytes > SMALL:
        raise ValueError("small_call: more than SMALL bytes")
    st = _SmallStage.get(dev)
    stream = torch.cuda.current_stream(st.d_in.device)
    st.h_in_np[:n] = src
    if n:
        st.d_in[:n].copy_(st.h_in[:n], non_blocking=True)
    fn(st.d_in, st.d_out)
    if out_nbytes:
        st.h_out[:out_nbytes].copy_(st.d_out[:out_nbytes], non_blocking=True)
    stream.synchronize()
    return st.h_out_np[:out_nbytes]


def _parallel_memmove(dst: int, src: int, nbytes: int) -> None:
    n = max(1, min(THREADS, nbytes >> 22))     # >= 4 MiB per thread
    step = -(-nbytes // n)
    futs = [_workers().submit(ctypes.memmove, dst + i * step, src + i * step, min(step, nbytes - i * step))
            for i in range(n) if i * step < nbytes]
    for f in futs:
        f.result()


def to_device(host: np.ndarray, device: torch.device | str = "cuda") -> torch.Tensor:
    """A contiguous host array -> a new CUDA tensor of the same dtype (flattened).
    Chunk k+1 is copied into one pinned buffer while chunk k's DMA drains the other."""
    dev = torch.device(device)
    host = np.ascontiguousarray(host).reshape(-1)
    if host.nbytes < SMALL:
        return torch.from_numpy(host).to(dev)
    out = torch.empty(host.size, dtype=torch.from_numpy(host[:1]).dtype, device=dev)
    raw_out = out.view(torch.uint8)
    src = host.ctypes.data
    stream = torch.cuda.current_stream(out.device)
    with _Stage(out.device) as bufs:
        for k, pos in enumerate(range(0, host.nbytes, CHUNK)):
            n = min(CHUNK, host.nbytes - pos)
            buf, done = bufs[k & 1]
            done.synchronize()                  # this buffer's previous DMA has finished
            _parallel_memmove(buf.data_ptr(), src + pos, n)
            raw_out[pos:pos + n].copy_(buf[:n], non_blocking=True)
            done.record(stream)
        stream.synchronize()
    return out


def _from_device(dev_bytes: torch.Tensor, dst: int) -> None:
    """Chunk k+1's DMA into one pinned buffer overlaps the copy of chunk k out of the other."""
    stream = torch.cuda.current_stream(dev_bytes.device)
    total = dev_bytes.numel()
    chunks = list(range(0, total, CHUNK))
    with _Stage(dev_bytes.device) as bufs:
        def issue(k):
            pos = chunks[k]
            buf, done = bufs[k & 1]
            buf[:min(CHUNK, total - pos)].copy_(dev_bytes[pos:pos + CHUNK], non_blocking=True)
            done.record(stream)
        issue(0)
        for k, pos in enumerate(chunks):
            if k + 1 < len(chunks):
                issue(k + 1)
            buf, done = bufs[k & 1]
            done.synchronize()
            _parallel_memmove(dst + pos, buf.data_ptr(), min(CHUNK, total - pos))


def to_bytes(dev_u8: torch.Tensor) -> bytes:
    """A CUDA uint8 tensor -> a new `bytes` object holding its contents."""
    flat = dev_u8.reshape(-1)
    if flat.numel() < SMALL:
        return flat.cpu().numpy().tobytes()
    out = _PyBytes_FromStringAndSize(None, flat.numel())   # uninitialised, filled below (sole owner)
    dst = _PyBytes_AsString(out)
    _advise_huge(dst, flat.numel())
    _from_device(flat.contiguous(), dst)
    return out


def to_numpy_f32(dev_f32: torch.Tensor) -> np.ndarray:
    """A CUDA float32 tensor -> a new writable float32 NumPy array."""
    flat = dev_f32.reshape(-1)
    if flat.numel() * 4 < SMALL:
        return flat.cpu().numpy()
    out = np.empty(flat.numel(), dtype=np.float32)
    _advise_huge(out.ctypes.data, out.nbytes)
    _from_device(flat.contiguous().view(torch.uint8), out.ctypes.data)
    return out
