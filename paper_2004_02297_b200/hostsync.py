"""CPU-master weight distribution: the paper's own setting.

The FP32 master weights live in HOST memory (the optimizer updates them on the
CPU); before every host->GPU transfer they are packed on the CPU (Bitpack,
PAPER.md:259-268, 351-452: the top RoundTo bytes of every weight), only the
packed stream crosses PCIe, and the GPU zero-fills the dropped bytes (Bitunpack,
PAPER.md:454-493). The reference restates the byte semantics in
codec.pack_vectorized / unpack (codec.py:149-197) and runs the caller order of
training.py:207-254; this class is that caller order with the codec split
across the two processors:

    host:   adt_pack_host (all cores, AVX-512 VBMI, l2-norm fused into the
            read) -> pinned staging buffer, cut into units of 64K weights
    link:   cudaMemcpyAsync of every finished run of units while the rest is
            still being packed (Σ n·r bytes instead of 4·Σ n)
    device: adt_unpack of the whole stream into the FP32 replicas

(one C call, adt_host_to_device; or adt_host_to_device_ring through a small
pinned ring when ring_bytes > 0). The norms come out of the host pass, so the
AWP decision (precision.PrecisionController) needs no device->host read.
Whether this beats copying FP32 depends on the host: the host pass streams
(4 + r)·n bytes through host DRAM next to the DMA's r·n, against 4·n for a raw
FP32 copy (bench.py `host_master`).
"""

from __future__ import annotations

import ctypes
import math
from typing import Sequence

import numpy as np
import torch

from . import _lib, engine
from .layout import PackedLayout
from .precision import FixedPrecision, PrecisionController
from .sync import SyncResult, flat_views

ZERO_COPY_BYTES = 2 << 20   # default HostWeightSync(zero_copy_bytes=): streams up to 2 MiB unpack from host memory
HOST_ALIGN = 64        # payload offsets: full 64-B lines for the packer's non-temporal stores


def _host_view(m, i: int) -> np.ndarray:
    """A host master as a flat float32 NumPy view of the caller's own memory
    (the CPU optimizer updates it in place between steps), never a copy."""
    if isinstance(m, torch.Tensor):
        if m.is_cuda:
            raise TypeError(f"master layer {i}: HostWeightSync takes host (CPU) masters; use WeightSync for "
                            "device-resident masters")
        m = m.detach().numpy()
    if not isinstance(m, np.ndarray) or m.dtype != np.float32:
        raise TypeError(f"master layer {i}: need a float32 NumPy array or CPU tensor")
    if not m.flags.c_contiguous:
        raise ValueError(f"master layer {i}: array is not C-contiguous (a flattened copy would be packed "
                         "instead of it)")
    return m.reshape(-1)


class HostWeightSync:
    """Host FP32 masters -> host pack -> packed H2D -> device unpack, per step.

    masters: per-layer float32 host arrays (NumPy or CPU tensors; pinned or
    not — only the staging buffer needs to be page-locked), read in place.
    replicas: per-layer CUDA float32 tensors (allocated when omitted).
    threads: host packer threads (0 = the process's whole CPU affinity).
    """

    def __init__(self, masters: Sequence, schedule=None, replicas: Sequence[torch.Tensor] | None = None,
                 device: torch.device | str | None = None, threads: int = 0, min_copy_bytes: int = 0,
                 ring_bytes: int = 0, slot_bytes: int = 384 << 10, direct_full: bool = True,
                 zero_copy_bytes: int = ZERO_COPY_BYTES):
        engine.require_cuda()
        self.masters = [_host_view(m, i) for i, m in enumerate(masters)]
        self.counts = [m.size for m in self.masters]
        L = len(self.masters)
        self.schedule = schedule if schedule is not None else FixedPrecision(L, 32)
        if self.schedule.num_layers != L:
            raise ValueError("schedule layer count differs from the number of master arrays")
        self.adaptive = isinstance(self.schedule, PrecisionController)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if replicas is None:
            replicas = [torch.empty(n, dtype=torch.float32, device=self.device) for n in self.counts]
        self.replicas = flat_views(replicas, "replica")
        if [r.numel() for r in self.replicas] != self.counts:
            raise ValueError("replica sizes differ from the masters")
        self.threads = int(threads)
        # direct_full: layers at full width (round_to 4) whose masters are
        # page-locked go to their replicas by DMA straight from the masters
        # (adt_host_to_device_ex, ADT_H2D_DIRECT_FULL) instead of through the
        # host packer and the device unpack: identical replicas and norms, the
        # same bytes on the link, a third of the host DRAM traffic for them.
        self.direct_full = bool(direct_full)
        self.direct = np.zeros(max(1, L), dtype=np.uint8)   # which layers the last launch sent that way
        self.min_copy_bytes = int(min_copy_bytes)
        # packed streams up to zero_copy_bytes skip the staging copy: the device
        # unpack reads them from the pinned staging buffer across the link
        # (ADT_H2D_ZERO_COPY). A copy's fixed cost (~10 us) exceeds its transfer
        # time there (profiles/r02_small_host.md); 0 = always copy.
        self.zero_copy_bytes = int(zero_copy_bytes)
        cap = PackedLayout.plan(self.counts, [4] * L, align=HOST_ALIGN).nbytes
        # ring_bytes = 0 (default): one pinned staging buffer as large as the
        # stream (adt_host_to_device). > 0: a small pinned ring of slot_bytes
        # slots (adt_host_to_device_ring) — measured 1.2-1.9x SLOWER on the B200
        # boxes (per-chunk copy + event overheads outweigh the DRAM traffic it
        # saves; profiles/r02_hostmaster.md), kept as an option. The device
        # buffer has room for every width: a re-plan never reallocates.
        self.ring_bytes, self.slot_bytes = int(ring_bytes), int(slot_bytes)
        stage = self.ring_bytes if self.ring_bytes else cap
        self.staging = torch.empty(max(64, stage + 64), dtype=torch.uint8, pin_memory=True)
        base = (-self.staging.data_ptr()) % 64
        self._stage_ptr = self.staging.data_ptr() + base        # 64-B aligned stream start
        self.packed = torch.empty(max(64, cap), dtype=torch.uint8, device=self.device)
        self.sumsq = np.zeros(max(1, L), dtype=np.float64)
        self._sumsq_ptr = self.sumsq.ctypes.data           # (ctypes attribute lookups cost ~1 us per launch)
        self._direct_ptr = self.direct.ctypes.data
        self._dma_done = torch.cuda.Event()
        self._dma_pending = False
        # device-side norms of the direct layers (their replica equals the master)
        self._dn_idx: list[int] = []
        self._dn_table = None
        self._dn_done = torch.cuda.Event()
        self._dn_pending = False
        self._plan(self.schedule.round_tos())

    def _plan(self, round_tos) -> None:
        self.layout = PackedLayout.plan(self.counts, round_tos, align=HOST_ALIGN)
        self._host_segs = _lib.segment_array([(m.ctypes.data if n else 0, n, off, r) for m, n, off, r in
                                              zip(self.masters, self.counts, self.layout.offsets,
                                                  self.layout.round_tos)])
        self.unpack_table = engine.SegmentTable(self.replicas, self.layout)

    @property
    def round_tos(self) -> list[int]:
        return list(self.layout.round_tos)

    @property
    def zero_copy(self) -> bool:
        """Whether the next launch's unpack reads the packed stream straight
        from the pinned staging buffer (small streams) instead of a device copy."""
        return self.ring_bytes == 0 and 0 < self.layout.nbytes <= self.zero_copy_bytes

    def stream_bytes(self) -> np.ndarray:
        """The packed stream the last launch's unpack read (a host copy, for
        checks): the device buffer, or under zero copy the pinned staging
        buffer itself. Call after the stream has passed the launch."""
        n = self.layout.nbytes
        if self.zero_copy:
            base = self._stage_ptr - self.staging.data_ptr()
            return self.staging.numpy()[base:base + n].copy()
        return self.packed[:n].cpu().numpy()

    @property
    def h2d_bytes(self) -> int:
        """Bytes one transfer moves over the link: the packed stream (payloads + < 64 B pad per layer)."""
        return self.layout.nbytes

    def launch(self, fused_norm: bool = True, stream: torch.cuda.Stream | None = None, events=None) -> None:
        """One transfer: pack on the host (norms fused when `fused_norm`),
        copy the packed stream as it is produced, unpack on the device. Returns
        when the host side is done; the copies and the unpack are queued on
        `stream` (default: the current stream). events = (e0, e1, e2): timing
        events recorded before the copies, between the copies and the unpack,
        and after the unpack (transfer.LedgerRecorder)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self._dma_pending:
            self._dma_done.synchronize()         # the staging buffer is free again
        if events is not None:
            events[0].record(s)
        dev_segs = self.unpack_table.array if events is None else None
        sums = self._sumsq_ptr if fused_norm else None
        lib = _lib.load()
        if self.ring_bytes:
            _lib.check(lib.adt_host_to_device_ring(
                self._host_segs, dev_segs, len(self.counts), self._stage_ptr, self.ring_bytes, self.slot_bytes,
                self.packed.data_ptr(), self.layout.nbytes, sums, self.threads, int(s.cuda_stream)))
        else:
            flags = (_lib.H2D_DIRECT_FULL | _lib.H2D_SKIP_DIRECT_NORMS) if (self.direct_full and dev_segs is not None) \
                else 0
            if dev_segs is not None and self.zero_copy:
                flags |= _lib.H2D_ZERO_COPY
            self._dn_pending = False
            _lib.check(lib.adt_host_to_device_ex(
                self._host_segs, dev_segs, len(self.counts), self._stage_ptr, self.packed.data_ptr(),
                self.layout.nbytes, sums, self.threads, self.min_copy_bytes, flags, self._direct_ptr,
                int(s.cuda_stream)))
            if fused_norm and flags and self.direct.any():
                self._direct_norms(s)
        if events is not None:
            events[1].record(s)
            engine.unpack(self.unpack_table, self.packed, s)
            events[2].record(s)
        self._dma_done.record(s)
        self._dma_pending = True

    def tune(self, threads=None, batches=None, reps: int = 3) -> dict:
        """Pick the packer thread count and the copy batch size for this set on
        this host (setup-time, like cudnn's benchmark mode): time whole
        transfers (launch -> stream sync, best of `reps`) over a small grid and
        keep the fastest. More threads are not always faster: the packers and
        the DMA share host DRAM, and once the pack runs ahead of the link extra
        threads only take bandwidth from the DMA; larger copy batches cost the
        calling thread (which also packs) fewer cudaMemcpyAsync calls (AlexNet
        mixed widths: 3.3 ms at 16 threads / 1 MiB, 3.1-3.2 ms at 6-8 threads /
        4-8 MiB; VGG-16 r = 1 needs all 16 threads; profiles/r02_small_host.md).
        Replicas are rewritten with the same values; the masters are only read.
        Returns {"<threads>x<batch KiB>": seconds}."""
        import time
        total = host_threads()
        if threads is None:
            threads = sorted({total, max(1, (3 * total) // 4), max(1, total // 2), max(1, (3 * total) // 8)},
                             reverse=True)
        if batches is None:
            batches = [b for b in (1 << 20, 4 << 20, 8 << 20) if 2 * b <= self.layout.nbytes] or [0]
        s = torch.cuda.current_stream(self.device)
        keep = (self.threads, self.min_copy_bytes)
        timings, best = {}, None
        for b in batches:
            for t in threads:
                self.threads, self.min_copy_bytes = int(t), int(b)
                self.launch(fused_norm=True)              # warm
                s.synchronize()
                dt = float("inf")
                for _ in range(reps):
                    t0 = time.perf_counter()
                    self.launch(fused_norm=True)
                    s.synchronize()
                    dt = min(dt, time.perf_counter() - t0)
                timings[f"{int(t)}x{int(b) >> 10}K"] = dt
                if best is None or dt < best[0]:
                    best = (dt, int(t), int(b))
        self.threads, self.min_copy_bytes = (best[1], best[2]) if best else keep
        return timings

    def tune_threads(self, candidates=None, reps: int = 3) -> dict:
        """tune() over thread counts only (copy batch unchanged); {threads: seconds}."""
        t = self.tune(threads=candidates, batches=[self.min_copy_bytes], reps=reps)
        return {int(k.split("x")[0]): v for k, v in t.items()}

    def _direct_norms(self, s) -> None:
        """The direct layers' sums of squares, on the device from their replicas
        (bit-equal to the masters at full width): adt_sumsq on `s` behind the
        copies, then an 8-B-per-layer device->host read that norms() waits for.
        A host read of those masters beside their DMA would slow the DMA
        (profiles/r02_host_direct.md)."""
        idx = [i for i in range(len(self.counts)) if self.direct[i]]
        if idx != self._dn_idx:
            self._dn_idx = idx
            lay = PackedLayout.plan([self.counts[i] for i in idx], [4] * len(idx))
            self._dn_table = engine.SegmentTable([self.replicas[i] for i in idx], lay)
            self._dn_dev = torch.empty(len(idx), dtype=torch.float64, device=self.device)
            self._dn_host = torch.empty(len(idx), dtype=torch.float64, pin_memory=True)
        engine.sumsq(self._dn_table, self._dn_dev, s)
        self._dn_host.copy_(self._dn_dev, non_blocking=True)
        self._dn_done.record(s)
        self._dn_pending = True

    def norms(self) -> list[float]:
        """precision.l2_norm of every master as of the last launch with the norm fused."""
        if self._dn_pending:
            self._dn_done.synchronize()
            for j, i in enumerate(self._dn_idx):
                self.sumsq[i] = float(self._dn_host[j])
            self._dn_pending = False
        return [math.sqrt(v) for v in self.sumsq[:len(self.counts)]]

    def step(self, batch: int = 0, observe: bool | None = None, events=None) -> SyncResult:
        """One batch (training.py:207-254 order, as sync.WeightSync.step): the
        transfer of the masters at the widths in force, with their norms — the
        observation of the post-update masters of batch - 1 — then the AWP
        decision and, if a width escalated, the transfer again at the new widths."""
        if observe is None:
            observe = self.adaptive and batch > 0
        used = self.round_tos
        self.launch(fused_norm=observe, events=events)
        res = SyncResult(round_tos=used)
        if not observe:
            return res
        res.trace = self.schedule.observe_all(self.norms(), batch=batch - 1)
        new = self.schedule.round_tos()
        if new != used:
            self._plan(new)
            self.launch(fused_norm=False)
            res.round_tos = new
            res.repacked = True
        return res

    def observe_final(self, batch: int) -> list[tuple]:
        """The observation after the last update (training.py:246-254): the
        norms of the masters as they are now, from a host pass (no transfer).
        A fixed schedule observes nothing (training.py:246): no rows."""
        if not self.adaptive:
            return []
        segs = self._host_segs
        scratch = np.empty(self.layout.nbytes + 64, dtype=np.uint8)
        base = (-scratch.ctypes.data) % 64
        _lib.check(_lib.load().adt_pack_host(segs, len(self.counts), scratch.ctypes.data + base,
                                              self.sumsq.ctypes.data, self.threads))
        return self.schedule.observe_all(self.norms(), batch=batch)


def pack_host(masters: Sequence, round_tos: Sequence[int], threads: int = 0,
              align: int = 16) -> tuple[np.ndarray, PackedLayout, np.ndarray]:
    """adt_pack_host over host arrays: (packed stream as a uint8 array, its
    layout, per-layer float64 sums of squares). Same bytes as the device pack."""
    hosts = [_host_view(m, i) for i, m in enumerate(masters)]
    lay = PackedLayout.plan([h.size for h in hosts], round_tos, align=align)
    buf = np.empty(lay.nbytes + 64, dtype=np.uint8)
    base = (-buf.ctypes.data) % 64
    out = buf[base:base + lay.nbytes]
    ss = np.zeros(max(1, len(hosts)), dtype=np.float64)
    segs = _lib.segment_array([(h.ctypes.data if n else 0, n, off, r)
                               for h, n, off, r in zip(hosts, lay.counts, lay.offsets, lay.round_tos)])
    _lib.check(_lib.load().adt_pack_host(segs, len(hosts), out.ctypes.data, ss.ctypes.data, int(threads)))
    return out, lay, ss[:len(hosts)]


def host_threads() -> int:
    n = ctypes.c_int(0)
    _lib.check(_lib.load().adt_host_threads(ctypes.byref(n)))
    return int(n.value)
