"""Device engine: multi-tensor pack / unpack / norm launches through libadt.

Everything here is stream-ordered on the caller's (or torch's current) CUDA
stream; buffers are torch tensors so the caching allocator owns lifetimes and
the C side allocates nothing (include/adt.h).
"""

from __future__ import annotations

import ctypes
import threading
from typing import Sequence

import torch

from . import _lib
from .layout import PackedLayout


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2004_02297_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    _lib.load()


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_weight(t: torch.Tensor, count: int, what: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what}: expected a CUDA tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{what}: expected float32, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    if t.numel() != count:
        raise ValueError(f"{what}: {t.numel()} weights, layout says {count}")
    ptr = t.data_ptr()
    if count and ptr % 16:
        raise ValueError(f"{what}: data pointer not 16-byte aligned")
    return ptr


class SegmentTable:
    """A prepared adt_segment[] over fixed weight tensors and a layout.

    Building the table costs Python time proportional to the layer count, so
    long-lived callers (WeightSync, bench) build it once and reuse it.
    """

    def __init__(self, weights: Sequence[torch.Tensor], layout: PackedLayout, sources: Sequence[int] | None = None):
        """`sources[l]`: index of the buffer layer l's payload lives in (unpack_multi)."""
        if len(weights) != layout.num_layers:
            raise ValueError(f"{len(weights)} tensors for a {layout.num_layers}-layer layout")
        self.layout = layout
        self.tensors = list(weights)  # keep alive
        src = list(sources) if sources is not None else [0] * layout.num_layers
        segs = []
        for i, (t, n, off, r) in enumerate(zip(weights, layout.counts, layout.offsets, layout.round_tos)):
            segs.append((_check_weight(t, n, f"layer {i}"), n, off, r, src[i]))
        self.nseg = len(segs)
        self.array = _lib.segment_array(segs)
        self.npartials = _lib.partials_count(self.array, self.nseg)


class SgdTable:
    """A prepared adt_sgd_segment[] (masters, velocities, gradients, layout)."""

    def __init__(self, masters, velocities, grads, layout: PackedLayout):
        n = layout.num_layers
        if not (len(masters) == len(velocities) == len(grads) == n):
            raise ValueError("masters, velocities, grads and layout disagree on the layer count")
        self.layout = layout
        self.tensors = (list(masters), list(velocities), list(grads))
        self.nseg = n
        self.array = (_lib.SgdSegment * max(1, n))()
        for i, (w, v, g, cnt, off, r) in enumerate(zip(masters, velocities, grads, layout.counts,
                                                     layout.offsets, layout.round_tos)):
            a = self.array[i]
            a.weights = _check_weight(w, cnt, f"master {i}")
            a.velocity = _check_weight(v, cnt, f"velocity {i}")
            a.grad = _check_weight(g, cnt, f"grad {i}")
            a.count, a.offset, a.round_to, a.reserved = cnt, off, r, 0
        self.npartials = sum((c + _lib.TILE_WEIGHTS - 1) // _lib.TILE_WEIGHTS for c in layout.counts) \
            * _lib.PARTIALS_PER_TILE


def sgd_pack(table: SgdTable, lr: float, momentum: float, weight_decay: float, packed: torch.Tensor,
             sumsq: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
             partials: torch.Tensor | None = None) -> None:
    """adt_sgd_pack: W, v updated in place (reference rounding), W' packed,
    W' norm partials / per-layer sums fused in (see pack())."""
    if packed.dtype != torch.uint8 or not packed.is_cuda or packed.numel() < table.layout.payload_end:
        raise ValueError("packed must be a CUDA uint8 tensor covering every layer's payload")
    sh = stream_handle(stream)
    if partials is None and sumsq is not None:
        partials = _Scratch.get(packed.device, sh, table.npartials)
    _lib.check(_lib.load().adt_sgd_pack(table.array, table.nseg, float(lr), float(momentum), float(weight_decay),
                                        packed.data_ptr(), sumsq.data_ptr() if sumsq is not None else None,
                                        partials.data_ptr() if partials is not None else None, sh))


class ReduceSgdTable:
    """A prepared adt_grad_segment[] for adt_reduce_sgd_pack: per layer piece,
    the master and velocity views, the packed layout, and the byte offset of
    the piece's gradients inside every contribution buffer."""

    def __init__(self, masters, velocities, grad_offsets: Sequence[int], layout: PackedLayout):
        n = layout.num_layers
        if not (len(masters) == len(velocities) == len(grad_offsets) == n):
            raise ValueError("masters, velocities, grad offsets and layout disagree on the layer count")
        self.layout = layout
        self.tensors = (list(masters), list(velocities))
        self.nseg = n
        self.array = (_lib.GradSegment * max(1, n))()
        for i, (w, v, go, cnt, off, r) in enumerate(zip(masters, velocities, grad_offsets, layout.counts,
                                                        layout.offsets, layout.round_tos)):
            a = self.array[i]
            a.weights = _check_weight(w, cnt, f"master {i}")
            a.velocity = _check_weight(v, cnt, f"velocity {i}")
            if go % 16:
                raise ValueError(f"piece {i}: gradient offset {go} not 16-byte aligned")
            a.count, a.offset, a.grad_offset, a.round_to, a.reserved = cnt, off, int(go), r, 0
        self.npartials = sum((c + _lib.TILE_WEIGHTS - 1) // _lib.TILE_WEIGHTS for c in layout.counts) \
            * _lib.PARTIALS_PER_TILE


def _ptr(t) -> int | None:
    """Device address of an optional guard word (a torch tensor view) or None."""
    return t.data_ptr() if t is not None else None


def reduce_sgd_pack(table: ReduceSgdTable, grads: Sequence[int], sample_counts: Sequence[int], lr: float,
                    momentum: float, weight_decay: float, packed: torch.Tensor,
                    sumsq: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
                    partials: torch.Tensor | None = None, abort: torch.Tensor | None = None) -> None:
    """adt_reduce_sgd_pack: the contributions at device addresses `grads`
    (local buffers or peer buckets mapped by ipc_open) are combined as
    net.gather_and_update does, the masters/velocities stepped in place, the
    new masters packed (+ norm partials / per-layer sums, see pack())."""
    if len(grads) != len(sample_counts) or not 1 <= len(grads) <= _lib.MAX_SOURCES:
        raise ValueError(f"need 1..{_lib.MAX_SOURCES} contributions with one sample count each")
    if packed.dtype != torch.uint8 or not packed.is_cuda or packed.numel() < table.layout.payload_end:
        raise ValueError("packed must be a CUDA uint8 tensor covering every layer's payload")
    sh = stream_handle(stream)
    if partials is None and sumsq is not None:
        partials = _Scratch.get(packed.device, sh, table.npartials)
    counts = (ctypes.c_int64 * len(sample_counts))(*[int(c) for c in sample_counts])
    _lib.check(_lib.load().adt_reduce_sgd_pack(
        table.array, table.nseg, _lib.pointer_array(grads), counts, len(grads), float(lr), float(momentum),
        float(weight_decay), packed.data_ptr(), sumsq.data_ptr() if sumsq is not None else None,
        partials.data_ptr() if partials is not None else None, _ptr(abort), sh))


class _Scratch:
    """Per (device, stream) norm scratch: the float64 partials of one pass,
    one buffer per stream in use (a handful). A buffer handed to a kernel on
    stream S must not return to the caching allocator while S may still use
    it (it was allocated on whatever stream was current): an outgrown buffer
    is marked as used on S (record_stream) before it is dropped, so the
    allocator reuses its memory only after S's queued work completes."""

    _lock = threading.Lock()
    _cache: dict = {}

    @classmethod
    def get(cls, device: torch.device, stream: int, n: int) -> torch.Tensor:
        key = (device.index, stream)
        with cls._lock:
            cur = cls._cache.get(key)
            if cur is None or cur.numel() < max(1, n):
                if cur is not None:
                    cur.record_stream(torch.cuda.ExternalStream(stream, device=device))
                cur = torch.empty(max(1, n), dtype=torch.float64, device=device)
                cls._cache[key] = cur
            return cur


def _device_of(table: SegmentTable) -> torch.device:
    for t in table.tensors:
        return t.device
    return torch.device("cuda", torch.cuda.current_device())


def pack(table: SegmentTable, packed: torch.Tensor, sumsq: torch.Tensor | None = None,
         stream: torch.cuda.Stream | None = None, partials: torch.Tensor | None = None) -> None:
    """adt_pack: every layer of `table` into `packed` (uint8, covering every payload).

    sumsq (float64[L])       -> per-layer sums of squares fused in (finalize on the same stream);
    partials only (no sumsq) -> the pass stores its norm partials for a later
                                finalize(...) on another stream.
    """
    if packed.dtype != torch.uint8 or not packed.is_cuda or packed.numel() < table.layout.payload_end:
        raise ValueError("packed must be a CUDA uint8 tensor covering every layer's payload")
    sh = stream_handle(stream)
    if sumsq is not None and (sumsq.dtype != torch.float64 or not sumsq.is_cuda or sumsq.numel() < table.nseg):
        raise ValueError("sumsq must be a CUDA float64 tensor with one entry per layer")
    if partials is None and sumsq is not None:
        partials = _Scratch.get(packed.device, sh, table.npartials)
    if partials is not None and (partials.dtype != torch.float64 or partials.numel() < table.npartials):
        raise ValueError("partials must be a float64 tensor of table.npartials entries")
    _lib.check(_lib.load().adt_pack(table.array, table.nseg, packed.data_ptr(),
                                    sumsq.data_ptr() if sumsq is not None else None,
                                    partials.data_ptr() if partials is not None else None, sh))


def finalize(table: SegmentTable, partials: torch.Tensor, sumsq: torch.Tensor,
             stream: torch.cuda.Stream | None = None) -> None:
    """adt_norm_finalize: per-layer fixed-order sums of a pack pass's partials."""
    if sumsq.dtype != torch.float64 or not sumsq.is_cuda or sumsq.numel() < table.nseg:
        raise ValueError("sumsq must be a CUDA float64 tensor with one entry per layer")
    _lib.check(_lib.load().adt_norm_finalize(table.array, table.nseg, partials.data_ptr(), sumsq.data_ptr(),
                                             stream_handle(stream)))


def unpack(table: SegmentTable, packed: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """adt_unpack: `packed` (CUDA, or pinned host = zero-copy) into the table's tensors."""
    if packed.dtype != torch.uint8 or packed.numel() < table.layout.payload_end:
        raise ValueError("packed must be a uint8 tensor covering every layer's payload")
    if not packed.is_cuda and not packed.is_pinned():
        raise ValueError("packed must live on the device or in pinned (page-locked) host memory")
    _lib.check(_lib.load().adt_unpack(table.array, table.nseg, packed.data_ptr(), stream_handle(stream)))


def unpack_multi(table: SegmentTable, sources: Sequence[int], stream: torch.cuda.Stream | None = None,
                 start_seg: int = -1, abort: torch.Tensor | None = None) -> None:
    """adt_unpack_multi(_ex): layer l's payload read from sources[table source index]
    (raw device addresses: local buffers or peer buffers mapped by ipc_open);
    start_seg >= 0 rotates the tile walk to start just before that segment;
    abort: the peer barrier's timeout word (the kernel does nothing once it is set)."""
    arr = _lib.pointer_array(sources)
    if start_seg >= 0 or abort is not None:
        _lib.check(_lib.load().adt_unpack_multi_ex(table.array, table.nseg, arr, len(sources), None, int(start_seg),
                                                   _ptr(abort), stream_handle(stream)))
    else:
        _lib.check(_lib.load().adt_unpack_multi(table.array, table.nseg, arr, len(sources), stream_handle(stream)))


def copy_multi(dst: torch.Tensor, sources: Sequence[int], offset: int, nbytes: int,
               stream: torch.cuda.Stream | None = None, abort: torch.Tensor | None = None) -> None:
    """dst[q*nbytes:(q+1)*nbytes] = bytes [offset, offset+nbytes) of sources[q]."""
    if dst.dtype != torch.uint8 or not dst.is_cuda or dst.numel() < nbytes * len(sources):
        raise ValueError("dst must be a CUDA uint8 tensor of len(sources)*nbytes")
    arr = _lib.pointer_array(sources)
    _lib.check(_lib.load().adt_copy_multi(dst.data_ptr(), arr, len(sources), offset, nbytes, _ptr(abort),
                                          stream_handle(stream)))


def peer_barrier(flag_ptrs: Sequence[int], rank: int, state: torch.Tensor, timeout_s: float = 30.0,
                 stream: torch.cuda.Stream | None = None) -> None:
    """adt_peer_barrier: stream-ordered barrier over peer memory. flag_ptrs[q]
    = rank q's int32[nranks] epoch array mapped here; state = this rank's
    int32[2] (epoch counter, timeout epoch = the abort word of the guarded
    kernels behind it). The wait gives up after `timeout_s` of device time."""
    if state.dtype != torch.int32 or not state.is_cuda or state.numel() < 2:
        raise ValueError("state must be a CUDA int32 tensor of 2 entries")
    _lib.check(_lib.load().adt_peer_barrier(_lib.pointer_array(flag_ptrs), len(flag_ptrs), rank, state.data_ptr(),
                                            max(1, int(timeout_s * 1e9)), stream_handle(stream)))


def ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(CUDA IPC handle of the allocation holding `t`, t's byte offset inside it)."""
    lib = _lib.load()
    buf = ctypes.create_string_buffer(lib.adt_ipc_handle_bytes())
    off = ctypes.c_uint64(0)
    _lib.check(lib.adt_ipc_get_handle(t.data_ptr(), buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


_ipc_lock = threading.Lock()
_ipc_maps: dict = {}     # handle bytes -> [base address, refcount]
_ipc_bases: dict = {}    # base address -> handle bytes


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation; returns its base device address here.
    One mapping per allocation per process (a caching allocator may carve
    several exported buffers out of one allocation): reference counted."""
    with _ipc_lock:
        ent = _ipc_maps.get(handle)
        if ent is not None:
            ent[1] += 1
            return ent[0]
        lib = _lib.load()
        out = ctypes.c_void_p(0)
        _lib.check(lib.adt_ipc_open(ctypes.create_string_buffer(handle, len(handle)), ctypes.byref(out)))
        _ipc_maps[handle] = [int(out.value), 1]
        _ipc_bases[int(out.value)] = handle
        return int(out.value)


def ipc_close(ptr: int) -> None:
    with _ipc_lock:
        handle = _ipc_bases.get(ptr)
        if handle is not None:
            ent = _ipc_maps[handle]
            ent[1] -= 1
            if ent[1] > 0:
                return
            del _ipc_maps[handle]
            del _ipc_bases[ptr]
        _lib.check(_lib.load().adt_ipc_close(ptr))


def sumsq(table: SegmentTable, out: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """adt_sumsq: float64 sum of squares of every layer (norm-only pass)."""
    if out.dtype != torch.float64 or not out.is_cuda or out.numel() < table.nseg:
        raise ValueError("out must be a CUDA float64 tensor with one entry per layer")
    sh = stream_handle(stream)
    parts = _Scratch.get(out.device, sh, table.npartials)
    _lib.check(_lib.load().adt_sumsq(table.array, table.nseg, out.data_ptr(), parts.data_ptr(), sh))


def sumsq_f64(x: torch.Tensor, out: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """adt_sumsq_f64: out[0] = float64 sum of squares of the float64 CUDA tensor x."""
    if x.dtype != torch.float64 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("x must be a contiguous CUDA float64 tensor")
    if out.dtype != torch.float64 or not out.is_cuda or out.numel() < 1:
        raise ValueError("out must be a CUDA float64 tensor")
    lib = _lib.load()
    np_ = ctypes.c_uint64(0)
    _lib.check(lib.adt_sumsq_f64_partials(x.numel(), ctypes.byref(np_)))
    sh = stream_handle(stream)
    parts = _Scratch.get(x.device, sh, int(np_.value))
    _lib.check(lib.adt_sumsq_f64(x.data_ptr() if x.numel() else None, x.numel(), parts.data_ptr(), out.data_ptr(),
                                 sh))


def roundtrip_max_tiles() -> int:
    v = ctypes.c_int(0)
    _lib.check(_lib.load().adt_roundtrip_max_tiles(ctypes.byref(v)))
    return int(v.value)


def roundtrip(masters: SegmentTable, replicas: SegmentTable, packed: torch.Tensor, sumsq: torch.Tensor | None,
              partials: torch.Tensor, barrier: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """adt_roundtrip: the whole single-GPU step of a small set in one launch
    (pack with fused norms -> grid barrier -> unpack -> per-layer sums)."""
    if barrier.dtype != torch.int32 or not barrier.is_cuda or barrier.numel() < 2:
        raise ValueError("barrier must be a CUDA int32 tensor of 2 zeros")
    _lib.check(_lib.load().adt_roundtrip(masters.array, replicas.array, masters.nseg, packed.data_ptr(),
                                         sumsq.data_ptr() if sumsq is not None else None, partials.data_ptr(),
                                         barrier.data_ptr(), stream_handle(stream)))


def sm_count() -> int:
    v = ctypes.c_int(0)
    _lib.check(_lib.load().adt_device_sm_count(ctypes.byref(v)))
    return int(v.value)


# ------------------------------------------------- device-resident AWP step
def pack_dyn(table: SegmentTable, packed: torch.Tensor, widths: torch.Tensor, partials: torch.Tensor | None = None,
             stream: torch.cuda.Stream | None = None) -> None:
    """adt_pack_dyn: capacity-layout table (round_to 4), per-layer widths read
    from the device uint8 tensor `widths`; optional norm partials."""
    _lib.check(_lib.load().adt_pack_dyn(table.array, table.nseg, packed.data_ptr(),
                                        partials.data_ptr() if partials is not None else None,
                                        widths.data_ptr(), stream_handle(stream)))


def unpack_dyn(table: SegmentTable, packed: torch.Tensor, widths: torch.Tensor,
               stream: torch.cuda.Stream | None = None) -> None:
    """adt_unpack_dyn: the inverse of pack_dyn at the same device widths."""
    _lib.check(_lib.load().adt_unpack_dyn(table.array, table.nseg, packed.data_ptr(), widths.data_ptr(),
                                          stream_handle(stream)))


def awp_observe(sumsq: torch.Tensor, device_struct, config_struct, stream: torch.cuda.Stream | None = None,
                abort: torch.Tensor | None = None) -> None:
    """adt_awp_observe: one device-side AWP observation of every layer."""
    _lib.check(_lib.load().adt_awp_observe(sumsq.data_ptr(), ctypes.byref(device_struct), ctypes.byref(config_struct),
                                           _ptr(abort), stream_handle(stream)))


def awp_fixup(masters: SegmentTable, replicas: SegmentTable, packed: torch.Tensor, escalated: torch.Tensor,
              widths_new: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
    """adt_awp_fixup: re-pack + re-unpack the layers adt_awp_observe listed as escalated."""
    _lib.check(_lib.load().adt_awp_fixup(masters.array, replicas.array, masters.nseg, packed.data_ptr(),
                                         escalated.data_ptr(), widths_new.data_ptr(), stream_handle(stream)))


def sgd_pack_dyn(table: SgdTable, lr: float, momentum: float, weight_decay: float, packed: torch.Tensor,
                 widths: torch.Tensor, partials: torch.Tensor | None = None,
                 stream: torch.cuda.Stream | None = None) -> None:
    """adt_sgd_pack_dyn: the fused update + pack at device-resident widths (capacity layout)."""
    _lib.check(_lib.load().adt_sgd_pack_dyn(table.array, table.nseg, float(lr), float(momentum), float(weight_decay),
                                            packed.data_ptr(), partials.data_ptr() if partials is not None else None,
                                            widths.data_ptr(), stream_handle(stream)))


def reduce_sgd_pack_dyn(table: ReduceSgdTable, grads: Sequence[int], sample_counts: Sequence[int], lr: float,
                        momentum: float, weight_decay: float, packed: torch.Tensor, widths: torch.Tensor,
                        partials: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
                        abort: torch.Tensor | None = None) -> None:
    """adt_reduce_sgd_pack_dyn: gradient combine + update + pack at device-resident widths."""
    if len(grads) != len(sample_counts) or not 1 <= len(grads) <= _lib.MAX_SOURCES:
        raise ValueError(f"need 1..{_lib.MAX_SOURCES} contributions with one sample count each")
    counts = (ctypes.c_int64 * len(sample_counts))(*[int(c) for c in sample_counts])
    _lib.check(_lib.load().adt_reduce_sgd_pack_dyn(
        table.array, table.nseg, _lib.pointer_array(grads), counts, len(grads), float(lr), float(momentum),
        float(weight_decay), packed.data_ptr(), partials.data_ptr() if partials is not None else None,
        widths.data_ptr(), _ptr(abort), stream_handle(stream)))


def _int32_array(values) -> ctypes.Array:
    arr = (ctypes.c_int32 * max(1, len(values)))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr


def unpack_multi_dyn(table: SegmentTable, sources: Sequence[int], widths: torch.Tensor,
                     stream: torch.cuda.Stream | None = None, start_seg: int = -1,
                     abort: torch.Tensor | None = None) -> None:
    """adt_unpack_multi_ex with device widths: gather-unpack with per-piece
    widths from device memory (and an optional rotated tile walk)."""
    _lib.check(_lib.load().adt_unpack_multi_ex(table.array, table.nseg, _lib.pointer_array(sources), len(sources),
                                               widths.data_ptr(), int(start_seg), _ptr(abort), stream_handle(stream)))


def awp_combine(tails: torch.Tensor, piece_layer: torch.Tensor, nlayers: int, sumsq: torch.Tensor,
                stream: torch.cuda.Stream | None = None, abort: torch.Tensor | None = None) -> None:
    """adt_awp_combine: per-layer sums from the gathered per-piece sums, rank-major order."""
    _lib.check(_lib.load().adt_awp_combine(tails.data_ptr(), piece_layer.numel(), piece_layer.data_ptr(), nlayers,
                                           sumsq.data_ptr(), _ptr(abort), stream_handle(stream)))


def awp_fixup_pieces(masters: SegmentTable, replicas: SegmentTable, seg_layer: Sequence[int], packed: torch.Tensor,
                     escalated: torch.Tensor, widths_new: torch.Tensor,
                     stream: torch.cuda.Stream | None = None, abort: torch.Tensor | None = None) -> None:
    """adt_awp_fixup_pieces: re-pack this rank's escalated pieces into its send buffer."""
    _lib.check(_lib.load().adt_awp_fixup_pieces(masters.array, replicas.array, masters.nseg, _int32_array(seg_layer),
                                                packed.data_ptr(), escalated.data_ptr(), widths_new.data_ptr(),
                                                _ptr(abort), stream_handle(stream)))


def awp_fixup_gather(replicas: SegmentTable, seg_layer: Sequence[int], sources: Sequence[int],
                     escalated: torch.Tensor, widths_new: torch.Tensor,
                     stream: torch.cuda.Stream | None = None, abort: torch.Tensor | None = None) -> None:
    """adt_awp_fixup_gather: re-unpack every rank's escalated pieces from their send buffers."""
    _lib.check(_lib.load().adt_awp_fixup_gather(replicas.array, replicas.nseg, _int32_array(seg_layer),
                                                _lib.pointer_array(sources), len(sources), escalated.data_ptr(),
                                                widths_new.data_ptr(), _ptr(abort), stream_handle(stream)))
