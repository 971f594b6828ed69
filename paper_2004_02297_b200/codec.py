"""Drop-in ADT codec: the reference `weightpack.codec` API on B200 kernels.

Same names, signatures, byte layout and exceptions as
/root/reference/pkg/src/weightpack/codec.py (cited per function). The
difference is where the bytes move: every pack/unpack runs the sm_100a
kernels in libadt.so. Inputs may be anything the reference accepts
(array-likes are cast to float32 with round-to-nearest-even and flattened in
row-major order, codec.py:110-113) or CUDA tensors, which stay on the device:

* host input  -> PackedBlock whose payload is `bytes` (as in the reference);
* CUDA tensor -> PackedBlock whose payload is a CUDA uint8 tensor (no copy to
  the host). `block.payload_bytes()` materialises it; equality compares bytes.

The batched entry points `pack_many` / `unpack_many` are the hot path: one
launch for all layers, norms fused into the pack.
"""

from __future__ import annotations

import struct
import warnings
from typing import BinaryIO, Sequence

import numpy as np
import torch

from . import engine, hostio
from .layout import PackedLayout, align_up

WORD_BYTES = 4
MIN_ROUND_TO = 1
MAX_ROUND_TO = 4
VECTOR_GROUP = 8  # codec.py:31 — kept for API parity (the GPU tile is 4096 weights)

STREAM_MAGIC = b"ADT1"
STREAM_VERSION = 1
_HEADER = struct.Struct("<4sBBQ")  # magic, version, round_to, weight_count (codec.py:33-36)
STREAM_HEADER_BYTES = _HEADER.size


class MalformedBlock(ValueError):
    """Raised when a packed block or stream is internally inconsistent (codec.py:48-49)."""


def check_round_to(round_to) -> int:
    """codec.py:52-57: an integer-valued byte count in [1, 4]."""
    try:
        r = int(round_to)
    except (TypeError, ValueError):
        raise ValueError(f"round_to must be an integer in [1, 4], got {round_to!r}") from None
    if r != round_to or r < MIN_ROUND_TO or r > MAX_ROUND_TO:
        raise ValueError(f"round_to must be an integer in [1, 4], got {round_to!r}")
    return r


def bits_to_round_to(bits: int) -> int:
    """codec.py:60-67: whole bytes that keep `bits` bits (14 -> 2)."""
    if not 1 <= bits <= 32:
        raise ValueError(f"bits must be in [1, 32], got {bits}")
    return (int(bits) + 7) // 8


def truncation_mask(round_to: int) -> int:
    """codec.py:70-73: the r*8 high bits a round trip preserves."""
    r = check_round_to(round_to)
    return (0xFFFFFFFF << (8 * (WORD_BYTES - r))) & 0xFFFFFFFF


class PackedBlock:
    """codec.py:76-107 — (round_to, weight_count, payload), immutable.

    `payload` is `bytes` for host-produced blocks or a CUDA uint8 tensor for
    device-resident ones; both must hold exactly weight_count*round_to bytes.
    """

    __slots__ = ("round_to", "weight_count", "payload")

    def __init__(self, round_to: int, weight_count: int, payload):
        r = check_round_to(round_to)
        if weight_count < 0:
            raise MalformedBlock(f"negative weight_count {weight_count}")
        if isinstance(payload, torch.Tensor):
            if payload.dtype != torch.uint8 or payload.dim() != 1:
                raise MalformedBlock("device payload must be a 1-D uint8 tensor")
            size = payload.numel()
        else:
            payload = bytes(payload)
            size = len(payload)
        expected = weight_count * r
        if size != expected:
            raise MalformedBlock(
                f"payload holds {size} bytes, expected {weight_count} weights * {r} = {expected}")
        object.__setattr__(self, "round_to", r)
        object.__setattr__(self, "weight_count", int(weight_count))
        object.__setattr__(self, "payload", payload)

    def __setattr__(self, name, value):
        raise AttributeError("PackedBlock is immutable")

    @property
    def on_device(self) -> bool:
        return isinstance(self.payload, torch.Tensor)

    def payload_bytes(self) -> bytes:
        if self.on_device:
            return hostio.to_bytes(self.payload)
        return self.payload

    def to_host(self) -> "PackedBlock":
        return self if not self.on_device else PackedBlock(self.round_to, self.weight_count, self.payload_bytes())

    @property
    def raw_bytes(self) -> int:
        """codec.py:99-102."""
        return self.weight_count * WORD_BYTES

    @property
    def wire_bytes(self) -> int:
        """codec.py:104-107: payload plus the 14-byte stream header."""
        return STREAM_HEADER_BYTES + self.weight_count * self.round_to

    def __eq__(self, other):
        if not isinstance(other, PackedBlock):
            return NotImplemented
        return (self.round_to == other.round_to and self.weight_count == other.weight_count
                and self.payload_bytes() == other.payload_bytes())

    def __hash__(self):
        return hash((self.round_to, self.weight_count, self.payload_bytes()))

    def __repr__(self):
        where = "cuda" if self.on_device else "host"
        return f"PackedBlock(round_to={self.round_to}, weight_count={self.weight_count}, payload=<{where} {self.weight_count * self.round_to} B>)"


# ------------------------------------------------------------------ inputs
def _device_words(weights) -> tuple[torch.Tensor, bool]:
    """codec.py:110-113 semantics -> (flat float32 CUDA tensor, came_from_device)."""
    engine.require_cuda()
    if isinstance(weights, torch.Tensor) and weights.is_cuda:
        t = weights.detach()
        if t.dtype != torch.float32:
            t = t.to(torch.float32)  # round-to-nearest-even, like astype(float32)
        t = t.contiguous().reshape(-1)
        if t.numel() and t.data_ptr() % 16:
            t = t.clone()
        return t, True
    if isinstance(weights, torch.Tensor):
        weights = weights.detach().numpy()
    host = np.ascontiguousarray(weights, dtype=np.float32).reshape(-1)
    if host.size == 0:
        return torch.empty(0, dtype=torch.float32, device="cuda"), False
    return hostio.to_device(host), False


def _pack_device(flat: torch.Tensor, r: int) -> torch.Tensor:
    n = flat.numel()
    layout = PackedLayout.plan([n], [r])
    out = torch.empty(max(16, layout.nbytes), dtype=torch.uint8, device=flat.device)
    engine.pack(engine.SegmentTable([flat], layout), out)
    return out[: n * r]


# -------------------------------------------------------------- per layer
def _host_words(weights) -> np.ndarray | None:
    """codec.py:110-113 for a host input: the flat float32 words, or None for
    a CUDA tensor."""
    if isinstance(weights, torch.Tensor):
        if weights.is_cuda:
            return None
        weights = weights.detach().numpy()
    return np.ascontiguousarray(weights, dtype=np.float32).reshape(-1)


def _pack_host_small(host: np.ndarray, r: int) -> PackedBlock:
    """A small host array (< hostio.SMALL bytes): one H2D, the pack kernel and
    one D2H queued back to back, one stream sync (hostio.small_call)."""
    n = host.size
    layout = PackedLayout.plan([n], [r])

    def fn(d_in, d_out):
        engine.pack(engine.SegmentTable([d_in[:4 * n].view(torch.float32)], layout), d_out)

    return PackedBlock(r, n, hostio.small_call(host, n * r, fn).tobytes())


def pack(weights, round_to: int) -> PackedBlock:
    """codec.py:116-130 (scalar reference) — here one multi-tensor kernel launch."""
    r = check_round_to(round_to)
    engine.require_cuda()
    host = _host_words(weights)
    if host is not None and 0 < host.nbytes < hostio.SMALL:
        return _pack_host_small(host, r)
    flat, on_dev = _device_words(weights)
    payload = _pack_device(flat, r)
    if on_dev:
        return PackedBlock(r, flat.numel(), payload)
    return PackedBlock(r, flat.numel(), hostio.to_bytes(payload))


def pack_vectorized(weights, round_to: int) -> PackedBlock:
    """codec.py:149-153 — identical bytes to pack() (same kernel)."""
    return pack(weights, round_to)


def pack_parallel(weights, round_to: int, worker_count: int) -> PackedBlock:
    """codec.py:156-180 — worker_count is validated; the output never depends
    on it, and the GPU tile partition is likewise invisible."""
    check_round_to(round_to)
    if worker_count < 1:
        raise ValueError(f"worker_count must be >= 1, got {worker_count}")
    return pack(weights, round_to)


def unpack(block: PackedBlock):
    """codec.py:183-197 — fresh writable float32 weights, low bytes zero.

    Host blocks return a numpy array (as the reference); device blocks return
    a CUDA float32 tensor.
    """
    r = check_round_to(block.round_to)
    n = block.weight_count
    size = block.payload.numel() if block.on_device else len(block.payload)
    if size != n * r:
        raise MalformedBlock(f"payload holds {size} bytes, expected {n * r}")
    engine.require_cuda()
    layout = PackedLayout.plan([n], [r])
    if n == 0:
        return torch.empty(0, dtype=torch.float32, device="cuda") if block.on_device else np.zeros(0, dtype=np.float32)
    if not block.on_device and 4 * n < hostio.SMALL:
        def fn(d_in, d_out):     # one H2D of the payload, the unpack, one D2H of the words, one sync
            engine.unpack(engine.SegmentTable([d_out[:4 * n].view(torch.float32)], layout), d_in)

        words = hostio.small_call(np.frombuffer(block.payload, dtype=np.uint8), 4 * n, fn)
        return words.view(np.float32).copy()            # a fresh writable array (codec.py:186)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    if block.on_device:
        src = block.payload
        if src.data_ptr() % 16:
            src = src.clone()
    else:
        with warnings.catch_warnings():  # read-only bytes: the view is only ever read (copied to the device)
            warnings.simplefilter("ignore", UserWarning)
            src = hostio.to_device(np.frombuffer(block.payload, dtype=np.uint8))
    engine.unpack(engine.SegmentTable([out], layout), src)
    return out if block.on_device else hostio.to_numpy_f32(out)


# ------------------------------------------------------------ container
def write_stream(stream: BinaryIO, block: PackedBlock) -> int:
    """codec.py:200-205 — '<4sBBQ' header then payload; returns bytes written."""
    header = _HEADER.pack(STREAM_MAGIC, STREAM_VERSION, block.round_to, block.weight_count)
    payload = block.payload_bytes()
    stream.write(header)
    stream.write(payload)
    return len(header) + len(payload)


def read_stream(stream: BinaryIO) -> PackedBlock:
    """codec.py:208-240 — validate the container, with byte-offset diagnostics."""
    header = stream.read(STREAM_HEADER_BYTES)
    if len(header) < STREAM_HEADER_BYTES:
        raise MalformedBlock(
            f"truncated header: stream ends at byte {len(header)}, need {STREAM_HEADER_BYTES}")
    magic, version, r, count = _HEADER.unpack(header)
    if magic != STREAM_MAGIC:
        raise MalformedBlock(f"bad magic {magic!r} at offset 0, expected {STREAM_MAGIC!r}")
    if version != STREAM_VERSION:
        raise MalformedBlock(f"unsupported version {version} at offset 4")
    if not MIN_ROUND_TO <= r <= MAX_ROUND_TO:
        raise MalformedBlock(f"round_to byte {r} at offset 5 outside [1, 4]")
    want = count * r
    payload = stream.read(want + 1)
    if len(payload) < want:
        raise MalformedBlock(
            f"truncated payload: stream ends at byte {STREAM_HEADER_BYTES + len(payload)}, "
            f"declared count {count} needs {want} payload bytes")
    if len(payload) > want:
        raise MalformedBlock(
            f"trailing data at offset {STREAM_HEADER_BYTES + want}: "
            f"declared count {count} accounts for only {want} payload bytes")
    return PackedBlock(r, count, payload)


# ------------------------------------------------------------ multi-tensor
def pack_many(weights: Sequence[torch.Tensor], round_tos: Sequence[int], *, with_norms: bool = False,
              out: torch.Tensor | None = None):
    """All layers in ONE launch: returns (packed uint8 buffer, layout, sumsq or None).

    Layer l's PackedBlock payload is packed[layout.span(l)]; with_norms fuses
    the float64 per-layer sums of squares (precision.l2_norm = sqrt) into the pass.
    """
    rs = [check_round_to(r) for r in round_tos]
    flats = []
    for w in weights:
        f, _ = _device_words(w)
        flats.append(f)
    layout = PackedLayout.plan([f.numel() for f in flats], rs)
    if out is None:
        out = torch.empty(max(16, layout.nbytes), dtype=torch.uint8, device="cuda")
    ss = torch.empty(len(flats), dtype=torch.float64, device="cuda") if with_norms else None
    engine.pack(engine.SegmentTable(flats, layout), out, ss)
    return out, layout, ss


def blocks_of(packed: torch.Tensor, layout: PackedLayout) -> list[PackedBlock]:
    """Per-layer device PackedBlocks viewing a pack_many buffer (no copies)."""
    return [PackedBlock(r, n, packed[layout.span(i)[0]:layout.span(i)[1]])
            for i, (n, r) in enumerate(zip(layout.counts, layout.round_tos))]


def unpack_many(packed: torch.Tensor, layout: PackedLayout, out: Sequence[torch.Tensor] | None = None):
    """Inverse of pack_many in one launch; returns the list of flat float32 tensors."""
    if out is None:
        out = [torch.empty(n, dtype=torch.float32, device="cuda") for n in layout.counts]
    engine.unpack(engine.SegmentTable(list(out), layout), packed)
    return list(out)


__all__ = [
    "WORD_BYTES", "MIN_ROUND_TO", "MAX_ROUND_TO", "VECTOR_GROUP", "STREAM_MAGIC", "STREAM_VERSION",
    "STREAM_HEADER_BYTES", "MalformedBlock", "check_round_to", "bits_to_round_to", "truncation_mask",
    "PackedBlock", "pack", "pack_vectorized", "pack_parallel", "unpack", "write_stream", "read_stream",
    "pack_many", "unpack_many", "blocks_of", "align_up",
]
