"""Wire-byte accounting of the weight stream.

The reference's `send_weights` (transfer.py:143-174) moves no data; it
records, per worker and layer, wire = 14-byte ADT1 header + n·r payload +
raw bias bytes, raw = 4n + bias bytes, and models the link time. Its ledger,
link and codec cost models are simulation (out of scope here); what carries
over is the byte arithmetic, which this module keeps identical so a B200 run
reports the same wire/raw figures the reference's ledger would — next to the
bytes the device path actually moves (payload only: the 16-byte alignment pad
and the headers never cross NVLink or PCIe).
"""

from __future__ import annotations

from dataclasses import dataclass

from .codec import STREAM_HEADER_BYTES, PackedBlock
from .layout import PackedLayout


@dataclass(frozen=True)
class WireRecord:
    """transfer.py:143-174 send_weights record (the byte fields)."""

    layer: int
    raw_bytes: int          # 4n + bias
    wire_bytes: int         # 14 + n·r + bias
    weight_raw_bytes: int   # 4n
    weight_wire_bytes: int  # 14 + n·r


def send_weights_bytes(block: PackedBlock, *, layer: int = 0, bias_bytes: int = 0) -> WireRecord:
    """The byte fields send_weights would record for `block` (transfer.py:160-171)."""
    return WireRecord(layer, block.raw_bytes + bias_bytes, block.wire_bytes + bias_bytes,
                      block.raw_bytes, block.wire_bytes)


def layout_records(layout: PackedLayout, bias_bytes=None) -> list[WireRecord]:
    """One record per layer of a multi-tensor pack (one worker)."""
    bias = list(bias_bytes) if bias_bytes is not None else [0] * layout.num_layers
    out = []
    for i, (n, r) in enumerate(zip(layout.counts, layout.round_tos)):
        raw, wire = 4 * n, STREAM_HEADER_BYTES + n * r
        out.append(WireRecord(i, raw + bias[i], wire + bias[i], raw, wire))
    return out


def weight_stream_ratio(records) -> float:
    """raw / wire over the weight stream (transfer.py:119-132, TransferLedger.weight_stream_bytes/ratio)."""
    raw = sum(r.weight_raw_bytes for r in records)
    wire = sum(r.weight_wire_bytes for r in records)
    if wire == 0:
        raise ValueError("no to-worker weight transfers recorded")
    return raw / wire
