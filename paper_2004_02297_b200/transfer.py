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


def return_gradients_bytes(parameter_count: int) -> WireRecord:
    """transfer.py:177-197, 247-251 (TransferBoundary.return_gradients ->
    send_to_host): one worker's gradients go back uncompressed — raw = wire =
    4 bytes per parameter, recorded for all layers at once (layer "all" -> -1
    here). On the B200 path these bytes are what the fused gradient reduce
    reads from every rank's bucket (peer loads or the all-to-all)."""
    if parameter_count < 0:
        raise ValueError(f"parameter_count must be >= 0, got {parameter_count}")
    nbytes = 4 * int(parameter_count)
    return WireRecord(-1, nbytes, nbytes, 0, 0)


def weight_stream_ratio(records) -> float:
    """raw / wire over the weight stream (transfer.py:119-132, TransferLedger.weight_stream_bytes/ratio)."""
    raw = sum(r.weight_raw_bytes for r in records)
    wire = sum(r.weight_wire_bytes for r in records)
    if wire == 0:
        raise ValueError("no to-worker weight transfers recorded")
    return raw / wire


def _loop_ms(fn, reps: int = 20, rounds: int = 5) -> float:
    """Device ms per call of `fn` (stream work only), from one CUDA graph of
    `reps` back-to-back calls replayed `rounds` times between two events."""
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(rounds):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (reps * rounds)


def measured_profile(sync, bias_bytes=None) -> dict:
    """The reference's per-phase profile (transfer.py:254-286, `profile_report`)
    with MEASURED B200 device times in place of its LinkModel / CodecCostModel,
    for one WeightSync step — the rows of the paper's Table 2:
    pack (with and without the fused l2-norm), unpack, standalone l2-norm, and the
    CPU->GPU weight transfer from pinned host memory, FP32 vs ADT-packed
    (memcpy + unpack, and the zero-copy unpack)."""
    import torch
    from . import engine
    lay = sync.layout
    pack_norm, fin_unpack = sync.phase_ms(True)
    pack_only, unpack_only = sync.phase_ms(False)
    sums = torch.empty(len(sync.masters), dtype=torch.float64, device=sync.device)
    norm_only = _loop_ms(lambda: engine.sumsq(sync.pack_table, sums))
    host_packed = torch.empty(lay.nbytes, dtype=torch.uint8, pin_memory=True)
    host_packed.copy_(sync.packed[:lay.nbytes])
    dev_packed = torch.empty(lay.nbytes, dtype=torch.uint8, device=sync.device)
    # FP32 side as one contiguous pinned buffer, like the packed stream (one copy each)
    host_fp32 = torch.cat([m.reshape(-1) for m in sync.masters]).cpu().pin_memory()
    dev_fp32 = torch.empty_like(host_fp32, device=sync.device)

    def raw_h2d():
        dev_fp32.copy_(host_fp32, non_blocking=True)

    def packed_h2d():
        dev_packed.copy_(host_packed, non_blocking=True)

    t_raw = _loop_ms(raw_h2d, reps=4, rounds=3)
    t_pk = _loop_ms(packed_h2d, reps=4, rounds=3)
    t_zc = _loop_ms(lambda: engine.unpack(sync.unpack_table, host_packed), reps=4, rounds=3)
    recs = layout_records(lay, bias_bytes)
    ms = 1e-3
    return {
        "phases": {
            "pack": {"device_s": pack_only * ms, "with_fused_l2_norm_s": pack_norm * ms},
            "unpack": {"device_s": unpack_only * ms, "with_concurrent_finalize_s": fin_unpack * ms},
            "l2_norm": {"fused_extra_s": max(0.0, pack_norm - pack_only) * ms, "standalone_s": norm_only * ms},
            "to_worker": {"raw_fp32_h2d_s": t_raw * ms, "packed_h2d_s": t_pk * ms,
                          "packed_h2d_plus_unpack_s": (t_pk + unpack_only) * ms,
                          "zero_copy_unpack_s": t_zc * ms},
        },
        "wire_bytes": {"to_worker": sum(r.wire_bytes for r in recs)},
        "raw_bytes": {"to_worker": sum(r.raw_bytes for r in recs)},
        "weight_stream": {"raw_bytes": sum(r.weight_raw_bytes for r in recs),
                          "wire_bytes": sum(r.weight_wire_bytes for r in recs),
                          "ratio": weight_stream_ratio(recs)},
    }
