"""Wire-byte accounting and the measured transfer ledger (SURVEY.md §8a row
A14, §8f item 3).

The reference's `send_weights` (transfer.py:143-174) moves no data; it
records, per worker and layer, wire = 14-byte ADT1 header + n·r payload +
raw bias bytes, raw = 4n + bias bytes, and MODELS the link and codec time
(LinkModel, CodecCostModel). Here the byte arithmetic is kept identical and
the times are MEASURED (CUDA events, host wall clock): `TransferLedger`,
`write_csv` (LEDGER_HEADER) and `profile_report` reproduce the reference's
schemas (transfer.py:19-140, 254-286) so its report tooling reads a B200 run;
`LedgerRecorder` fills them from a running WeightSync / HostWeightSync. The
payload bytes are what the device path actually moves (the 16-byte alignment
pad and the headers never cross NVLink or PCIe).
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


# ------------------------------------------------ measured ledger (§8f item 3)
# The reference's ledger schema (transfer.py:19-140) and run profile
# (transfer.py:254-286), filled with MEASURED B200 times in place of its
# LinkModel / CodecCostModel: CUDA events around the device kernels, wall
# clock around the host packer. The byte columns are the reference's
# arithmetic (send_weights / send_to_host) unchanged, so a reference report
# (report.py) reads these files as it reads its own.

TO_WORKER = "to_worker"
TO_HOST = "to_host"
LEDGER_HEADER = ("batch", "direction", "layer", "raw_bytes", "wire_bytes", "pack_s", "unpack_s", "link_s")
PHASES = ("to_worker", "to_host", "forward", "backward", "update", "l2_norm", "pack", "unpack")


class EmptyLedger(ValueError):
    """transfer.py:34-35 — a report was requested for a ledger with no records."""


@dataclass(frozen=True)
class TransferRecord:
    """transfer.py:59-78: one boundary crossing; `layer` is an index or "all".
    pack_seconds / unpack_seconds / link_seconds are measured here."""

    batch: int
    direction: str
    layer: int | str
    raw_bytes: int
    wire_bytes: int
    pack_seconds: float
    unpack_seconds: float
    link_seconds: float
    weight_raw_bytes: int = 0
    weight_wire_bytes: int = 0


class TransferLedger:
    """transfer.py:81-140: append-only log with the same aggregation helpers
    and the same CSV text (write_csv), records from several threads allowed."""

    def __init__(self) -> None:
        import threading
        self._records: list[TransferRecord] = []
        self._lock = threading.Lock()

    def append(self, record: TransferRecord) -> None:
        with self._lock:
            self._records.append(record)

    def __len__(self) -> int:
        return len(self._records)

    @property
    def records(self) -> tuple[TransferRecord, ...]:
        return tuple(self._records)

    def _select(self, direction):
        return self._records if direction is None else [r for r in self._records if r.direction == direction]

    def total_wire_bytes(self, direction: str | None = None) -> int:
        return sum(r.wire_bytes for r in self._select(direction))

    def total_raw_bytes(self, direction: str | None = None) -> int:
        return sum(r.raw_bytes for r in self._select(direction))

    def total_link_seconds(self, direction: str | None = None) -> float:
        return sum(r.link_seconds for r in self._select(direction))

    def total_pack_seconds(self) -> float:
        return sum(r.pack_seconds for r in self._records)

    def total_unpack_seconds(self) -> float:
        return sum(r.unpack_seconds for r in self._records)

    def weight_stream_bytes(self) -> tuple[int, int]:
        sel = self._select(TO_WORKER)
        return sum(r.weight_raw_bytes for r in sel), sum(r.weight_wire_bytes for r in sel)

    def weight_stream_ratio(self) -> float:
        raw, wire = self.weight_stream_bytes()
        if wire == 0:
            raise EmptyLedger("no to-worker weight transfers recorded")
        return raw / wire

    def write_csv(self, stream) -> None:
        """transfer.py:134-140: header line, then one line per record (floats as repr)."""
        stream.write(",".join(LEDGER_HEADER) + "\n")
        for r in self._records:
            stream.write(f"{r.batch},{r.direction},{r.layer},{r.raw_bytes},{r.wire_bytes},"
                         f"{r.pack_seconds!r},{r.unpack_seconds!r},{r.link_seconds!r}\n")


def record_weights(ledger: TransferLedger, *, batch: int, layer: int, count: int, round_to: int, bias_bytes: int = 0,
                   pack_seconds: float = 0.0, unpack_seconds: float = 0.0, link_seconds: float = 0.0) -> TransferRecord:
    """send_weights (transfer.py:143-174) for one layer: wire = 14 + n*r + bias, raw = 4n + bias."""
    raw, wire = 4 * count, STREAM_HEADER_BYTES + count * round_to
    rec = TransferRecord(batch, TO_WORKER, layer, raw + bias_bytes, wire + bias_bytes, float(pack_seconds),
                         float(unpack_seconds), float(link_seconds), raw, wire)
    ledger.append(rec)
    return rec


def record_gradients(ledger: TransferLedger, *, batch: int, parameter_count: int,
                     link_seconds: float = 0.0) -> TransferRecord:
    """send_to_host via TransferBoundary.return_gradients (transfer.py:177-197, 247-251):
    raw = wire = 4 * parameter_count, layer "all"."""
    n = 4 * int(parameter_count)
    rec = TransferRecord(batch, TO_HOST, "all", n, n, 0.0, 0.0, float(link_seconds))
    ledger.append(rec)
    return rec


def profile_report(ledger: TransferLedger, wall_times) -> dict:
    """transfer.py:254-286, the same keys: phases[name]["wall_s"] for every
    PHASES name, the transfer phases' "modeled_link_s" and the codec phases'
    "modeled_s" (here: the MEASURED sums from the ledger, under the
    reference's key names so report.py reads it), and the byte totals."""
    if len(ledger) == 0:
        raise EmptyLedger("ledger has no records")
    phases = {name: {"wall_s": float(wall_times.get(name, 0.0))} for name in PHASES}
    phases["to_worker"]["modeled_link_s"] = ledger.total_link_seconds(TO_WORKER)
    phases["to_host"]["modeled_link_s"] = ledger.total_link_seconds(TO_HOST)
    phases["pack"]["modeled_s"] = ledger.total_pack_seconds()
    phases["unpack"]["modeled_s"] = ledger.total_unpack_seconds()
    raw, wire = ledger.weight_stream_bytes()
    return {
        "phases": phases,
        "wire_bytes": {TO_WORKER: ledger.total_wire_bytes(TO_WORKER), TO_HOST: ledger.total_wire_bytes(TO_HOST)},
        "raw_bytes": {TO_WORKER: ledger.total_raw_bytes(TO_WORKER), TO_HOST: ledger.total_raw_bytes(TO_HOST)},
        "weight_stream": {"raw_bytes": raw, "wire_bytes": wire, "ratio": (raw / wire) if wire else None},
    }


class LedgerRecorder:
    """Runs a WeightSync / HostWeightSync step by step and appends, per step,
    one to_worker record per worker and layer (training.py:214-225) with
    MEASURED seconds, and optionally the workers' to_host gradient records.

    WeightSync (one GPU, masters in HBM): pack_s / unpack_s from CUDA events
    around the multi-tensor pack and unpack kernels of the step; no bytes
    cross a link (link_s = 0). HostWeightSync (masters in host memory):
    pack_s = wall time of the host pack, link_s = the device-side span of the
    packed-stream copies (they overlap the packing), unpack_s = the GPU unpack.
    One launch covers every layer, so a step's time is split over the layers
    in proportion to their algorithmic bytes (4 + r) * n — stated, not modeled.
    `wall` accumulates the per-phase seconds for profile_report."""

    def __init__(self, sync, ledger: TransferLedger | None = None, workers: int = 1, bias_bytes=None):
        self.sync = sync
        self.ledger = ledger if ledger is not None else TransferLedger()
        self.workers = int(workers)
        self.bias = list(bias_bytes) if bias_bytes is not None else [0] * len(sync.counts)
        self.wall = {name: 0.0 for name in PHASES}

    def _split(self, seconds: float, counts, rts) -> list[float]:
        w = [(4 + r) * n for n, r in zip(counts, rts)]
        tot = sum(w) or 1
        return [seconds * x / tot for x in w]

    def step(self, batch: int, **kw):
        import time
        import torch
        from .hostsync import HostWeightSync
        sync = self.sync
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        if isinstance(sync, HostWeightSync):
            t0 = time.perf_counter()
            res = sync.step(batch=batch, events=ev, **kw)
            host_s = time.perf_counter() - t0
            torch.cuda.synchronize()
            link_s, unpack_s, pack_s = ev[0].elapsed_time(ev[1]) * 1e-3, ev[1].elapsed_time(ev[2]) * 1e-3, host_s
        else:
            res = sync.step(batch=batch, events=ev, **kw)
            torch.cuda.synchronize()
            pack_s, unpack_s, link_s = ev[0].elapsed_time(ev[1]) * 1e-3, ev[1].elapsed_time(ev[2]) * 1e-3, 0.0
        rts = res.round_tos if res.round_tos is not None else sync.round_tos
        counts = sync.counts
        for name, v in (("pack", pack_s), ("unpack", unpack_s * self.workers), ("to_worker", link_s * self.workers)):
            self.wall[name] += v
        ps, us, ls = (self._split(x, counts, rts) for x in (pack_s, unpack_s, link_s))
        for _ in range(self.workers):
            for layer, (n, r) in enumerate(zip(counts, rts)):
                record_weights(self.ledger, batch=batch, layer=layer, count=n, round_to=r,
                               bias_bytes=self.bias[layer], pack_seconds=ps[layer], unpack_seconds=us[layer],
                               link_seconds=ls[layer])
        return res

    def gradients(self, batch: int, parameter_count: int, link_seconds: float = 0.0) -> None:
        """One to_host record per worker (TransferBoundary.return_gradients)."""
        for _ in range(self.workers):
            record_gradients(self.ledger, batch=batch, parameter_count=parameter_count, link_seconds=link_seconds)
        self.wall["to_host"] += link_seconds * self.workers

    def report(self, wall_times=None) -> dict:
        w = dict(self.wall)
        w.update(wall_times or {})
        return profile_report(self.ledger, w)
