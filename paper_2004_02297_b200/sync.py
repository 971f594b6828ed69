"""Per-step weight distribution with ADT + AWP on one device.

Reference caller contract (training.py:207-254):
  batch b: pack every layer of the FP32 master at the controller's current
  widths -> each worker unpacks its replica -> ... -> update master ->
  l2-norm of every post-update master layer -> observe_batch -> widths for b+1.

B200 flow (one pack launch with the norm fused, one unpack launch):
  step(b): pack W_b at the widths in force (norm of W_b fused into the same
  read), unpack into the replicas, then read the L float64 sums back, observe
  them (this is the reference's end-of-batch-(b-1) observation of the
  post-update master W_b), and if any width escalated, re-plan and re-pack /
  re-unpack at the new widths. Escalations are rare (at most
  log2-ish (32-initial)/step per layer per run), so the common step is exactly
  two kernel launches and one 8·L-byte device->host read, with results
  byte-identical to the reference's order. step(0) observes nothing (the
  reference's first observation is of the post-update-0 master), and
  observe_final() runs a norm-only pass for the last post-update master.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import engine
from .layout import PackedLayout
from .precision import FixedPrecision, PrecisionController


class NonFiniteParameters(FloatingPointError):
    """net.py:20 — an update left a layer's weights outside the finite range.

    Raised after the step that produced the non-finite weights has been
    applied to every layer (one fused kernel steps all layers; the check reads
    the fused norms afterwards), whereas the reference raises at the first bad
    layer before updating the later ones (net.py:246-257): when it is raised
    here, masters and velocities of every layer hold the post-step values."""


def flat_views(tensors: Sequence[torch.Tensor], what: str) -> list[torch.Tensor]:
    """1-D views of the caller's CUDA float32 tensors. A non-contiguous tensor
    (e.g. a transposed weight) is refused: flattening it would copy, and the
    in-place updates and unpacks would then land in the copy, not in the
    caller's tensor."""
    out = []
    for i, t in enumerate(tensors):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
            raise TypeError(f"{what} layer {i}: need a CUDA float32 tensor")
        if not t.is_contiguous():
            raise ValueError(f"{what} layer {i}: tensor is not contiguous (its flattened copy would be written "
                             "instead of it); pass .contiguous() storage")
        out.append(t.detach().view(-1))
    return out


@dataclass
class SyncResult:
    round_tos: list[int]             # widths the replicas were produced with this step
    trace: list[tuple] = field(default_factory=list)  # TRACE_HEADER rows observed this step
    repacked: bool = False           # a width escalated and the step was redone


class WeightSync:
    """Masters (CUDA float32 tensors, one per layer) -> packed bytes -> replicas."""

    def __init__(self, masters: Sequence[torch.Tensor], schedule=None,
                 replicas: Sequence[torch.Tensor] | None = None, graphed: bool = True,
                 awp_on_device: bool = False, trace_ring: int = 256, fuse_small: bool = False):
        """graphed: step() replays its kernels from a CUDA graph captured once
        per packed layout (one graph launch instead of three ctypes launches
        and the stream bookkeeping per step).

        awp_on_device: the AWP decision runs on the GPU (adt_awp_observe) and a
        whole step — pack, norm, decide, re-pack of escalated layers, unpack —
        is one CUDA graph with no device->host read; step() returns at once
        and the trace rows come back in batches through drain_trace() (at the
        latest every `trace_ring` observations, automatically). Layers keep
        fixed capacity offsets in the packed buffer (room for 4 bytes/weight);
        each payload is still exactly the reference's n*r bytes.

        fuse_small: sets of at most one 4096-weight tile per SM and <= 16
        layers (LeNet) run the whole step as ONE cooperative launch
        (adt_roundtrip: pack + norms, grid barrier, unpack) instead of three
        dependent launches — the same bytes, norms and replicas. Off by
        default: measured slower on a B200 (LeNet 12.3 vs 6.2 us per step back
        to back, profiles/r02_ab_small_step.md)."""
        engine.require_cuda()
        self.graphed = graphed
        self.fuse_small = bool(fuse_small)
        self._small = False
        self._rt_barrier = None
        self.masters = flat_views(masters, "master")
        self.counts = [m.numel() for m in self.masters]
        self.schedule = schedule if schedule is not None else FixedPrecision(len(self.masters), 32)
        if self.schedule.num_layers != len(self.masters):
            raise ValueError("schedule layer count differs from the number of master tensors")
        self.adaptive = isinstance(self.schedule, PrecisionController)
        dev = self.masters[0].device if self.masters else torch.device("cuda")
        if replicas is None:
            replicas = [torch.empty_like(m) for m in self.masters]
        self.replicas = flat_views(replicas, "replica")
        self.sumsq = torch.zeros(len(self.masters), dtype=torch.float64, device=dev)
        self._host_sumsq = torch.empty(len(self.masters), dtype=torch.float64, pin_memory=True)
        # The norm finalize (a tiny per-layer reduction of the pack's partials)
        # runs on a side stream, concurrently with the unpack.
        self._side = torch.cuda.Stream(device=dev)
        self._fin_done = torch.cuda.Event()
        self._fin_pending = False
        self._partials = None
        self._graphs = None      # {(fused_norm, split): graphs} for the current layout
        self.velocities = None   # momentum buffers, created by the first update()
        self._grad_stage = {}    # gather_and_update: staging buckets for per-layer gradient lists
        self._reduce_table = None
        self.device = dev
        self.layout = None
        self.packed = None
        self._plan(self.schedule.round_tos())
        self.awp_on_device = bool(awp_on_device)
        self._dawp = None
        if self.awp_on_device:
            self._init_device_awp(trace_ring)

    # --------------------------------------------- device-resident AWP mode
    def _init_device_awp(self, ring: int) -> None:
        from .awp_device import DeviceAwp
        if not self.adaptive:
            raise ValueError("awp_on_device needs a PrecisionController schedule")
        self._dawp = DeviceAwp(self.schedule, self.device, ring)
        cap = PackedLayout.plan(self.counts, [4] * len(self.counts))
        self.capacity_layout = cap
        if self.packed.numel() < cap.nbytes:
            self.packed = torch.empty(max(16, cap.nbytes), dtype=torch.uint8, device=self.device)
        self._cap_pack = engine.SegmentTable(self.masters, cap)
        self._cap_unpack = engine.SegmentTable(self.replicas, cap)
        self._agraphs = {}
        self._trace_log = []

    def _device_step_kernels(self, observe: bool) -> None:
        """pack(A) -> [finalize -> observe(-> B, escalated list)] || unpack(A) -> fixup -> A = B."""
        d = self._dawp
        main = torch.cuda.current_stream()
        engine.pack_dyn(self._cap_pack, self.packed, d.widths, self._partials if observe else None, main)
        if observe:
            self._side.wait_stream(main)
            engine.finalize(self._cap_pack, self._partials, self.sumsq, self._side)
            engine.awp_observe(self.sumsq, d.struct, d.config, self._side)
        engine.unpack_dyn(self._cap_unpack, self.packed, d.widths, main)
        if observe:
            main.wait_stream(self._side)
            engine.awp_fixup(self._cap_pack, self._cap_unpack, self.packed, d.escalated, d.widths_new, main)
            d.widths.copy_(d.widths_new)

    def _step_device(self, batch: int, observe: bool) -> SyncResult:
        d = self._dawp
        if observe and not d.label_set:
            d.set_next_label(batch - 1)
        if self.graphed:
            g = self._agraphs.get(observe)
            if g is None:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._device_step_kernels(observe)
                self._agraphs[observe] = g
            g.replay()
        else:
            self._device_step_kernels(observe)
        if observe:
            d.pending += 1
            if d.pending >= d.ring_steps:
                self._trace_log += d.drain()
        return SyncResult(round_tos=None)

    def _update_device(self, launch, batch: int) -> SyncResult:
        """Device-AWP form of _update_step: the fused update + pack at the
        device widths, then [finalize -> observe] || unpack -> fixup, with
        no host read; the trace rows (labelled `batch`) and the finite-weights
        check (NonFiniteParameters, from the rows' norms) come at the next
        drain_trace()."""
        d = self._dawp
        main = torch.cuda.current_stream()
        d.counter[1].fill_(int(batch))
        d.label_set = True
        launch(main)
        self._side.wait_stream(main)
        engine.finalize(self._cap_pack, self._partials, self.sumsq, self._side)
        engine.awp_observe(self.sumsq, d.struct, d.config, self._side)
        engine.unpack_dyn(self._cap_unpack, self.packed, d.widths, main)
        main.wait_stream(self._side)
        engine.awp_fixup(self._cap_pack, self._cap_unpack, self.packed, d.escalated, d.widths_new, main)
        d.widths.copy_(d.widths_new)
        self._check_finite = True
        d.pending += 1
        if d.pending >= d.ring_steps:
            self._trace_log += d.drain()
        return SyncResult(round_tos=None)

    def drain_trace(self) -> list[tuple]:
        """awp_on_device: every trace row (TRACE_HEADER) observed since the
        last call, in order; synchronises and refreshes the host controller
        (schedule.state(), round_tos) from the device."""
        if not self.awp_on_device:
            raise RuntimeError("drain_trace() is for awp_on_device=True (step() returns the rows otherwise)")
        rows = self._trace_log + self._dawp.drain()
        self._trace_log = []
        if getattr(self, "_check_finite", False):
            bad = next((r for r in rows if not math.isfinite(r[2])), None)
            if bad is not None:
                raise NonFiniteParameters(f"layer {bad[1]} parameters left the finite range (batch {bad[0]})")
        return rows

    def _plan(self, round_tos):
        self._graphs = None
        self._timed = None
        self.layout = PackedLayout.plan(self.counts, round_tos)
        if self.packed is None or self.packed.numel() < self.layout.nbytes:
            # capacity for every width up to 4 bytes: re-plans never reallocate
            cap = PackedLayout.plan(self.counts, [4] * len(self.counts)).nbytes
            self.packed = torch.empty(max(16, cap), dtype=torch.uint8, device=self.device)
        self.pack_table = engine.SegmentTable(self.masters, self.layout)
        self.unpack_table = engine.SegmentTable(self.replicas, self.layout)
        if self._partials is None or self._partials.numel() < self.pack_table.npartials:
            self._partials = torch.empty(max(1, self.pack_table.npartials), dtype=torch.float64, device=self.device)
        ntiles = self.pack_table.npartials // 8
        self._small = (self.fuse_small and 0 < ntiles <= engine.roundtrip_max_tiles()
                       and 1 <= len(self.counts) <= 16)
        if self._small and self._rt_barrier is None:
            self._rt_barrier = torch.zeros(2, dtype=torch.int32, device=self.device)

    @property
    def round_tos(self) -> list[int]:
        if getattr(self, "_dawp", None) is not None:
            return self._dawp.round_tos()            # device read
        return list(self.layout.round_tos)

    def launch(self, fused_norm: bool, mid_event: torch.cuda.Event | None = None) -> None:
        """The device work of one step on the current stream, no host sync:
        pack (+ norm partials), [side stream: finalize -> self.sumsq], unpack
        (small sets without a requested pack/unpack split: one adt_roundtrip)."""
        self._host_widths_only()
        main = torch.cuda.current_stream()
        if self._small and mid_event is None:
            if self._fin_pending:
                main.wait_event(self._fin_done)
            engine.roundtrip(self.pack_table, self.unpack_table, self.packed, self.sumsq if fused_norm else None,
                             self._partials, self._rt_barrier, main)
            self._fin_done.record(main)
            self._fin_pending = True
            return
        if fused_norm:
            if self._fin_pending:
                main.wait_event(self._fin_done)  # previous finalize done reading the partials
            engine.pack(self.pack_table, self.packed, None, main, partials=self._partials)
            self._side.wait_stream(main)
            engine.finalize(self.pack_table, self._partials, self.sumsq, self._side)
            self._fin_done.record(self._side)
            self._fin_pending = True
        else:
            engine.pack(self.pack_table, self.packed, None, main)
        if mid_event is not None:
            mid_event.record(main)
        engine.unpack(self.unpack_table, self.packed, main)

    def _host_widths_only(self) -> None:
        if getattr(self, "awp_on_device", False):
            raise RuntimeError("launch()/launch_graphed()/phase_ms() use the host-planned widths; with "
                               "awp_on_device=True the widths live on the device: use step()")

    def launch_graphed(self, fused_norm: bool, mid_event: torch.cuda.Event | None = None) -> None:
        """launch() replayed from CUDA graphs captured once per layout: one
        graph [pack -> fork(finalize on the side branch) | unpack -> join], or,
        when the caller wants the pack/unpack split (`mid_event`), two graphs
        with the event recorded between them. Removes the per-step host launch
        cost (ctypes + stream bookkeeping): LeNet 39.6 -> 18.7 us per step."""
        self._host_widths_only()
        split = mid_event is not None
        key = (fused_norm, split)
        if self._graphs is None:
            self._graphs = {}                # per (fused_norm, split); dropped by every re-plan
        graphs = self._graphs.get(key)
        if graphs is None:
            graphs = self._graphs[key] = self._capture(fused_norm, split)
        graphs[0].replay()
        if split:
            mid_event.record(torch.cuda.current_stream())
            graphs[1].replay()

    def phase_ms(self, fused_norm: bool, reps: int = 20, rounds: int = 5) -> tuple[float, float]:
        """Average device time of each phase of the step, measured as `reps`
        back-to-back copies of that phase in one CUDA graph timed by two events
        outside it (event nodes inside a graph cost several us each, which would
        distort short kernels): (pack ms, finalize||unpack ms). Synchronizes."""
        self._host_widths_only()
        key = ("phase", fused_norm, reps, self.layout)
        if getattr(self, "_timed", None) is None or self._timed[0] != key:
            self.launch(fused_norm)
            torch.cuda.synchronize()
            self._fin_pending = False
            g_pack, g_rest = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_pack):
                for _ in range(reps):
                    engine.pack(self.pack_table, self.packed, None, torch.cuda.current_stream(),
                                partials=self._partials if fused_norm else None)
            with torch.cuda.graph(g_rest):
                cap = torch.cuda.current_stream()
                for _ in range(reps):
                    if fused_norm:
                        self._side.wait_stream(cap)
                        engine.finalize(self.pack_table, self._partials, self.sumsq, self._side)
                    engine.unpack(self.unpack_table, self.packed, cap)
                    if fused_norm:
                        cap.wait_stream(self._side)
            self._timed = (key, g_pack, g_rest)
        _, g_pack, g_rest = self._timed
        out = []
        for g in (g_pack, g_rest):
            g.replay()                                   # warm
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(rounds):
                g.replay()
            b.record()
            b.synchronize()
            out.append(a.elapsed_time(b) / (rounds * reps))
        return out[0], out[1]

    def _capture(self, fused_norm: bool, split: bool):
        self.launch(fused_norm)              # eager warm-up (lazy CUDA init, scratch)
        torch.cuda.synchronize()
        self._fin_pending = False

        def pack():
            engine.pack(self.pack_table, self.packed, None, torch.cuda.current_stream(),
                        partials=self._partials if fused_norm else None)

        def rest():
            cap = torch.cuda.current_stream()
            if fused_norm:
                self._side.wait_stream(cap)
                engine.finalize(self.pack_table, self._partials, self.sumsq, self._side)
            engine.unpack(self.unpack_table, self.packed, cap)
            if fused_norm:
                cap.wait_stream(self._side)

        if not split:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if self._small:                  # the one-launch step (adt_roundtrip)
                    engine.roundtrip(self.pack_table, self.unpack_table, self.packed,
                                     self.sumsq if fused_norm else None, self._partials, self._rt_barrier,
                                     torch.cuda.current_stream())
                else:
                    pack()
                    rest()
            return (g,)
        g_pack, g_rest = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_pack):
            pack()
        with torch.cuda.graph(g_rest):
            rest()
        return g_pack, g_rest

    def read_norms(self) -> list[float]:
        """Per-layer l2 norms (precision.l2_norm) of the masters as of the last
        launch with the norm fused: one 8·L-byte device->host read + sync."""
        self._side.wait_stream(torch.cuda.current_stream())  # graphed finalize runs on the main stream's graph
        with torch.cuda.stream(self._side):  # queued behind the (eager) finalize
            self._host_sumsq.copy_(self.sumsq, non_blocking=True)
        self._side.synchronize()
        return [math.sqrt(v) for v in self._host_sumsq.tolist()]

    def step(self, batch: int = 0, observe: bool | None = None, events=None) -> SyncResult:
        """One batch of weight distribution (see module doc for the ordering).
        events = (e0, e1, e2): CUDA timing events recorded before the pack,
        between pack and unpack, and after the unpack (transfer.LedgerRecorder)."""
        if observe is None:
            observe = self.adaptive and batch > 0
        if self.awp_on_device:
            if events is not None:
                raise ValueError("per-phase events need the host-planned step (awp_on_device=False)")
            return self._step_device(batch, observe)
        used = self.round_tos
        main = torch.cuda.current_stream()
        if events is not None:
            events[0].record(main)
        if self.graphed:
            self.launch_graphed(fused_norm=observe, mid_event=events[1] if events is not None else None)
        else:
            self.launch(fused_norm=observe, mid_event=events[1] if events is not None else None)
        if events is not None:
            events[2].record(main)
        res = SyncResult(round_tos=used)
        if not observe:
            return res
        res.trace = self.schedule.observe_all(self.read_norms(), batch=batch - 1)
        new = self.schedule.round_tos()
        if new != used:
            self._plan(new)
            self.launch(fused_norm=False)
            res.round_tos = new
            res.repacked = True
        return res

    def update(self, grads: Sequence[torch.Tensor], lr: float, momentum: float = 0.9,
               weight_decay: float = 5e-4, batch: int = 0) -> SyncResult:
        """Fused optimizer step + distribution of the updated weights.

        Reference order (training.py:240-254, then the next batch's :209-225):
        update W_b -> W_{b+1} (net.py:236-246) -> l2-norms of W_{b+1} ->
        observe (trace rows labelled `batch`) -> pack W_{b+1} at the new
        widths -> unpack. Here one kernel does the update, packs W_{b+1} at
        the widths in force and fuses its norms; the norms are observed and,
        if a width escalated, W_{b+1} is re-packed (without updating again).
        The replicas then hold batch b+1's weights.

        `grads` is the ALREADY AVERAGED gradient, applied as is. The
        reference's gather_and_update (net.py:203-257) always forms
        pairwise_sum(g_c * f32(n_c)) / f32(total), even for one contribution,
        and g * n / n is not always bit-equal to g in float32: for bit parity
        with the reference use gather_and_update([GradientSet(g, [], n)]).
        """
        if len(grads) != len(self.masters):
            from .grads import ShapeMismatch
            raise ShapeMismatch("one gradient tensor per layer")
        self._ensure_velocities()
        g = [t.detach().reshape(-1) for t in grads]
        if self.awp_on_device:
            table = engine.SgdTable(self.masters, self.velocities, g, self.capacity_layout)
            d = self._dawp
            return self._update_device(lambda main: engine.sgd_pack_dyn(
                table, lr, momentum, weight_decay, self.packed, d.widths, self._partials, main), batch)
        table = engine.SgdTable(self.masters, self.velocities, g, self.layout)

        def launch(main):
            engine.sgd_pack(table, lr, momentum, weight_decay, self.packed, None, main, partials=self._partials)
        return self._update_step(launch, batch)

    def gather_and_update(self, contributions, lr: float, momentum: float = 0.9, weight_decay: float = 5e-4,
                          batch: int = 0) -> SyncResult:
        """net.gather_and_update (net.py:203-257) + distribution, fused.

        `contributions`: 1..16 worker gradient sets — `grads.GradBucket`s (used
        in place) or objects with `weight_grads` / `sample_count` (a
        `grads.GradientSet`, staged into a bucket). One kernel combines them
        with the reference's sample-count weighting and pairwise_sum tree,
        steps W and v, packs W' and fuses its norm; then the replicas are
        unpacked and AWP observes, exactly as update()."""
        from .grads import GradBucket, ShapeMismatch
        if not contributions:
            raise ShapeMismatch("no gradient contributions")          # net.py:218-219
        if len(contributions) > 16:
            raise ValueError("gather_and_update takes 1..16 gradient contributions")
        buckets = []
        for i, c in enumerate(contributions):
            if isinstance(c, GradBucket):
                b = c
            else:
                if len(c.weight_grads) != len(self.masters):
                    raise ShapeMismatch(f"contribution has {len(c.weight_grads)} layers, network has {len(self.masters)}")
                stage = self._grad_stage.get(i)
                if stage is None:
                    stage = self._grad_stage[i] = GradBucket(self.counts, self.device)
                b = stage.load(c.weight_grads)
                b.sample_count = int(c.sample_count)
            if list(b.counts) != list(self.counts):
                raise ShapeMismatch("gradient bucket layer sizes differ from the masters")
            buckets.append(b)
        self._ensure_velocities()
        key = self.capacity_layout if self.awp_on_device else self.layout
        if self._reduce_table is None or self._reduce_table[0] != key:
            offs = [buckets[0].byte_offset(l) for l in range(len(self.masters))]
            self._reduce_table = (key, engine.ReduceSgdTable(self.masters, self.velocities, offs, key))
        table = self._reduce_table[1]
        ptrs = [b.flat.data_ptr() for b in buckets]
        counts = [b.sample_count for b in buckets]
        if self.awp_on_device:
            d = self._dawp
            return self._update_device(lambda main: engine.reduce_sgd_pack_dyn(
                table, ptrs, counts, lr, momentum, weight_decay, self.packed, d.widths, self._partials, main), batch)

        def launch(main):
            engine.reduce_sgd_pack(table, ptrs, counts, lr, momentum, weight_decay, self.packed, None, main,
                                   partials=self._partials)
        return self._update_step(launch, batch)

    def _ensure_velocities(self) -> None:
        if self.velocities is None:
            self.velocities = [torch.zeros_like(m) for m in self.masters]

    def _update_step(self, launch, batch: int) -> SyncResult:
        main = torch.cuda.current_stream()
        if self._fin_pending:
            main.wait_event(self._fin_done)
        launch(main)
        self._side.wait_stream(main)
        engine.finalize(self.pack_table, self._partials, self.sumsq, self._side)
        self._fin_done.record(self._side)
        self._fin_pending = True
        engine.unpack(self.unpack_table, self.packed, main)
        used = self.round_tos
        res = SyncResult(round_tos=used)
        norms = self.read_norms()
        bad = [i for i, n in enumerate(norms) if not math.isfinite(n)]
        if bad:
            raise NonFiniteParameters(f"layer {bad[0]} parameters left the finite range")
        if not self.adaptive:
            return res
        res.trace = self.schedule.observe_all(norms, batch=batch)
        new = self.schedule.round_tos()
        if new != used:
            self._plan(new)
            self.launch(fused_norm=False)
            res.round_tos = new
            res.repacked = True
        return res

    def _norm_pass(self) -> list[float]:
        main = torch.cuda.current_stream()
        if self._fin_pending:
            main.wait_event(self._fin_done)
        engine.sumsq(self.pack_table, self.sumsq)
        self._side.wait_stream(main)
        return self.read_norms()

    def observe_final(self, batch: int) -> list[tuple]:
        """Norm-only pass over the masters (the observation after the last
        update, training.py:246-254); returns its trace rows labelled `batch`.
        A fixed schedule observes nothing (the reference only observes in
        adaptive mode, training.py:246): no rows."""
        if not self.adaptive:
            return []
        if self.awp_on_device:
            d = self._dawp
            rows = self.drain_trace()
            engine.sumsq(self._cap_pack, self.sumsq)
            d.set_next_label(batch)
            engine.awp_observe(self.sumsq, d.struct, d.config)
            # an escalation decided by this last observation is in force from now
            # on (round_tos, any later step): widths A <- B, as every step does
            d.widths.copy_(d.widths_new)
            self._trace_log = rows          # kept for the next drain_trace(); return only this observation
            last = d.drain()
            return last
        return self.schedule.observe_all(self._norm_pass(), batch=batch)

    def norms(self) -> list[float]:
        """Current per-layer l2 norms of the masters (norm-only pass)."""
        return self._norm_pass()
