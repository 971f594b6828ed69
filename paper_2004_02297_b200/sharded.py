"""Multi-GPU weight distribution: shard-pack -> exchange packed bytes -> unpack.

The reference simulates data-parallel workers in one process and only
*accounts* the bytes each worker would receive (training.py:214-225,
transfer.py:143-174). Here every rank is one GPU (torchrun): rank p packs its
contiguous shard of the concatenated layers at the AWP widths (norm partials
fused into the same read), only packed bytes cross NVLink, and every rank
unpacks the whole stream into its full FP32 replica. Two transports:

* p2p (default on one node, `transport="auto"`): every rank's send buffers are
  mapped into every other rank (CUDA IPC); after a device-side barrier
  (adt_peer_barrier) each rank's unpack kernel reads its peers' payloads over
  NVLink directly (adt_unpack_multi) — the gather and the unpack are one pass;
* nccl: `all_gather_into_tensor` (ncclAllGather, uint8) into a receive
  buffer in chunks, each chunk unpacked as soon as it lands (ChunkedGather;
  the fallback when the GPUs are not peers).

Send buffer of rank p (S_max bytes, identical size on every rank):
    [piece payloads, 16-B aligned | pad | float64 sum of squares per piece]
Every rank combines the per-piece sums from all tails in fixed rank order and
sees bit-identical norms -> identical AWP decisions with no extra collective
(SURVEY.md §8e). The same class runs the data-parallel update (the gradient
return path, `update`) and, with `awp_on_device=True`, takes the AWP decision
on every GPU so that a step involves no host round trip.

Shards are balanced by packed bytes Σ n·r and cut at multiples of the
4096-weight tile inside a layer, so every piece starts 16-B aligned on both
the FP32 and the packed side.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import torch

from . import engine
from ._lib import TILE_WEIGHTS
from .layout import align_up
from .precision import FixedPrecision, PrecisionController
from .grads import GradBucket, ShapeMismatch, bucket_offsets, shard_ranges
from .sync import NonFiniteParameters, SyncResult


@dataclass(frozen=True)
class Piece:
    layer: int
    lo: int          # first weight (multiple of TILE_WEIGHTS unless 0)
    hi: int
    offset: int      # byte offset inside the owning rank's send buffer


@dataclass(frozen=True)
class ShardPlan:
    counts: tuple[int, ...]
    round_tos: tuple[int, ...]
    world: int
    pieces: tuple[tuple[Piece, ...], ...]   # per rank
    payload_cap: int                        # bytes reserved for payloads (16-B multiple)
    max_pieces: int
    send_bytes: int                          # S_max: payload_cap + 8 * max_pieces
    align: int = 16                          # piece offsets are multiples of this

    @staticmethod
    def plan(counts: Sequence[int], round_tos: Sequence[int], world: int, align: int = 16) -> "ShardPlan":
        """align = 48 (SPLIT_ALIGN) makes every piece splittable at any 48-B
        multiple of the send buffer (chunk_segments)."""
        counts = tuple(int(c) for c in counts)
        round_tos = tuple(int(r) for r in round_tos)
        if world < 1:
            raise ValueError("world size must be >= 1")
        total = sum(n * r for n, r in zip(counts, round_tos))
        # walk the concatenated stream tile by tile; rank p takes bytes up to
        # ceil(total * (p+1) / world), cut on tile boundaries.
        per_rank: list[list[tuple[int, int, int]]] = [[] for _ in range(world)]
        rank, done = 0, 0
        target = lambda p: -(-total * (p + 1) // world)  # noqa: E731
        for layer, (n, r) in enumerate(zip(counts, round_tos)):
            lo = 0
            while lo < n:
                while rank < world - 1 and done >= target(rank):
                    rank += 1
                if rank == world - 1:
                    hi = n
                else:
                    want = max(1, target(rank) - done)            # bytes still owed to this rank
                    tiles = -(-want // (TILE_WEIGHTS * r))          # round up to whole tiles
                    hi = min(n, lo + tiles * TILE_WEIGHTS)
                per_rank[rank].append((layer, lo, hi))
                done += (hi - lo) * r
                lo = hi
        pieces, cap = [], 0
        for p in range(world):
            off, lst = 0, []
            for layer, lo, hi in per_rank[p]:
                lst.append(Piece(layer, lo, hi, off))
                off = align_up(off + (hi - lo) * round_tos[layer], align)
            cap = max(cap, off)
            pieces.append(tuple(lst))
        max_pieces = max(1, max(len(x) for x in pieces))
        cap = align_up(max(cap, 16), align)
        return ShardPlan(counts, round_tos, world, tuple(pieces), cap, max_pieces,
                         align_up(cap + 8 * max_pieces), align)

    def with_widths(self, round_tos: Sequence[int]) -> "ShardPlan":
        """The same ownership (every rank keeps its (layer, lo, hi) pieces) at
        new widths: only the packed offsets and buffer sizes change. Used once
        masters are sharded (update()), where moving ownership would move
        master/velocity state between ranks."""
        round_tos = tuple(int(r) for r in round_tos)
        pieces, cap = [], 0
        for lst0 in self.pieces:
            off, lst = 0, []
            for pc in lst0:
                lst.append(Piece(pc.layer, pc.lo, pc.hi, off))
                off = align_up(off + (pc.hi - pc.lo) * round_tos[pc.layer], self.align)
            cap = max(cap, off)
            pieces.append(tuple(lst))
        cap = align_up(max(cap, 16), self.align)
        return ShardPlan(self.counts, round_tos, self.world, tuple(pieces), cap, self.max_pieces,
                         align_up(cap + 8 * self.max_pieces), self.align)

    def rank_payload_bytes(self, rank: int) -> int:
        return sum((pc.hi - pc.lo) * self.round_tos[pc.layer] for pc in self.pieces[rank])

    def combine_sumsq(self, tails) -> list[float]:
        """tails[q][k] = float64 sum of squares of rank q's k-th piece ->
        per-layer totals, summed in fixed (rank, piece) order."""
        out = [0.0] * len(self.counts)
        for q in range(self.world):
            for k, pc in enumerate(self.pieces[q]):
                out[pc.layer] += float(tails[q][k])
        return out


SPLIT_ALIGN = 48     # a multiple of 4r bytes for r = 1..4 and of 16


@dataclass(frozen=True)
class ChunkedGather:
    """The nccl transport's send buffer cut into byte ranges gathered one
    after another, so the unpack of chunk c overlaps the gather of chunk c+1.

    bounds[c] .. bounds[c+1] is chunk c of every rank's send buffer (the same
    cut on every rank; the payload split in near-equal SPLIT_ALIGN multiples,
    the norm tail in the last chunk). Chunk c is gathered rank-major into
    region[c] .. region[c+1] of the receive buffer. segments[c] lists the
    parts of the pieces whose packed bytes lie in chunk c:
    (rank, layer, lo, hi, round_to, byte offset in the receive buffer)."""
    bounds: tuple[int, ...]
    region: tuple[int, ...]
    segments: tuple[tuple[tuple[int, int, int, int, int, int], ...], ...]

    @staticmethod
    def cut(plan: ShardPlan, chunks: int) -> "ChunkedGather":
        if plan.align % SPLIT_ALIGN:
            raise ValueError(f"chunked gather needs a plan with piece offsets aligned to {SPLIT_ALIGN} B")
        S, cap = plan.send_bytes, plan.payload_cap
        step = align_up(-(-cap // max(1, chunks)), SPLIT_ALIGN)
        bounds = [0] + [c * step for c in range(1, max(1, chunks)) if c * step < cap] + [S]
        region = [0]
        for c in range(len(bounds) - 1):
            region.append(region[-1] + plan.world * (bounds[c + 1] - bounds[c]))
        segs = [[] for _ in range(len(bounds) - 1)]
        for q in range(plan.world):
            for pc in plan.pieces[q]:
                r = plan.round_tos[pc.layer]
                a, e = pc.offset, pc.offset + (pc.hi - pc.lo) * r
                for c in range(len(bounds) - 1):
                    b0, b1 = bounds[c], bounds[c + 1]
                    s, t = max(a, b0), min(e, b1)
                    if s < t:    # s - a, t - a: multiples of 4r (or the piece end)
                        segs[c].append((q, pc.layer, pc.lo + (s - a) // r, pc.lo + (t - a) // r, r,
                                        region[c] + q * (b1 - b0) + (s - b0)))
        return ChunkedGather(tuple(bounds), tuple(region), tuple(tuple(x) for x in segs))

    def tails(self, recv: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
        """(world, 8 * max_pieces) uint8 view of every rank's gathered norm tail."""
        b = self.bounds[-2]
        width = self.bounds[-1] - b
        return recv[self.region[-2]:self.region[-1]].view(plan.world, width)[
            :, plan.payload_cap - b:plan.payload_cap - b + 8 * plan.max_pieces]


class PeerTimeout(RuntimeError):
    """A device-side peer barrier gave up waiting for another rank (a stalled
    or dead peer). The kernels queued behind it did no work (the abort guard),
    so replicas, masters and the AWP state hold the last good step's values;
    the exchange cannot continue — rebuild the ShardedWeightSync."""


def peer_transport(dist, group=None) -> str:
    """"p2p" when every rank's GPU can map every other rank's memory (NVLink /
    NVSwitch peers on one node: the fused peer-read kernels apply), else
    "nccl". Collective: every rank must call it; all get the same answer."""
    dev = torch.cuda.current_device()
    info = (socket_host(), dev)
    everyone = [None] * dist.get_world_size(group)
    dist.all_gather_object(everyone, info, group=group)
    if len({h for h, _ in everyone}) != 1:
        ok = False                                  # several hosts: no CUDA IPC
    else:
        ok = all(d == dev or torch.cuda.can_device_access_peer(dev, d) for _, d in everyone)
    votes = [None] * len(everyone)
    dist.all_gather_object(votes, ok, group=group)
    return "p2p" if all(votes) else "nccl"


def socket_host() -> str:
    import socket
    return socket.gethostname()


class ShardedWeightSync:
    """Per-step packed weight distribution across the ranks of `group`.

    `masters[l]` are this rank's FP32 master tensors (full layer shape; only
    this rank's shard ranges are read), `replicas[l]` receive every weight.

    transport = "auto" (default): "p2p" when all ranks' GPUs are peers on one
        node and every rank can map the others' memory, else "nccl"
        (peer_transport, then a vote on the first peer mapping).
    transport = "nccl": pack -> ncclAllGather(uint8) of the packed send
        buffers, `nccl_chunks` byte ranges queued at once -> unpack of each
        range as it completes.
    transport = "p2p": every rank's send buffer is mapped into every other
        rank with CUDA IPC; after one stream-ordered barrier each rank unpacks
        straight out of its peers' send buffers over NVLink
        (adt_unpack_multi) — the gather and the unpack are one kernel, and the
        gathered stream is never written to or re-read from HBM. Send buffers
        alternate between two slots so one barrier per step covers both the
        read-after-write and the write-after-read hazard.
    """

    def __init__(self, masters: Sequence[torch.Tensor], schedule=None, replicas=None, group=None,
                 transport: str = "auto", awp_on_device: bool = False, trace_ring: int = 256,
                 nccl_chunks: int = 4, barrier_timeout_s: float = 30.0, collectives_at_world1: bool = False):
        """awp_on_device (p2p transport): every rank runs the AWP decision on
        its GPU from the gathered per-piece sums (identical inputs, so
        identical decisions), pieces keep capacity offsets in the send
        buffers, and a step — pack, norm, barrier, gather-unpack, decide,
        re-pack + re-gather of escalated pieces — is device work only (one
        CUDA graph per send slot); trace rows come back via drain_trace().

        nccl_chunks (nccl transport): the packed send buffers are gathered in
        this many byte ranges (ChunkedGather), each unpacked as soon as it
        lands, so the unpack overlaps the rest of the all-gather.

        barrier_timeout_s (p2p transport): how long a device-side barrier waits
        for the other ranks. On timeout every kernel behind it that reads peer
        memory skips its work (abort guard) and the next call on this object
        raises PeerTimeout: each call first waits for the previous step to
        finish on the device, so the failure surfaces within one step.

        collectives_at_world1 (nccl transport, tests): with a single rank, still
        run the chunked all-gather and the gradient all_to_all through the
        process group instead of short-cutting them (a one-rank NCCL group
        exercises the real NCCL calls, stream waits and chunk bookkeeping on a
        one-GPU box, where NCCL refuses two ranks on one device)."""
        import torch.distributed as dist
        engine.require_cuda()
        if transport not in ("nccl", "p2p", "auto"):
            raise ValueError("transport must be 'nccl', 'p2p' or 'auto'")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._collect = self.world > 1 or bool(collectives_at_world1)
        self.transport = peer_transport(dist, group) if transport == "auto" else transport
        from .sync import flat_views
        self.masters = flat_views(masters, "master")
        self.counts = [m.numel() for m in self.masters]
        self.schedule = schedule if schedule is not None else FixedPrecision(len(self.masters), 32)
        self.adaptive = isinstance(self.schedule, PrecisionController)
        self.device = self.masters[0].device
        if replicas is None:
            replicas = [torch.empty_like(m) for m in self.masters]
        self.replicas = flat_views(replicas, "replica")
        if barrier_timeout_s <= 0:
            raise ValueError("barrier_timeout_s must be > 0")
        self.barrier_timeout_s = float(barrier_timeout_s)
        self._abort = None         # p2p: the barrier's timeout word (device), guard of every peer-reading kernel
        self._poll_event = None
        self.send = self.recv = None
        self._slot = 0
        self._peer = None      # p2p: per slot, every rank's send-buffer address in this process
        self._opened = []
        self.velocities = None     # momentum buffers (only this rank's shard ranges are stepped)
        self._gpeer = None         # p2p: (bucket data_ptr, every rank's bucket address here)
        self._gopened = []
        self._bopened = []         # p2p: peers' barrier flag arrays mapped here
        self._grecv = None         # nccl: all-to-all'd gradient slices of this rank's shard
        if self.transport == "p2p" and not self._init_barrier():
            if transport == "p2p":
                raise RuntimeError("transport='p2p': a rank could not map its peers' memory (CUDA IPC)")
            self.transport = "nccl"              # "auto": every rank saw the same vote
        if nccl_chunks < 1:
            raise ValueError("nccl_chunks must be >= 1")
        self.nccl_chunks = int(nccl_chunks)
        self._align = SPLIT_ALIGN if self.transport == "nccl" else 16
        self._chunked = None
        self.awp_on_device = bool(awp_on_device)
        self._dawp = None
        if self.awp_on_device:
            if self.transport != "p2p" or not self.adaptive:
                raise ValueError("awp_on_device needs transport='p2p' and a PrecisionController schedule")
            # capacity offsets: ownership and layout never change with the widths
            self.plan = ShardPlan.plan(self.counts, [4] * len(self.counts), self.world)
            self._owners_fixed = True
            self._plan([4] * len(self.counts))
            self._init_device_awp(trace_ring)
        else:
            self._plan(self.schedule.round_tos())

    # --------------------------------------------- device-resident AWP mode
    def _init_device_awp(self, ring: int) -> None:
        from .awp_device import DeviceAwp
        d = self._dawp = DeviceAwp(self.schedule, self.device, ring)
        self._side = torch.cuda.Stream(device=self.device)
        self._sumsq_dev = torch.zeros(len(self.counts), dtype=torch.float64, device=self.device)
        mine = self.plan.pieces[self.rank]
        self._mine_layers = [pc.layer for pc in mine]
        self._all_layers = [pc.layer for q in range(self.world) for pc in self.plan.pieces[q]]
        dev = self.device
        self._idx_mine = torch.tensor(self._mine_layers, dtype=torch.int64, device=dev)
        self._idx_all = torch.tensor(self._all_layers, dtype=torch.int64, device=dev)
        n_m, n_a = max(1, len(mine)), max(1, len(self._all_layers))
        self._pw_mine = torch.zeros(n_m, dtype=torch.uint8, device=dev)
        self._pw_all = torch.zeros(n_a, dtype=torch.uint8, device=dev)
        self._pw_mine_new = torch.zeros(n_m, dtype=torch.uint8, device=dev)
        self._pw_all_new = torch.zeros(n_a, dtype=torch.uint8, device=dev)
        # piece k of rank q sits at tails[q * max_pieces + k]; -1 marks an empty slot
        m = self.plan.max_pieces
        pl = [-1] * (self.world * m)
        for q in range(self.world):
            for k, pc in enumerate(self.plan.pieces[q]):
                pl[q * m + k] = pc.layer
        self._piece_layer = torch.tensor(pl, dtype=torch.int32, device=dev)
        self._my_reps = engine.SegmentTable([self.replicas[pc.layer][pc.lo:pc.hi] for pc in mine],
                                            self.pack_table.layout)
        self._dgraphs = {}
        self._trace_log = []

    def _device_step_kernels(self, slot: int, observe: bool, pack=None) -> None:
        """pack(widths A) [-> norm tails] -> barrier -> [gather tails -> combine -> observe(-> B)]
        || gather-unpack(A) -> re-pack own escalated pieces -> barrier -> re-gather them -> A = B.
        `pack(send, widths, partials, stream)` replaces the plain pack (the DP update)."""
        d = self._dawp
        main = torch.cuda.current_stream()
        send = self.send[slot]
        torch.index_select(d.widths, 0, self._idx_mine, out=self._pw_mine[:len(self._mine_layers)])
        torch.index_select(d.widths, 0, self._idx_all, out=self._pw_all[:len(self._all_layers)])
        if pack is None:
            engine.pack_dyn(self.pack_table, send, self._pw_mine, self._partials if observe else None, main)
        else:
            pack(send, self._pw_mine, self._partials, main)
        if observe:
            engine.finalize(self.pack_table, self._partials, self._tail(send), main)
        self._barrier()
        ab = self._abort
        if observe:
            engine.copy_multi(self.tails, self._peer[slot], self.plan.payload_cap, 8 * self.plan.max_pieces, abort=ab)
            self._side.wait_stream(main)
            m = self.plan.max_pieces
            engine.awp_combine(self.tails[:self.world * 8 * m].view(torch.float64), self._piece_layer,
                               len(self.counts), self._sumsq_dev, self._side, abort=ab)
            engine.awp_observe(self._sumsq_dev, d.struct, d.config, self._side, abort=ab)
        engine.unpack_multi_dyn(self.unpack_table, self._peer[slot], self._pw_all, main, start_seg=self._unpack_start,
                                abort=ab)
        if observe:
            main.wait_stream(self._side)
            torch.index_select(d.widths_new, 0, self._idx_mine, out=self._pw_mine_new[:len(self._mine_layers)])
            torch.index_select(d.widths_new, 0, self._idx_all, out=self._pw_all_new[:len(self._all_layers)])
            engine.awp_fixup_pieces(self.pack_table, self._my_reps, self._mine_layers, send, d.escalated,
                                    self._pw_mine_new, main, abort=ab)
            self._barrier()
            engine.awp_fixup_gather(self.unpack_table, self._all_layers, self._peer[slot], d.escalated,
                                    self._pw_all_new, main, abort=ab)
            d.widths.copy_(d.widths_new)
        self._mirror_abort()

    def _step_device(self, batch: int, observe: bool, graphed: bool = True) -> SyncResult:
        self._poll_abort()
        d = self._dawp
        if observe and not d.label_set:
            d.set_next_label(batch - 1)
        slot = self._slot
        self._slot ^= 1
        if graphed:
            key = (slot, observe)
            g = self._dgraphs.get(key)
            if g is None:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._device_step_kernels(slot, observe)
                self._dgraphs[key] = g
            g.replay()
        else:
            self._device_step_kernels(slot, observe)
        self._step_queued()
        if observe:
            d.pending += 1
            if d.pending >= d.ring_steps:
                self._trace_log += self._drain_device()
        return SyncResult(round_tos=None)

    def _drain_device(self) -> list[tuple]:
        self.check_barrier()
        rows = self._dawp.drain()
        if getattr(self, "_check_finite", False):
            bad = next((r for r in rows if not math.isfinite(r[2])), None)
            if bad is not None:
                raise NonFiniteParameters(f"layer {bad[1]} parameters left the finite range (batch {bad[0]})")
        return rows

    def drain_trace(self) -> list[tuple]:
        """awp_on_device: the trace rows observed since the last call (every
        rank gets the same rows); refreshes the host controller."""
        if not self.awp_on_device:
            raise RuntimeError("drain_trace() is for awp_on_device=True")
        rows = self._trace_log + self._drain_device()
        self._trace_log = []
        return rows

    # ------------------------------------------------------------- planning
    def _plan(self, round_tos):
        from .layout import PackedLayout
        if getattr(self, "_owners_fixed", False):
            self.plan = self.plan.with_widths(round_tos)
        else:
            self.plan = ShardPlan.plan(self.counts, round_tos, self.world, self._align)
        S = self.plan.send_bytes
        if self.send is None or self.send[0].numel() < S:
            widest = [4] * len(self.counts)
            cap = max(S, (self.plan.with_widths(widest) if getattr(self, "_owners_fixed", False)
                          else ShardPlan.plan(self.counts, widest, self.world, self._align)).send_bytes)
            self._alloc(cap)
        if self.transport == "p2p":
            need = self.world * 8 * self.plan.max_pieces
            if getattr(self, "tails", None) is None or self.tails.numel() < need:
                self.tails = torch.zeros(need, dtype=torch.uint8, device=self.device)
        mine = self.plan.pieces[self.rank]
        views = [self.masters[pc.layer][pc.lo:pc.hi] for pc in mine]
        lay = PackedLayout(tuple(pc.hi - pc.lo for pc in mine), tuple(self.plan.round_tos[pc.layer] for pc in mine),
                           tuple(pc.offset for pc in mine), self.plan.payload_cap)
        self.pack_table = engine.SegmentTable(views, lay)
        if getattr(self, "_partials", None) is None or self._partials.numel() < self.pack_table.npartials:
            self._partials = torch.empty(max(1, self.pack_table.npartials), dtype=torch.float64, device=self.device)
        outs, cnt, rs, offs, srcs = [], [], [], [], []
        for q in range(self.world):
            for pc in self.plan.pieces[q]:
                outs.append(self.replicas[pc.layer][pc.lo:pc.hi])
                cnt.append(pc.hi - pc.lo)
                rs.append(self.plan.round_tos[pc.layer])
                # nccl: offsets inside the gathered buffer; p2p: inside rank q's own send buffer
                offs.append(pc.offset if self.transport == "p2p" else q * S + pc.offset)
                srcs.append(q if self.transport == "p2p" else 0)
        self.unpack_layout = PackedLayout(tuple(cnt), tuple(rs), tuple(offs), S * self.world)
        # p2p: this rank's gather-unpack walk starts just before its own pieces, so
        # at any moment the ranks pull from different peers (not one owner in lockstep)
        self._unpack_start = sum(len(self.plan.pieces[q]) for q in range(self.rank))
        self.grad_ranges = shard_ranges(self.plan, self.counts)
        self._reduce_table = None
        self._graphs = None
        self.unpack_table = engine.SegmentTable(outs, self.unpack_layout,
                                                sources=srcs if self.transport == "p2p" else None)
        if self.transport == "nccl" and self._collect:
            self._chunked = ChunkedGather.cut(self.plan, self.nccl_chunks)
            self._chunk_tables = []
            for segs in self._chunked.segments:
                if not segs:
                    self._chunk_tables.append(None)
                    continue
                lay = PackedLayout(tuple(hi - lo for _, _, lo, hi, _, _ in segs), tuple(r for *_, r, _ in segs),
                                   tuple(off for *_, off in segs), S * self.world)
                self._chunk_tables.append(engine.SegmentTable(
                    [self.replicas[layer][lo:hi] for _, layer, lo, hi, _, _ in segs], lay))

    def _alloc(self, cap: int) -> None:
        nslots = 2 if self.transport == "p2p" else 1
        self._close_peers()
        # p2p: a peer may still be reading our previous send buffers until it
        # reaches the handle exchange below (it syncs on its own unpack first),
        # so they stay referenced (not recycled by the caching allocator) until then.
        retired = self.send
        self.send = [torch.zeros(cap, dtype=torch.uint8, device=self.device) for _ in range(nslots)]
        if self.transport == "nccl":
            # one rank: unpack straight from the send buffer (no gather, no copy)
            self.recv = self.send[0] if not self._collect else torch.zeros(cap * self.world, dtype=torch.uint8,
                                                                            device=self.device)
            return
        handles = [engine.ipc_handle(b) for b in self.send]
        everyone = [None] * self.world
        self.dist.all_gather_object(everyone, handles, group=self.group)
        self._peer = []
        for slot in range(nslots):
            ptrs = []
            for q in range(self.world):
                if q == self.rank:
                    ptrs.append(self.send[slot].data_ptr())
                else:
                    handle, offset = everyone[q][slot]
                    base = engine.ipc_open(handle)
                    self._opened.append(base)
                    ptrs.append(base + offset)
            self._peer.append(ptrs)
        del retired

    def _close_peers(self) -> None:
        for p in self._opened:
            engine.ipc_close(p)
        self._opened = []

    def __del__(self):
        try:
            self._close_peers()
            for p in self._gopened + self._bopened:
                engine.ipc_close(p)
        except Exception:
            pass

    @property
    def round_tos(self) -> list[int]:
        if getattr(self, "_dawp", None) is not None:
            return self._dawp.round_tos()            # device read
        return list(self.plan.round_tos)

    # ------------------------------------------------------------- one step
    def _init_barrier(self) -> bool:
        """p2p: every rank's epoch-flag array, IPC-mapped into every rank, for
        the device-side barrier (adt_peer_barrier). This is the first peer
        mapping; every rank votes on its success, so a failure on any rank
        returns False everywhere (no rank is left waiting in a collective)."""
        self._flags = torch.zeros(self.world, dtype=torch.int32, device=self.device)
        self._bstate = torch.zeros(2, dtype=torch.int32, device=self.device)
        self._abort = self._bstate[1:2]
        self._abort_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._poll_event = torch.cuda.Event()
        self._poll_pending = False
        handle = engine.ipc_handle(self._flags)
        everyone = [None] * self.world
        self.dist.all_gather_object(everyone, handle, group=self.group)
        self._flag_ptrs = []
        ok = True
        try:
            for q in range(self.world):
                if q == self.rank:
                    self._flag_ptrs.append(self._flags.data_ptr())
                else:
                    base = engine.ipc_open(everyone[q][0])
                    self._bopened.append(base)
                    self._flag_ptrs.append(base + everyone[q][1])
        except RuntimeError:
            ok = False
        votes = [None] * self.world
        self.dist.all_gather_object(votes, ok, group=self.group)
        if all(votes):
            return True
        for p in self._bopened:
            engine.ipc_close(p)
        self._bopened, self._flag_ptrs = [], []
        return False

    def _barrier(self) -> None:
        """Stream-ordered cross-rank barrier: every rank's pack is complete
        (and its previous unpack, by stream order) before anyone reads. One
        32-thread kernel: each rank stores its epoch into every peer's flag
        array over NVLink and waits for all of them in its own — no NCCL
        launch, no host round trip, capturable in a CUDA graph."""
        engine.peer_barrier(self._flag_ptrs, self.rank, self._bstate, timeout_s=self.barrier_timeout_s)

    def _mirror_abort(self) -> None:
        """Queue the D2H copy of the abort word into pinned memory at the end of
        a step (captured into the step's graph when capturing)."""
        if self.transport == "p2p":
            self._abort_host.copy_(self._abort, non_blocking=True)

    def _step_queued(self) -> None:
        if self.transport == "p2p":
            self._poll_event.record()
            self._poll_pending = True

    def _poll_abort(self) -> None:
        """Before queueing more work: wait for the previous step (so the host
        is at most one step ahead of the device) and raise PeerTimeout if its
        barrier gave up."""
        if self.transport != "p2p":
            return
        if self._poll_pending:
            self._poll_event.synchronize()
            self._poll_pending = False
            if int(self._abort_host[0]):
                self._aborted = int(self._abort_host[0])
        if getattr(self, "_aborted", 0):
            raise PeerTimeout(f"rank {self.rank}: peer barrier epoch {self._aborted} timed out after "
                              f"{self.barrier_timeout_s:g} s waiting for a peer; the step's peer reads were skipped")

    def check_barrier(self) -> None:
        """Raise PeerTimeout if a device barrier gave up waiting for a peer (its
        bounded wait returns instead of hanging the GPU). Synchronizes."""
        if self.transport == "p2p":
            bad = int(self._bstate[1].item())
            if bad:
                self._aborted = bad
                raise PeerTimeout(f"rank {self.rank}: peer barrier epoch {bad} timed out waiting for a peer")

    def launch(self, fused_norm: bool, mid_event: torch.cuda.Event | None = None) -> None:
        """pack shard (norm finalized into the send tail) -> exchange -> unpack."""
        self._poll_abort()
        S = self.plan.send_bytes
        if self.transport == "nccl":
            send = self.send[0][:S]
            engine.pack(self.pack_table, send, self._tail(send) if fused_norm else None)
            self._gather_unpack(send, mid_event)
            return
        slot = self._slot
        self._slot ^= 1
        self._p2p_step(slot, fused_norm, mid_event)
        self._step_queued()

    def _gather_unpack(self, send: torch.Tensor, mid_event=None) -> None:
        """nccl transport: all-gather the packed send buffers chunk by chunk
        (every chunk's collective is queued at once, so they run back to back
        on NCCL's stream) and unpack each chunk on this stream as soon as its
        gather completes: the unpack of chunk c overlaps the gather of c+1.
        mid_event (if given) is recorded once the gathers are queued."""
        stream = torch.cuda.current_stream()
        if not self._collect:                    # one rank: recv is the send buffer
            if mid_event is not None:
                mid_event.record(stream)
            engine.unpack(self.unpack_table, self.recv)
            return
        ch, recv = self._chunked, self.recv
        works = [self.dist.all_gather_into_tensor(recv[ch.region[c]:ch.region[c + 1]],
                                                  send[ch.bounds[c]:ch.bounds[c + 1]],
                                                  group=self.group, async_op=True)
                 for c in range(len(ch.bounds) - 1)]
        if mid_event is not None:
            mid_event.record(stream)
        for work, table in zip(works, self._chunk_tables):
            work.wait()                          # this stream waits for chunk c's gather
            if table is not None:
                engine.unpack(table, recv)

    def _p2p_step(self, slot: int, fused_norm: bool, mid_event=None) -> None:
        send = self.send[slot]
        engine.pack(self.pack_table, send, self._tail(send) if fused_norm else None,
                    partials=self._partials if fused_norm else None)
        self._barrier()
        if mid_event is not None:
            mid_event.record(torch.cuda.current_stream())
        if fused_norm:
            engine.copy_multi(self.tails, self._peer[slot], self.plan.payload_cap, 8 * self.plan.max_pieces,
                              abort=self._abort)
        engine.unpack_multi(self.unpack_table, self._peer[slot], start_seg=self._unpack_start, abort=self._abort)
        self._mirror_abort()

    def launch_graphed(self, fused_norm: bool) -> None:
        """p2p: launch() replayed from CUDA graphs — every op of the step is a
        device kernel (pack, the peer barrier with its device-side epoch, the
        tail gather, the fused gather-unpack), so one graph per send slot
        captures it and a step costs one graph launch. Other transports run
        eagerly."""
        if self.transport != "p2p":
            self.launch(fused_norm)
            return
        self._poll_abort()
        key = (fused_norm, self.plan)
        if getattr(self, "_graphs", None) is None or self._graphs[0] != key:
            graphs = []
            for slot in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._p2p_step(slot, fused_norm)
                graphs.append(g)
            self._graphs = (key, graphs)
        slot = self._slot
        self._slot ^= 1
        self._graphs[1][slot].replay()
        self._step_queued()

    def _tail(self, send: torch.Tensor) -> torch.Tensor:
        base = self.plan.payload_cap
        return send[base:base + 8 * self.plan.max_pieces].view(torch.float64)

    def _norms(self) -> list[float]:
        self.check_barrier()
        S, base, m = self.plan.send_bytes, self.plan.payload_cap, self.plan.max_pieces
        if self.transport == "nccl":
            g = (self._chunked.tails(self.recv, self.plan) if self._collect
                 else self.recv[:S].view(1, S)[:, base:base + 8 * m]).contiguous()
        else:
            g = self.tails[:self.world * 8 * m].view(self.world, 8 * m)
        tails = g.view(torch.float64).view(self.world, m).cpu().tolist()
        return [math.sqrt(v) for v in self.plan.combine_sumsq(tails)]

    def step(self, batch: int = 0, observe: bool | None = None) -> SyncResult:
        if observe is None:
            observe = self.adaptive and batch > 0
        if self.awp_on_device:
            return self._step_device(batch, observe)
        used = self.round_tos
        self.launch_graphed(fused_norm=observe)   # p2p: one graph replay; nccl: eager
        res = SyncResult(round_tos=used)
        if not observe:
            return res
        res.trace = self.schedule.observe_all(self._norms(), batch=batch - 1)
        new = self.schedule.round_tos()
        if new != used:
            self._plan(new)
            self.launch(fused_norm=False)
            res.round_tos = new
            res.repacked = True
        return res

    # ------------------------------------------- gradient return (§8f #4)
    def _grad_sources(self, bucket: GradBucket) -> tuple[list[int], int]:
        """Device addresses of every rank's gradients for this rank's shard,
        in rank order, and the byte base the piece offsets are relative to."""
        b0, b1 = self.grad_ranges[self.rank]
        if self.transport == "p2p":
            if self._gpeer is None or self._gpeer[0] != bucket.flat.data_ptr():
                for p in self._gopened:
                    engine.ipc_close(p)
                self._gopened = []
                handle = engine.ipc_handle(bucket.flat)
                everyone = [None] * self.world
                self.dist.all_gather_object(everyone, handle, group=self.group)
                ptrs = []
                for q in range(self.world):
                    if q == self.rank:
                        ptrs.append(bucket.flat.data_ptr())
                    else:
                        base = engine.ipc_open(everyone[q][0])
                        self._gopened.append(base)
                        ptrs.append(base + everyone[q][1])
                self._gpeer = (bucket.flat.data_ptr(), ptrs)
            return self._gpeer[1], 0
        mine = b1 - b0
        if self._grecv is None or self._grecv.numel() < max(4, mine * self.world):
            self._grecv = torch.empty(max(4, mine * self.world), dtype=torch.float32, device=self.device)
        if self._collect:
            splits = [e - b for b, e in self.grad_ranges]
            self.dist.all_to_all_single(self._grecv[:mine * self.world], bucket.flat[:sum(splits)],
                                        output_split_sizes=[mine] * self.world, input_split_sizes=splits,
                                        group=self.group)
            base = self._grecv.data_ptr()
            return [base + 4 * mine * q for q in range(self.world)], 4 * b0
        return [bucket.flat.data_ptr()], 0

    def update(self, bucket: GradBucket, sample_counts, lr: float, momentum: float = 0.9,
               weight_decay: float = 5e-4, batch: int = 0) -> SyncResult:
        """One data-parallel step (net.gather_and_update, net.py:203-257, over
        the ranks' gradient buckets, then the weight distribution):

        every rank's bucket -> [fused: gather this rank's shard of all ranks'
        gradients (p2p: peer loads over NVLink; nccl: all_to_all), combine
        them with the reference's weighting and pairwise tree, momentum-step
        the master shard, pack it at the AWP widths, fuse its norm]
        -> exchange packed bytes -> unpack every replica -> AWP observe.

        `sample_counts[q]` = rank q's GradientSet.sample_count. Only this
        rank's shard of `masters` / `velocities` is stepped (the masters are
        sharded, as in the paper's single master copy); the replicas hold
        every updated weight, truncated to the widths in force."""
        if len(sample_counts) != self.world:
            raise ValueError("one sample count per rank")
        if list(bucket.counts) != list(self.counts):
            raise ShapeMismatch("gradient bucket layer sizes differ from the masters")
        self._poll_abort()
        if self.velocities is None:
            self.velocities = [torch.zeros_like(m) for m in self.masters]
        self._owners_fixed = True
        grads, rel = self._grad_sources(bucket)
        if self._reduce_table is None:
            offs, _ = bucket_offsets(self.counts)
            mine = self.plan.pieces[self.rank]
            self._reduce_table = engine.ReduceSgdTable(
                [self.masters[pc.layer][pc.lo:pc.hi] for pc in mine],
                [self.velocities[pc.layer][pc.lo:pc.hi] for pc in mine],
                [4 * (offs[pc.layer] + pc.lo) - rel for pc in mine], self.pack_table.layout)
        if self.awp_on_device:
            d = self._dawp
            d.counter[1].fill_(int(batch))       # trace label of this observation
            d.label_set = True
            slot = self._slot
            self._slot ^= 1
            table = self._reduce_table

            def fused(send, widths, partials, stream):
                self._barrier()                  # every rank's gradients are written
                engine.reduce_sgd_pack_dyn(table, grads, sample_counts, lr, momentum, weight_decay, send, widths,
                                           partials, stream, abort=self._abort)
            self._device_step_kernels(slot, True, pack=fused)
            self._step_queued()
            self._check_finite = True
            d.pending += 1
            if d.pending >= d.ring_steps:
                self._trace_log += self._drain_device()
            return SyncResult(round_tos=None)
        S = self.plan.send_bytes
        if self.transport == "nccl":
            send = self.send[0][:S]
        else:
            slot = self._slot
            self._slot ^= 1
            send = self.send[slot]
            self._barrier()                      # every rank's gradients are written
        engine.reduce_sgd_pack(self._reduce_table, grads, sample_counts, lr, momentum, weight_decay, send,
                               self._tail(send), abort=self._abort)
        if self.transport == "nccl":
            self._gather_unpack(send)
        else:
            self._barrier()                      # every shard is stepped and packed
            engine.copy_multi(self.tails, self._peer[slot], self.plan.payload_cap, 8 * self.plan.max_pieces,
                              abort=self._abort)
            engine.unpack_multi(self.unpack_table, self._peer[slot], start_seg=self._unpack_start, abort=self._abort)
        used = self.round_tos
        res = SyncResult(round_tos=used)
        norms = self._norms()
        bad = [i for i, n in enumerate(norms) if not math.isfinite(n)]
        if bad:
            raise NonFiniteParameters(f"layer {bad[0]} parameters left the finite range")
        if not self.adaptive:
            return res
        res.trace = self.schedule.observe_all(norms, batch=batch)
        new = self.schedule.round_tos()
        if new != used:
            # re-pack the owners' (already stepped) master shards at the new
            # widths; ownership is fixed, so no master state moves
            self._plan(new)
            self.launch(fused_norm=False)
            res.round_tos = new
            res.repacked = True
        return res
