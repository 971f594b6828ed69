"""Multi-GPU weight distribution: shard-pack -> all-gather packed bytes -> unpack.

The reference simulates data-parallel workers in one process and only
*accounts* the bytes each worker would receive (training.py:214-225,
transfer.py:143-174). Here every rank is one GPU (torchrun, NCCL over
NVLink 5): rank p packs its contiguous shard of the concatenated layers at
the AWP widths (norm partials fused into the same read), one
`all_gather_into_tensor` (ncclAllGather on uint8) moves ONLY packed bytes,
and every rank unpacks the whole gathered stream into its full FP32 replica.

Send buffer of rank p (S_max bytes, identical size on every rank):
    [piece payloads, 16-B aligned | pad | float64 sum of squares per piece]
The norm tail rides the same collective, so every rank combines the per-piece
sums in fixed rank order and sees bit-identical norms -> identical AWP
decisions on every rank with no extra collective.

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
from .sync import SyncResult


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

    @staticmethod
    def plan(counts: Sequence[int], round_tos: Sequence[int], world: int) -> "ShardPlan":
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
                off = align_up(off + (hi - lo) * round_tos[layer])
            cap = max(cap, off)
            pieces.append(tuple(lst))
        max_pieces = max(1, max(len(x) for x in pieces))
        cap = align_up(max(cap, 16))
        return ShardPlan(counts, round_tos, world, tuple(pieces), cap, max_pieces,
                         align_up(cap + 8 * max_pieces))

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


class ShardedWeightSync:
    """Per-step packed weight distribution across the ranks of `group`.

    `masters[l]` are this rank's FP32 master tensors (full layer shape; only
    this rank's shard ranges are read), `replicas[l]` receive every weight.

    transport = "nccl": pack -> ncclAllGather(uint8) of the packed send
        buffers -> unpack the gathered stream.
    transport = "p2p": every rank's send buffer is mapped into every other
        rank with CUDA IPC; after one stream-ordered barrier each rank unpacks
        straight out of its peers' send buffers over NVLink
        (adt_unpack_multi) — the gather and the unpack are one kernel, and the
        gathered stream is never written to or re-read from HBM. Send buffers
        alternate between two slots so one barrier per step covers both the
        read-after-write and the write-after-read hazard.
    """

    def __init__(self, masters: Sequence[torch.Tensor], schedule=None, replicas=None, group=None,
                 transport: str = "nccl"):
        import torch.distributed as dist
        engine.require_cuda()
        if transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        self.dist = dist
        self.group = group
        self.transport = transport
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.masters = [m.detach().reshape(-1) for m in masters]
        self.counts = [m.numel() for m in self.masters]
        self.schedule = schedule if schedule is not None else FixedPrecision(len(self.masters), 32)
        self.adaptive = isinstance(self.schedule, PrecisionController)
        self.device = self.masters[0].device
        if replicas is None:
            replicas = [torch.empty_like(m) for m in self.masters]
        self.replicas = [r.reshape(-1) for r in replicas]
        self.send = self.recv = None
        self._slot = 0
        self._peer = None      # p2p: per slot, every rank's send-buffer address in this process
        self._opened = []
        self._plan(self.schedule.round_tos())

    # ------------------------------------------------------------- planning
    def _plan(self, round_tos):
        from .layout import PackedLayout
        self.plan = ShardPlan.plan(self.counts, round_tos, self.world)
        S = self.plan.send_bytes
        if self.send is None or self.send[0].numel() < S:
            cap = max(S, ShardPlan.plan(self.counts, [4] * len(self.counts), self.world).send_bytes)
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
        self.unpack_table = engine.SegmentTable(outs, self.unpack_layout,
                                                sources=srcs if self.transport == "p2p" else None)

    def _alloc(self, cap: int) -> None:
        nslots = 2 if self.transport == "p2p" else 1
        self._close_peers()
        self.send = [torch.zeros(cap, dtype=torch.uint8, device=self.device) for _ in range(nslots)]
        if self.transport == "nccl":
            # one rank: unpack straight from the send buffer (no gather, no copy)
            self.recv = self.send[0] if self.world == 1 else torch.zeros(cap * self.world, dtype=torch.uint8,
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

    def _close_peers(self) -> None:
        for p in self._opened:
            engine.ipc_close(p)
        self._opened = []

    def __del__(self):
        try:
            self._close_peers()
        except Exception:
            pass

    @property
    def round_tos(self) -> list[int]:
        return list(self.plan.round_tos)

    # ------------------------------------------------------------- one step
    def _barrier(self) -> None:
        """Stream-ordered cross-rank barrier: every rank's pack is complete
        (and its previous unpack, by stream order) before anyone reads."""
        if self.dist.get_backend(self.group) == "nccl":
            if not hasattr(self, "_flag"):
                self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.dist.all_reduce(self._flag, group=self.group)
        else:  # gloo (tests): host-side
            torch.cuda.current_stream().synchronize()
            self.dist.barrier(group=self.group)

    def launch(self, fused_norm: bool, mid_event: torch.cuda.Event | None = None) -> None:
        """pack shard (norm finalized into the send tail) -> exchange -> unpack."""
        S = self.plan.send_bytes
        if self.transport == "nccl":
            send, recv = self.send[0][:S], self.recv[:S * self.world]
            engine.pack(self.pack_table, send, self._tail(send) if fused_norm else None)
            if self.world > 1:
                self.dist.all_gather_into_tensor(recv, send, group=self.group)
            if mid_event is not None:
                mid_event.record(torch.cuda.current_stream())
            engine.unpack(self.unpack_table, recv)
            return
        slot = self._slot
        self._slot ^= 1
        send = self.send[slot]
        engine.pack(self.pack_table, send, self._tail(send) if fused_norm else None)
        self._barrier()
        if mid_event is not None:
            mid_event.record(torch.cuda.current_stream())
        if fused_norm:
            engine.copy_multi(self.tails, self._peer[slot], self.plan.payload_cap, 8 * self.plan.max_pieces)
        engine.unpack_multi(self.unpack_table, self._peer[slot])

    def _tail(self, send: torch.Tensor) -> torch.Tensor:
        base = self.plan.payload_cap
        return send[base:base + 8 * self.plan.max_pieces].view(torch.float64)

    def _norms(self) -> list[float]:
        S, base, m = self.plan.send_bytes, self.plan.payload_cap, self.plan.max_pieces
        if self.transport == "nccl":
            g = self.recv[:S * self.world].view(self.world, S)[:, base:base + 8 * m].contiguous()
        else:
            g = self.tails[:self.world * 8 * m].view(self.world, 8 * m)
        tails = g.view(torch.float64).view(self.world, m).cpu().tolist()
        return [math.sqrt(v) for v in self.plan.combine_sumsq(tails)]

    def step(self, batch: int = 0, observe: bool | None = None) -> SyncResult:
        if observe is None:
            observe = self.adaptive and batch > 0
        used = self.round_tos
        self.launch(fused_norm=observe)
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
