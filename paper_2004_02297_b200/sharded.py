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
    """Per-step packed weight all-gather across the ranks of `group`.

    `masters[l]` are this rank's FP32 master tensors (full layer shape; only
    this rank's shard ranges are read), `replicas[l]` receive every weight.
    """

    def __init__(self, masters: Sequence[torch.Tensor], schedule=None, replicas=None, group=None):
        import torch.distributed as dist
        engine.require_cuda()
        self.dist = dist
        self.group = group
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
        self._plan(self.schedule.round_tos())

    def _plan(self, round_tos):
        from .layout import PackedLayout
        self.plan = ShardPlan.plan(self.counts, round_tos, self.world)
        S = self.plan.send_bytes
        if self.send is None or self.send.numel() < S:
            cap = ShardPlan.plan(self.counts, [4] * len(self.counts), self.world).send_bytes
            self.send = torch.zeros(cap, dtype=torch.uint8, device=self.device)
            # one rank: unpack straight from the send buffer (no gather, no copy)
            self.recv = self.send if self.world == 1 else torch.zeros(cap * self.world, dtype=torch.uint8,
                                                                       device=self.device)
        mine = self.plan.pieces[self.rank]
        # pack table over this rank's pieces (views into the masters)
        views = [self.masters[pc.layer][pc.lo:pc.hi] for pc in mine]
        lay = PackedLayout(tuple(pc.hi - pc.lo for pc in mine), tuple(self.plan.round_tos[pc.layer] for pc in mine),
                           tuple(pc.offset for pc in mine), self.plan.payload_cap)
        self.pack_table = engine.SegmentTable(views, lay)
        # norm tail view inside the send buffer
        self.tail = self.send[self.plan.payload_cap:self.plan.payload_cap + 8 * self.plan.max_pieces].view(torch.float64)
        # unpack table over every rank's pieces in the gathered buffer
        outs, cnt, rs, offs = [], [], [], []
        for q in range(self.world):
            for pc in self.plan.pieces[q]:
                outs.append(self.replicas[pc.layer][pc.lo:pc.hi])
                cnt.append(pc.hi - pc.lo)
                rs.append(self.plan.round_tos[pc.layer])
                offs.append(q * S + pc.offset)
        self.unpack_layout = PackedLayout(tuple(cnt), tuple(rs), tuple(offs), S * self.world)
        self.unpack_table = engine.SegmentTable(outs, self.unpack_layout)

    @property
    def round_tos(self) -> list[int]:
        return list(self.plan.round_tos)

    def launch(self, fused_norm: bool, mid_event: torch.cuda.Event | None = None) -> None:
        """pack shard (norm finalized into the send tail) -> ncclAllGather -> unpack."""
        S = self.plan.send_bytes
        send = self.send[:S]
        recv = self.recv[:S * self.world]
        engine.pack(self.pack_table, send, self.tail if fused_norm else None)
        if self.world > 1:
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
        if mid_event is not None:
            mid_event.record(torch.cuda.current_stream())
        engine.unpack(self.unpack_table, recv)

    def _norms(self) -> list[float]:
        S = self.plan.send_bytes
        base = self.plan.payload_cap
        m = self.plan.max_pieces
        g = self.recv[:S * self.world].view(self.world, S)[:, base:base + 8 * m].contiguous()
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
