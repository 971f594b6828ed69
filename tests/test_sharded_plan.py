"""ShardPlan host logic + a real world_size-2 collective on CPU (gloo).

The GPU box has one GPU, so the N>1 path's host side is covered here: the
plan's partition, alignment and layout, and a gloo all_gather of packed shard
buffers (bytes produced by the C oracle in this test) that every rank must
reassemble into exactly the reference's per-layer payloads and norms."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2004_02297_b200 import workloads
from paper_2004_02297_b200.sharded import ShardPlan

TILE = 4096


def check_plan(plan, counts, rs):
    covered = [[] for _ in counts]
    for q in range(plan.world):
        off_end = 0
        for pc in plan.pieces[q]:
            assert pc.offset % 16 == 0 and pc.offset >= off_end
            assert pc.lo % TILE == 0
            covered[pc.layer].append((pc.lo, pc.hi))
            off_end = pc.offset + (pc.hi - pc.lo) * rs[pc.layer]
        assert off_end <= plan.payload_cap
    for layer, spans in enumerate(covered):
        spans.sort()
        pos = 0
        for lo, hi in spans:
            assert lo == pos and hi > lo
            pos = hi
        assert pos == counts[layer]
    assert plan.send_bytes % 16 == 0 and plan.send_bytes >= plan.payload_cap + 8 * plan.max_pieces


@pytest.mark.parametrize("name", ["lenet", "alexnet", "vgg16", "resnet50"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_partition_is_exact_and_balanced(name, world):
    counts = workloads.counts_of(name)
    rs = [(i % 4) + 1 for i in range(len(counts))] if name == "alexnet" else [1] * len(counts)
    plan = ShardPlan.plan(counts, rs, world)
    check_plan(plan, counts, rs)
    total = sum(n * r for n, r in zip(counts, rs))
    if world > 1 and total > 64 * TILE * world:
        worst = max(plan.rank_payload_bytes(q) for q in range(world))
        assert worst <= total / world + 4 * TILE * 4 + 16 * len(counts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, rs, q, chunks=0):
    """chunks = 0: one all_gather_into_tensor of the send buffers; chunks > 0:
    the nccl transport's chunked gather (ChunkedGather, async collectives
    queued at once, completed in order)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle as C
    from paper_2004_02297_b200.sharded import SPLIT_ALIGN, ChunkedGather
    rng = np.random.default_rng(1)
    layers = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    plan = ShardPlan.plan(counts, rs, world, SPLIT_ALIGN if chunks else 16)
    S = plan.send_bytes
    send = np.zeros(S, np.uint8)
    sums = np.zeros(plan.max_pieces, np.float64)
    for k, pc in enumerate(plan.pieces[rank]):
        seg = layers[pc.layer][pc.lo:pc.hi]
        b = np.frombuffer(C.pack(seg, rs[pc.layer]), np.uint8)
        send[pc.offset:pc.offset + b.size] = b
        sums[k] = C.sumsq(seg)
    send[plan.payload_cap:plan.payload_cap + 8 * plan.max_pieces] = sums.view(np.uint8)
    recv = torch.zeros(S * world, dtype=torch.uint8)
    if chunks:
        ch = ChunkedGather.cut(plan, chunks)
        src = torch.from_numpy(send)
        works = [dist.all_gather_into_tensor(recv[ch.region[c]:ch.region[c + 1]], src[ch.bounds[c]:ch.bounds[c + 1]],
                                             async_op=True) for c in range(len(ch.bounds) - 1)]
        for w_ in works:
            w_.wait()
        tails = [t.view(np.float64) for t in ch.tails(recv, plan).numpy()]
        recv = recv.numpy()
        located = [(layer, lo, recv[off:off + (hi - lo) * r].tobytes())
                   for segs in ch.segments for _, layer, lo, hi, r, off in segs]
    else:
        dist.all_gather_into_tensor(recv, torch.from_numpy(send))
        recv = recv.numpy()
        tails = [recv[qq * S + plan.payload_cap: qq * S + plan.payload_cap + 8 * plan.max_pieces].view(np.float64)
                 for qq in range(world)]
        located = [(pc.layer, pc.lo, recv[qq * S + pc.offset:qq * S + pc.offset + (pc.hi - pc.lo) * rs[pc.layer]]
                    .tobytes()) for qq in range(world) for pc in plan.pieces[qq]]
    ok = True
    # reassemble every layer's payload from the gathered pieces
    for layer, (w, r) in enumerate(zip(layers, rs)):
        got = b"".join(p for _, p in sorted((lo, p) for lyr, lo, p in located if lyr == layer))
        ok &= got == C.pack(w, r)
    norms = [math.sqrt(v) for v in plan.combine_sumsq(tails)]
    for w, n in zip(layers, norms):
        ref = math.sqrt(C.sumsq(w))
        ok &= abs(n - ref) <= 1e-12 * ref
    q.put((rank, ok, [float(x) for x in norms]))
    dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [0, 3])
def test_gloo_world2_packed_allgather_reassembles_reference_payloads(chunks):
    counts = [20 * 25, 50 * 20 * 25, 3 * TILE + 17, 10 * 500, 9 * TILE]
    rs = [1, 2, 3, 4, 2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, rs, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    # identical norm bits on both ranks -> identical AWP decisions
    assert res[0][2] == res[1][2]


# ------------------------------------------- gradient return (§8f #4) host logic
@pytest.mark.parametrize("name", ["lenet", "alexnet", "resnet50"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_grad_shard_ranges_tile_the_bucket(name, world):
    from paper_2004_02297_b200.grads import bucket_offsets, shard_ranges
    counts = workloads.counts_of(name)
    rs = [(i % 4) + 1 for i in range(len(counts))]
    plan = ShardPlan.plan(counts, rs, world)
    offs, total = bucket_offsets(counts)
    assert all(o % 4 == 0 for o in offs) and total % 4 == 0
    ranges = shard_ranges(plan, counts)
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    for (b0, e0), (b1, _) in zip(ranges, ranges[1:]):
        assert e0 == b1 and b0 <= e0
    for q, (b, e) in enumerate(ranges):
        assert b % 4 == 0
        for pc in plan.pieces[q]:
            lo = offs[pc.layer] + pc.lo
            assert b <= lo and lo + (pc.hi - pc.lo) <= e
    # fixed ownership at new widths keeps every piece, moves only packed offsets
    wide = plan.with_widths([4] * len(counts))
    check_plan(wide, counts, [4] * len(counts))
    assert [[(p.layer, p.lo, p.hi) for p in x] for x in wide.pieces] == \
        [[(p.layer, p.lo, p.hi) for p in x] for x in plan.pieces]


def _a2a_worker(rank, world, port, counts, rs, q):
    """The NCCL transport's gradient exchange on CPU (gloo all_to_all_single):
    each rank must receive every rank's gradients for exactly its own pieces,
    and combining them (oracle) must equal the reference's combine of the
    full layers restricted to those pieces."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import weightpack_oracle as O
    from paper_2004_02297_b200.grads import bucket_offsets, shard_ranges
    plan = ShardPlan.plan(counts, rs, world)
    offs, total = bucket_offsets(counts)
    rng = np.random.default_rng(5)
    grads = [[rng.standard_normal(n, dtype=np.float32) for n in counts] for _ in range(world)]
    sc = [3, 64, 17][:world]
    flat = np.zeros(total, np.float32)
    for layer, g in enumerate(grads[rank]):
        flat[offs[layer]:offs[layer] + g.size] = g
    ranges = shard_ranges(plan, counts)
    b0, b1 = ranges[rank]
    mine = b1 - b0
    recv = torch.zeros(mine * world)
    dist.all_to_all_single(recv, torch.from_numpy(flat), output_split_sizes=[mine] * world,
                           input_split_sizes=[e - b for b, e in ranges])
    recv = recv.numpy()
    ok = True
    for pc in plan.pieces[rank]:
        rel = offs[pc.layer] + pc.lo - b0
        n = pc.hi - pc.lo
        contrib = [recv[c * mine + rel:c * mine + rel + n] for c in range(world)]
        got = O.combine_gradients(contrib, sc)
        want = O.combine_gradients([g[pc.layer] for g in grads], sc)[pc.lo:pc.hi]
        ok &= np.array_equal(got.view(np.uint32), want.view(np.uint32))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_alltoall_gradient_shards_match_reference_combine(world):
    counts = [20 * 25, 50 * 20 * 25, 3 * TILE + 17, 10 * 500, 9 * TILE]
    rs = [1, 2, 3, 4, 2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, counts, rs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res)


# ------------------------------------------- chunked all-gather (nccl transport)
@pytest.mark.parametrize("name,world,chunks", [("lenet", 2, 4), ("resnet50", 3, 4), ("resnet50", 8, 7),
                                               ("ragged", 2, 1), ("ragged", 4, 5), ("ragged", 5, 64)])
def test_chunked_gather_reassembles_every_piece(name, world, chunks):
    """Simulate the chunk-by-chunk all-gather in NumPy: every unpack segment
    of every chunk must address exactly its piece's packed bytes in the
    owner's send buffer, the parts must tile each piece in order, and every
    kernel-side alignment (16-B packed offsets, 4-weight FP32 starts) holds."""
    if name == "ragged":
        counts = [5, 4096 * 3 + 7, 1, 70000, 16, 4096 * 9 + 4095, 12345]
    else:
        counts = workloads.counts_of(name)
    check_chunked(counts, [(i % 4) + 1 for i in range(len(counts))], world, chunks)


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(1, 40000), min_size=1, max_size=9), st.data(),
       st.integers(1, 9), st.integers(1, 12))
def test_chunked_gather_property(counts, data, world, chunks):
    rs = data.draw(st.lists(st.integers(1, 4), min_size=len(counts), max_size=len(counts)))
    check_chunked(counts, rs, world, chunks)


def check_chunked(counts, rs, world, chunks):
    from paper_2004_02297_b200.sharded import SPLIT_ALIGN, ChunkedGather
    plan = ShardPlan.plan(counts, rs, world, SPLIT_ALIGN)
    check_plan(plan, counts, rs)
    assert all(pc.offset % SPLIT_ALIGN == 0 for x in plan.pieces for pc in x)
    ch = ChunkedGather.cut(plan, chunks)
    S = plan.send_bytes
    assert ch.bounds[0] == 0 and ch.bounds[-1] == S and list(ch.bounds) == sorted(set(ch.bounds))
    assert all(b % SPLIT_ALIGN == 0 for b in ch.bounds[:-1]) and ch.bounds[-2] < max(plan.payload_cap, 1)
    assert ch.region[-1] == world * S
    sends = [((np.arange(S, dtype=np.int64) * 7 + q * 13) % 251).astype(np.uint8) for q in range(world)]
    recv = np.zeros(world * S, np.uint8)
    for c in range(len(ch.bounds) - 1):                 # the chunk's rank-major all-gather
        b0, b1 = ch.bounds[c], ch.bounds[c + 1]
        for q in range(world):
            recv[ch.region[c] + q * (b1 - b0):ch.region[c] + (q + 1) * (b1 - b0)] = sends[q][b0:b1]
    parts = {}
    for segs in ch.segments:
        for q, layer, lo, hi, r, off in segs:
            assert off % 16 == 0 and lo % 4 == 0 and hi > lo
            parts.setdefault((q, layer), []).append((lo, hi, r, off))
    for q in range(world):
        for pc in plan.pieces[q]:
            got = parts.pop((q, pc.layer))
            r = plan.round_tos[pc.layer]
            pos = pc.lo
            for lo, hi, rr, off in got:                 # chunk order = stream order
                assert lo == pos and rr == r
                want = sends[q][pc.offset + (lo - pc.lo) * r:pc.offset + (hi - pc.lo) * r]
                assert np.array_equal(recv[off:off + (hi - lo) * r], want)
                pos = hi
            assert pos == pc.hi
    assert not parts
    tails = ch.tails(torch.from_numpy(recv), plan).numpy()
    base, m = plan.payload_cap, plan.max_pieces
    for q in range(world):
        assert np.array_equal(tails[q], sends[q][base:base + 8 * m])


def test_chunked_gather_refuses_unsplittable_plan():
    from paper_2004_02297_b200.sharded import ChunkedGather
    with pytest.raises(ValueError):
        ChunkedGather.cut(ShardPlan.plan([100, 200], [3, 1], 2), 4)
