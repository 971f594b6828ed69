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


def _worker(rank, world, port, counts, rs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle as C
    rng = np.random.default_rng(1)
    layers = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    plan = ShardPlan.plan(counts, rs, world)
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
    dist.all_gather_into_tensor(recv, torch.from_numpy(send))
    recv = recv.numpy()
    ok = True
    # reassemble every layer's payload from the gathered pieces
    for layer, (w, r) in enumerate(zip(layers, rs)):
        parts = []
        for qq in range(world):
            for pc in plan.pieces[qq]:
                if pc.layer == layer:
                    base = qq * S + pc.offset
                    parts.append((pc.lo, recv[base:base + (pc.hi - pc.lo) * r].tobytes()))
        got = b"".join(p for _, p in sorted(parts))
        ok &= got == C.pack(w, r)
    tails = [recv[qq * S + plan.payload_cap: qq * S + plan.payload_cap + 8 * plan.max_pieces].view(np.float64)
             for qq in range(world)]
    norms = [math.sqrt(v) for v in plan.combine_sumsq(tails)]
    for w, n in zip(layers, norms):
        ref = math.sqrt(C.sumsq(w))
        ok &= abs(n - ref) <= 1e-12 * ref
    q.put((rank, ok, [float(x) for x in norms]))
    dist.destroy_process_group()


def test_gloo_world2_packed_allgather_reassembles_reference_payloads():
    counts = [20 * 25, 50 * 20 * 25, 3 * TILE + 17, 10 * 500, 9 * TILE]
    rs = [1, 2, 3, 4, 2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, rs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    # identical norm bits on both ranks -> identical AWP decisions
    assert res[0][2] == res[1][2]
