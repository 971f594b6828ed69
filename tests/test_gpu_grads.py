"""GPU parity of the gradient return path.

adt_reduce_sgd_pack combines 1..16 worker gradient contributions exactly as
the reference's net.gather_and_update (net.py:203-257: sample-count weights,
pairwise_sum tree, division by the total, momentum step) and packs the new
master in the same pass. Bar: W', v' and packed bytes bit-exact with the
reference (golden_reduce_sgd.npz, produced by the reference itself); AWP
decisions identical; norms within 1e-6 relative.

The multi-rank form (ShardedWeightSync.update, p2p transport: the peers'
gradient buckets read over CUDA IPC inside the kernel, the device-side peer
barrier) runs as 2 and 3 processes sharing cuda:0 — the boxes have one GPU.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch

from oracle import weightpack_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adt():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2004_02297_b200 as adt
    return adt


def test_reduce_sgd_pack_matches_reference(adt, golden_reduce_sgd):
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.grads import GradBucket
    from paper_2004_02297_b200.layout import PackedLayout
    for i, c in enumerate(golden_reduce_sgd):
        r = (i % 4) + 1
        n = c["w"].size
        w = torch.from_numpy(c["w"].reshape(-1).copy()).cuda()
        v = torch.from_numpy(c["v"].reshape(-1).copy()).cuda()
        buckets = [GradBucket([n]).load([torch.from_numpy(g.reshape(-1).copy()).cuda()]) for g in c["g"]]
        lay = PackedLayout.plan([n], [r])
        packed = torch.zeros(lay.nbytes, dtype=torch.uint8, device="cuda")
        ss = torch.empty(1, dtype=torch.float64, device="cuda")
        table = engine.ReduceSgdTable([w], [v], [0], lay)
        engine.reduce_sgd_pack(table, [b.flat.data_ptr() for b in buckets], c["counts"], *c["hp"], packed, ss)
        torch.cuda.synchronize()
        w1 = c["w1"].reshape(-1)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), w1.view(np.uint32)), (i, len(c["counts"]))
        assert np.array_equal(v.cpu().numpy().view(np.uint32), c["v1"].reshape(-1).view(np.uint32)), i
        lo, hi = lay.span(0)
        assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(w1, r), i
        assert math.sqrt(float(ss.item())) == pytest.approx(O.l2_norm(w1), rel=1e-12)


def test_reduce_sgd_pack_every_contribution_count(adt):
    """NC = 1..16 over a multi-layer ragged set (several tiles per layer,
    ragged tails, r = 1..4) against the oracle's combine + step."""
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.grads import GradBucket
    from paper_2004_02297_b200.layout import PackedLayout
    rng = np.random.default_rng(3)
    counts = [4096 * 2 + 5, 300, 4096 * 3, 77]
    rs = [1, 2, 3, 4]
    hp = (0.03, 0.9, 5e-4)
    lay = PackedLayout.plan(counts, rs)
    for nc in range(1, 17):
        w0 = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        v0 = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.01) for n in counts]
        gs = [[rng.standard_normal(n, dtype=np.float32) * np.float32(0.05) for n in counts] for _ in range(nc)]
        sc = [int(x) for x in rng.integers(1, 100, nc)]
        buckets = [GradBucket(counts).load([torch.from_numpy(x).cuda() for x in g]) for g in gs]
        w = [torch.from_numpy(x.copy()).cuda() for x in w0]
        v = [torch.from_numpy(x.copy()).cuda() for x in v0]
        packed = torch.zeros(lay.nbytes, dtype=torch.uint8, device="cuda")
        ss = torch.empty(len(counts), dtype=torch.float64, device="cuda")
        table = engine.ReduceSgdTable(w, v, [buckets[0].byte_offset(l) for l in range(len(counts))], lay)
        engine.reduce_sgd_pack(table, [b.flat.data_ptr() for b in buckets], sc, *hp, packed, ss)
        torch.cuda.synchronize()
        for l in range(len(counts)):
            w1, v1 = O.gather_and_update_weights(w0[l], v0[l], [g[l] for g in gs], sc, *hp)
            assert np.array_equal(w[l].cpu().numpy().view(np.uint32), w1.view(np.uint32)), (nc, l)
            assert np.array_equal(v[l].cpu().numpy().view(np.uint32), v1.view(np.uint32)), (nc, l)
            lo, hi = lay.span(l)
            assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(w1, rs[l]), (nc, l)
            assert math.sqrt(float(ss[l].item())) == pytest.approx(O.l2_norm(w1), rel=1e-12)


def test_reduce_sgd_pack_argument_errors(adt):
    from paper_2004_02297_b200 import _lib, engine
    from paper_2004_02297_b200.layout import PackedLayout
    w = torch.zeros(64, device="cuda")
    v = torch.zeros(64, device="cuda")
    g = torch.zeros(64, device="cuda")
    lay = PackedLayout.plan([64], [2])
    packed = torch.zeros(lay.nbytes, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        engine.ReduceSgdTable([w], [v], [4], lay)            # misaligned gradient offset
    table = engine.ReduceSgdTable([w], [v], [0], lay)
    with pytest.raises(ValueError):
        engine.reduce_sgd_pack(table, [g.data_ptr()] * 17, [1] * 17, 0.1, 0.9, 0.0, packed)
    with pytest.raises(_lib.AdtError):
        engine.reduce_sgd_pack(table, [g.data_ptr() + 4], [1], 0.1, 0.9, 0.0, packed)   # misaligned buffer


def test_weightsync_gather_and_update_walk(adt):
    """20 batches of WeightSync.gather_and_update with 3 weighted worker
    contributions (GradientSet lists and GradBuckets) and AWP, vs the oracle
    in the reference's order: combine + update -> norm -> observe -> pack at
    the new widths -> unpack."""
    from paper_2004_02297_b200.grads import GradBucket, GradientSet
    rng = np.random.default_rng(22)
    counts = [500, 25000, 4096 * 3 + 7, 5000]
    L = len(counts)
    hp = (0.05, 0.9, 5e-4)
    sc = [64, 17, 40]
    w_ref = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    v_ref = [np.zeros(n, np.float32) for n in counts]
    kw = dict(threshold=-2e-3, interval=3, step_bits=8, initial_bits=8)
    octl = O.OracleController(L, **kw)
    masters = [torch.from_numpy(w.copy()).cuda() for w in w_ref]
    sync = adt.WeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**kw)))
    sync.step(batch=0)
    bucket = GradBucket(counts, sample_count=sc[2])
    for b in range(20):
        grads = [[np.float32(0.4 + 0.1 * k) * w + rng.standard_normal(w.size, dtype=np.float32) * np.float32(0.002)
                  for w in w_ref] for k in range(3)]
        contribs = [GradientSet([torch.from_numpy(x).cuda() for x in grads[k]], [], sc[k]) for k in range(2)]
        contribs.append(bucket.load([torch.from_numpy(x).cuda() for x in grads[2]]))
        res = sync.gather_and_update(contribs, *hp, batch=b)
        for i in range(L):
            w_ref[i], v_ref[i] = O.gather_and_update_weights(w_ref[i], v_ref[i], [g[i] for g in grads], sc, *hp)
            octl.observe_layer(i, O.l2_norm(w_ref[i]))
        rs = [octl.round_to(i) for i in range(L)]
        assert res.round_tos == rs, b
        for i in range(L):
            assert np.array_equal(masters[i].cpu().numpy().view(np.uint32), w_ref[i].view(np.uint32)), (b, i)
            want = w_ref[i].view(np.uint32) & np.uint32(O.keep_mask(rs[i]))
            assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), (b, i)
        assert [row[5] for row in res.trace] == [octl.bits[i] for i in range(L)]
    assert max(sync.round_tos) > 1


def test_gather_and_update_nonfinite_raises(adt):
    from paper_2004_02297_b200.grads import GradientSet
    m = [torch.ones(100, device="cuda")]
    sync = adt.WeightSync(m)
    g = torch.full((100,), 3.0e38, device="cuda")
    with pytest.raises(adt.NonFiniteParameters):
        sync.gather_and_update([GradientSet([g], [], 64), GradientSet([g], [], 64)], lr=1.0)


def test_gather_and_update_shape_mismatch(adt):
    """net.py:218-229: no contributions, or gradients that do not fit the
    layers, raise ShapeMismatch (a ValueError) before any device work."""
    from paper_2004_02297_b200.grads import GradBucket, GradientSet
    sync = adt.WeightSync([torch.ones(100, device="cuda"), torch.ones(30, device="cuda")])
    with pytest.raises(adt.ShapeMismatch):
        sync.gather_and_update([], lr=0.1)
    with pytest.raises(adt.ShapeMismatch):
        sync.gather_and_update([GradientSet([torch.ones(100, device="cuda")], [], 4)], lr=0.1)
    with pytest.raises(adt.ShapeMismatch):
        sync.gather_and_update([GradientSet([torch.ones(100, device="cuda"), torch.ones(31, device="cuda")], [], 4)],
                               lr=0.1)
    with pytest.raises(adt.ShapeMismatch):
        sync.gather_and_update([GradBucket([100, 31])], lr=0.1)
    assert issubclass(adt.ShapeMismatch, ValueError)


# ------------------------------------------------ two ranks sharing cuda:0
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q, transport="p2p"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        extra = {}
        if transport == "nccl-real":             # one rank on a real NCCL communicator, collectives kept
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
            transport, extra = "nccl", dict(collectives_at_world1=True, nccl_chunks=3)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2004_02297_b200 as adt
        from paper_2004_02297_b200.grads import GradBucket
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        counts = [20 * 25, 50 * 20 * 25, 3 * 4096 + 17, 10 * 500, 9 * 4096]
        if transport.endswith("-tiny"):          # two tiles in all: some rank owns nothing
            transport, counts = transport[:-5], [37, 4100]
        L = len(counts)
        hp = (0.05, 0.9, 5e-4)
        sc = [48, 80, 17, 5, 64, 33, 9, 21][:world]
        rng = np.random.default_rng(11)          # same stream on every rank
        w_ref = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        v_ref = [np.zeros(n, np.float32) for n in counts]
        masters = [torch.from_numpy(w.copy()).cuda() for w in w_ref]
        kw = dict(threshold=-2e-3, interval=2, step_bits=8, initial_bits=8)
        octl = O.OracleController(L, **kw)
        sync = ShardedWeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**kw)), transport=transport,
                                 **extra)
        bucket = GradBucket(counts)
        ok, notes, seen = True, [], []
        for b in range(8):
            grads = [[np.float32(0.5 + 0.2 * k) * w + rng.standard_normal(w.size, dtype=np.float32)
                      * np.float32(0.002) for w in w_ref] for k in range(world)]
            bucket.load([torch.from_numpy(x).cuda() for x in grads[rank]])
            res = sync.update(bucket, sc, *hp, batch=b)
            torch.cuda.synchronize()
            for i in range(L):
                w_ref[i], v_ref[i] = O.gather_and_update_weights(w_ref[i], v_ref[i], [g[i] for g in grads], sc, *hp)
                octl.observe_layer(i, O.l2_norm(w_ref[i]))
            rs = [octl.round_to(i) for i in range(L)]
            if res.round_tos != rs:
                ok = False
                notes.append(f"batch {b}: widths {res.round_tos} != {rs}")
            for i in range(L):
                want = w_ref[i].view(np.uint32) & np.uint32(O.keep_mask(rs[i]))
                if not np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want):
                    ok = False
                    notes.append(f"batch {b} layer {i} replica mismatch")
            for row in res.trace:
                ref = O.l2_norm(w_ref[row[1]])
                if abs(row[2] - ref) > 1e-6 * ref:
                    ok = False
                    notes.append(f"norm {row} vs {ref}")
                seen.append(row[2])
        q.put((rank, ok, notes, seen, sync.round_tos))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface child failures to the parent
        import traceback
        q.put((rank, False, [traceback.format_exc()], [], []))


@pytest.mark.parametrize("world,transport", [(2, "p2p"), (3, "p2p"), (8, "p2p"), (2, "nccl"), (3, "nccl"),
                                             (3, "p2p-tiny"), (3, "nccl-tiny"), (1, "nccl-real")])
def test_sharded_update_processes_sharing_one_gpu(world, transport):
    """transport="nccl": the all_to_all gradient exchange + all-gather path,
    run over gloo with CUDA tensors (NCCL refuses two ranks on one device).
    "nccl-real": the same path on a real one-rank NCCL communicator
    (collectives_at_world1: all_to_all_single and the chunked
    all_gather_into_tensor go through NCCL, its streams and work.wait())."""
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, notes, _, _ in res:
        assert ok, (rank, notes[:5])
    assert all(r[3] == res[0][3] for r in res) and len(res[0][3]) > 0   # identical norm bits on every rank
    assert all(r[4] == res[0][4] for r in res) and max(res[0][4]) > 1


def test_device_awp_gather_and_update_matches_host(adt):
    """gather_and_update with the AWP decision on the device (no host read per
    step) vs the host-controller WeightSync: identical masters, replicas,
    widths and trace rows; update() likewise."""
    from paper_2004_02297_b200.grads import GradBucket
    rng = np.random.default_rng(23)
    counts = [500, 25000, 4096 * 3 + 7, 5000]
    L = len(counts)
    hp = (0.05, 0.9, 5e-4)
    kw = dict(threshold=-2e-3, interval=3, step_bits=8, initial_bits=8)
    w0 = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    host = adt.WeightSync([torch.from_numpy(w.copy()).cuda() for w in w0],
                          adt.PrecisionController(L, adt.PrecisionConfig(**kw)))
    dev = adt.WeightSync([torch.from_numpy(w.copy()).cuda() for w in w0],
                         adt.PrecisionController(L, adt.PrecisionConfig(**kw)), awp_on_device=True, trace_ring=8)
    buckets = [GradBucket(counts, sample_count=c) for c in (64, 17, 40)]
    want = []
    for b in range(24):
        for k, bk in enumerate(buckets):
            bk.load([torch.from_numpy(np.float32(0.4 + 0.1 * k) * m.cpu().numpy()
                                      + rng.standard_normal(n, dtype=np.float32) * np.float32(0.002)).cuda()
                     for m, n in zip(host.masters, counts)])
        want += host.gather_and_update(buckets, *hp, batch=b).trace
        dev.gather_and_update(buckets, *hp, batch=b)
        if b % 6 == 5:
            assert dev.round_tos == host.round_tos, b
            for x, y in zip(host.masters + host.replicas, dev.masters + dev.replicas):
                assert torch.equal(x, y), b
    got = dev.drain_trace()
    assert got == want
    assert max(host.round_tos) > 1
    # update() (one pre-averaged gradient)
    g = [torch.randn(n, device="cuda") * 0.01 for n in counts]
    r1 = host.update(g, *hp, batch=24).trace
    dev.update(g, *hp, batch=24)
    assert dev.drain_trace() == r1
    assert all(torch.equal(x, y) for x, y in zip(host.replicas, dev.replicas))


def _device_rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2004_02297_b200 as adt
        from paper_2004_02297_b200.grads import GradBucket
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        counts = [20 * 25, 50 * 20 * 25, 3 * 4096 + 17, 10 * 500, 9 * 4096]
        L = len(counts)
        hp = (0.05, 0.9, 5e-4)
        sc = [48, 80, 17][:world]
        rng = np.random.default_rng(11)
        w_ref = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        v_ref = [np.zeros(n, np.float32) for n in counts]
        masters = [torch.from_numpy(w.copy()).cuda() for w in w_ref]
        kw = dict(threshold=-2e-3, interval=2, step_bits=8, initial_bits=8)
        octl = O.OracleController(L, **kw)
        sync = ShardedWeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**kw)), transport="p2p",
                                 awp_on_device=True, trace_ring=4)
        bucket = GradBucket(counts)
        ok, notes, want = True, [], []
        for b in range(8):
            grads = [[np.float32(0.5 + 0.2 * k) * w + rng.standard_normal(w.size, dtype=np.float32)
                      * np.float32(0.002) for w in w_ref] for k in range(world)]
            bucket.load([torch.from_numpy(x).cuda() for x in grads[rank]])
            sync.update(bucket, sc, *hp, batch=b)
            torch.cuda.synchronize()
            for i in range(L):
                w_ref[i], v_ref[i] = O.gather_and_update_weights(w_ref[i], v_ref[i], [g[i] for g in grads], sc, *hp)
                octl.observe_layer(i, O.l2_norm(w_ref[i]))
                want.append((b, i, octl.bits[i], octl.counter[i]))
            rs = [octl.round_to(i) for i in range(L)]
            if sync.round_tos != rs:
                ok = False
                notes.append(f"batch {b}: widths {sync.round_tos} != {rs}")
            for i in range(L):
                want_w = w_ref[i].view(np.uint32) & np.uint32(O.keep_mask(rs[i]))
                if not np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want_w):
                    ok = False
                    notes.append(f"batch {b} layer {i} replica mismatch")
        rows = sync.drain_trace()
        if [(r[0], r[1], r[5], r[4]) for r in rows] != want:
            ok = False
            notes.append(f"trace {[(r[0], r[1], r[5], r[4]) for r in rows][:4]} vs {want[:4]}")
        q.put((rank, ok, notes[:5], [r[2] for r in rows]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, [traceback.format_exc()], []))


def test_sharded_update_p2p_device_awp_two_processes():
    """The whole data-parallel step with the AWP decision on the device:
    fused gradient reduce over peer buckets + SGD + pack at device widths,
    gathered norms, device decision, re-pack/re-gather of escalated pieces."""
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, notes, _ in res:
        assert ok, (rank, notes)
    assert res[0][3] == res[1][3] and len(res[0][3]) > 0


@pytest.mark.parametrize("nc", [1, 3, 8])
def test_reduce_sgd_pack_full_alexnet_matches_per_op_torch(adt, nc):
    """The fused gradient combine + SGD + pack at the full AlexNet set against
    the same arithmetic as separate float32 torch ops (each op rounds once;
    no alpha= forms, which may contract to FMA): masters, velocities and packed
    payloads bit-identical — the full-size counterpart of the golden tests."""
    from paper_2004_02297_b200 import engine, workloads
    from paper_2004_02297_b200.grads import GradBucket
    from paper_2004_02297_b200.layout import PackedLayout
    counts = workloads.counts_of("alexnet")
    rs = [(b + 7) // 8 for b in workloads.default_bits("alexnet")]
    lr, mu, wd = 0.01, 0.9, 5e-4
    g = torch.Generator(device="cuda").manual_seed(11)
    w = [torch.randn(n, device="cuda", generator=g) * 0.1 for n in counts]
    v = [torch.randn(n, device="cuda", generator=g) * 0.01 for n in counts]
    w_ref, v_ref = [x.clone() for x in w], [x.clone() for x in v]
    sc = [int(x) for x in torch.randint(1, 200, (nc,), generator=torch.Generator().manual_seed(nc))]
    buckets = []
    for _ in range(nc):
        b = GradBucket(counts)
        b.flat.normal_(generator=g).mul_(0.05)
        buckets.append(b)
    lay = PackedLayout.plan(counts, rs)
    packed = torch.empty(lay.nbytes, dtype=torch.uint8, device="cuda")
    table = engine.ReduceSgdTable(w, v, [buckets[0].byte_offset(l) for l in range(len(counts))], lay)
    engine.reduce_sgd_pack(table, [b.flat.data_ptr() for b in buckets], sc, lr, mu, wd, packed)
    total = torch.tensor(float(sum(sc)), dtype=torch.float32, device="cuda")
    for l in range(len(counts)):
        level = [b.views[l].reshape(-1) * torch.tensor(float(c), device="cuda") for b, c in zip(buckets, sc)]
        while len(level) > 1:                     # net.py pairwise_sum association
            carry = level[-1:] if len(level) % 2 else []
            level = [a + b for a, b in zip(level[0::2], level[1::2])] + carry
        gl = level[0] / total
        gl = gl + wd * w_ref[l]
        v_ref[l] = v_ref[l] * mu + gl
        w_ref[l] = w_ref[l] - lr * v_ref[l]
    ref_packed, ref_lay, _ = adt.pack_many(w_ref, rs)
    for l in range(len(counts)):
        assert torch.equal(w[l].view(torch.int32), w_ref[l].view(torch.int32)), l
        assert torch.equal(v[l].view(torch.int32), v_ref[l].view(torch.int32)), l
        lo, hi = lay.span(l)
        rlo, rhi = ref_lay.span(l)
        assert torch.equal(packed[lo:hi], ref_packed[rlo:rhi]), l
