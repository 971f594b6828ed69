"""GPU tests of the multi-rank path on ONE device (the boxes have one GPU).

* virtual ranks in one process: every rank's packed send buffer is a local
  allocation; adt_unpack_multi must reassemble the reference's bytes;
* two processes sharing cuda:0 (gloo for the host-side exchange): the real
  ShardedWeightSync(transport="p2p") path — CUDA IPC mapping of the peer's send
  buffers, the peer-read norm tails and the fused gather-unpack — against the
  oracle, including an AWP escalation that re-plans the shards.
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


def test_unpack_multi_virtual_ranks(adt):
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    from paper_2004_02297_b200.sharded import ShardPlan
    rng = np.random.default_rng(4)
    counts = [500, 25000, 3 * 4096 + 17, 5000, 9 * 4096]
    rs = [1, 2, 3, 4, 2]
    hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in counts]
    world = 3
    plan = ShardPlan.plan(counts, rs, world)
    bufs = []
    for q in range(world):
        b = np.zeros(plan.send_bytes, np.uint8)
        for pc in plan.pieces[q]:
            pay = np.frombuffer(O.pack_vectorized(hosts[pc.layer][pc.lo:pc.hi], rs[pc.layer]), np.uint8)
            b[pc.offset:pc.offset + pay.size] = pay
        bufs.append(torch.from_numpy(b).cuda())
    outs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in counts]
    views, cnt, rr, offs, srcs = [], [], [], [], []
    for q in range(world):
        for pc in plan.pieces[q]:
            views.append(outs[pc.layer][pc.lo:pc.hi])
            cnt.append(pc.hi - pc.lo)
            rr.append(rs[pc.layer])
            offs.append(pc.offset)
            srcs.append(q)
    lay = PackedLayout(tuple(cnt), tuple(rr), tuple(offs), plan.send_bytes)
    table = engine.SegmentTable(views, lay, sources=srcs)
    # the rotated walk (each rank starting before its own pieces) changes only the order
    for start in (-1, 0, 1, len(views) // 2, len(views) - 1, len(views) + 3):
        for o in outs:
            o.fill_(float("nan"))
        engine.unpack_multi(table, [b.data_ptr() for b in bufs], start_seg=start)
        torch.cuda.synchronize()
        for h, r, o in zip(hosts, rs, outs):
            assert np.array_equal(o.cpu().numpy().view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r))), start


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
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2004_02297_b200 as adt
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        if transport == "auto-ipcfail":           # rank 1 cannot map peer memory
            transport = "auto"
            if rank == 1:
                from paper_2004_02297_b200 import _lib, engine

                def refuse(handle):
                    raise _lib.AdtError(-1, "peer mapping refused (test)")
                engine.ipc_open = refuse
        counts = [20 * 25, 50 * 20 * 25, 3 * 4096 + 17, 10 * 500, 9 * 4096]
        if transport.endswith("-tiny"):          # one tile in all: the other ranks own nothing
            transport, counts = transport[:-5], [37]
        rng = np.random.default_rng(11)
        hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        masters = [torch.from_numpy(h.copy()).cuda() for h in hosts]
        cfg = adt.PrecisionConfig(threshold=-1e-3, interval=1, step_bits=8, initial_bits=8)
        chunks = 4
        if transport.startswith("nccl") and transport != "nccl":   # "nccl<k>": k gather chunks
            transport, chunks = "nccl", int(transport[4:])
        sync = ShardedWeightSync(masters, adt.PrecisionController(len(counts), cfg), transport=transport,
                                 nccl_chunks=chunks)
        ok, notes, norms_seen = True, [], []
        for step in range(4):
            res = sync.step(batch=step)
            torch.cuda.synchronize()
            for i, (h, r) in enumerate(zip(hosts, res.round_tos)):
                want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
                if not np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want):
                    ok = False
                    notes.append(f"step {step} layer {i} r={r} replica mismatch")
            for row in res.trace:
                ref = O.l2_norm(hosts[row[1]])
                if abs(row[2] - ref) > 1e-12 * ref:
                    ok = False
                    notes.append(f"norm {row}")
                norms_seen.append(row[2])
            # shrink every layer by 1% -> delta < threshold -> escalation each step (re-plan)
            for m, h in zip(masters, hosts):
                h *= np.float32(0.99)
                m.copy_(torch.from_numpy(h))
        if transport == "auto" and sync.transport != "nccl":
            ok = False
            notes.append(f"transport {sync.transport} after a failed peer mapping")
        q.put((rank, ok, notes, norms_seen, sync.round_tos))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface child failures to the parent
        q.put((rank, False, [repr(e)], [], []))


@pytest.mark.parametrize("transport", ["p2p", "nccl", "nccl1", "nccl7", "auto-ipcfail", "p2p-tiny", "nccl-tiny"])
def test_sync_two_processes_one_gpu(transport):
    """transport="nccl" runs its all-gather code path over gloo here (CUDA
    tensors; NCCL itself refuses two ranks on one device) in 4 chunks ("nccl1",
    "nccl7": 1 / 7 chunks, the unpack of each overlapping the next gather). "auto-ipcfail":
    one rank's peer mapping fails -> every rank falls back to the all-gather."""
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, transport)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, notes, _, _ in res:
        assert ok, (rank, notes[:5])
    assert res[0][3] == res[1][3] and len(res[0][3]) > 0   # identical norm bits on both ranks
    assert res[0][4] == res[1][4] and max(res[0][4]) > 1    # both escalated identically


def test_peer_barrier_two_virtual_ranks_and_timeout(adt):
    """adt_peer_barrier in one process: two 'ranks' on two streams meet (each
    publishes into the other's flag array and waits for both); a lone rank
    times out after its poll budget, records the epoch and returns."""
    from paper_2004_02297_b200 import engine
    flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    states = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    ptrs = [f.data_ptr() for f in flags]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(5):
        for r in (1, 0):
            engine.peer_barrier(ptrs, r, states[r], stream=streams[r])
    torch.cuda.synchronize()
    for r in range(2):
        assert states[r].tolist() == [5, 0]
        assert flags[r].tolist() == [5, 5]
    lone = torch.zeros(2, dtype=torch.int32, device="cuda")
    lone_flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    engine.peer_barrier([f.data_ptr() for f in lone_flags], 0, lone, timeout_s=0.05)
    torch.cuda.synchronize()
    assert lone.tolist() == [1, 1]             # epoch 1 published, and its wait timed out
    # the timeout word guards every peer-reading kernel queued behind it: none does any work
    from paper_2004_02297_b200.layout import PackedLayout
    lay = PackedLayout.plan([5000], [2])
    src = torch.randint(0, 255, (lay.nbytes,), dtype=torch.uint8, device="cuda")
    out = torch.full((5000,), 7.0, device="cuda")
    table = engine.SegmentTable([out], lay, sources=[0])
    engine.unpack_multi(table, [src.data_ptr()], abort=lone[1:2])
    dst = torch.zeros(64, dtype=torch.uint8, device="cuda")
    engine.copy_multi(dst, [src.data_ptr()], 0, 64, abort=lone[1:2])
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    engine.peer_barrier([f.data_ptr() for f in lone_flags], 0, lone, timeout_s=5.0)   # fails fast now
    t1.record()
    torch.cuda.synchronize()
    assert torch.all(out == 7.0) and torch.all(dst == 0)
    assert lone.tolist() == [2, 1] and t0.elapsed_time(t1) < 100.0
    engine.unpack_multi(table, [src.data_ptr()], abort=states[0][1:2])   # a clear word: the kernel runs
    torch.cuda.synchronize()
    assert not torch.all(out == 7.0)


def _stall_main(rank, world, port, q, stall, release, mode):
    """Two ranks step together, then rank 1 stalls (stops calling; stays alive).
    Rank 0 must raise PeerTimeout within one step, with replicas and masters
    left exactly as the last good step wrote them: mode "step" (the failing
    step returns, the next call raises) or "update" (the failing update raises
    itself: it reads the norms back)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2004_02297_b200.grads import GradBucket
        from paper_2004_02297_b200.precision import FixedPrecision
        from paper_2004_02297_b200.sharded import PeerTimeout, ShardedWeightSync
        counts = [500, 3 * 4096 + 17, 25000]
        rng = np.random.default_rng(5)
        hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
        masters = [torch.from_numpy(h.copy()).cuda() for h in hosts]

        class Mixed(FixedPrecision):
            def round_tos(self):
                return [1, 3, 2]

        sync = ShardedWeightSync(masters, Mixed(len(counts), 32), transport="p2p", barrier_timeout_s=1.0)
        bucket = GradBucket(counts, torch.device("cuda"))
        bucket.flat.normal_(0.0, 0.01)
        for b in range(3):
            sync.step(batch=b)
        sync.update(bucket, [64, 64], lr=0.1)     # maps the peers' gradient buckets (a collective)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 1:
            stall.set()
            release.wait(120)                 # alive (memory still mapped), but not stepping
            q.put((rank, True, [], None))
            return
        stall.wait(60)
        reps = [r.clone() for r in sync.replicas]
        before = [m.clone() for m in masters]
        notes, raised_at = [], None
        if mode == "step":
            for m in masters:
                m.mul_(2.0)                   # a completed step would change every replica
            before = [m.clone() for m in masters]
            for call in range(4):
                try:
                    sync.step(batch=3 + call)
                except PeerTimeout:
                    raised_at = call
                    break
            if raised_at != 1:
                notes.append(f"PeerTimeout at call {raised_at}, expected 1 (the call after the failed step)")
        else:
            try:
                sync.update(bucket, [64, 64], lr=0.1)
                notes.append("the update whose barrier timed out did not raise")
            except PeerTimeout:
                raised_at = 0
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(zip(reps, sync.replicas)):
            if not torch.equal(a, b):
                notes.append(f"replica {i} changed by the failed step")
        if any(not torch.equal(a, b) for a, b in zip(before, masters)):
            notes.append("masters stepped with stale gradients")
        for fn in (lambda: sync.step(batch=9), lambda: sync.update(bucket, [64, 64], lr=0.1)):
            try:
                fn()
                notes.append("a call after the timeout did not raise")
            except PeerTimeout:
                pass
        release.set()
        q.put((rank, not notes, notes, raised_at))
    except Exception as e:  # surface child failures to the parent
        release.set()
        q.put((rank, False, [repr(e)], None))


@pytest.mark.parametrize("mode", ["step", "update"])
def test_p2p_stalled_peer_raises_within_one_step(mode):
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    stall, release = ctx.Event(), ctx.Event()
    port = _free_port()
    procs = [ctx.Process(target=_stall_main, args=(r, 2, port, q, stall, release, mode)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, notes, _ in res:
        assert ok, (rank, notes)


def _graphed_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2004_02297_b200.precision import FixedPrecision
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        counts = [500, 3 * 4096 + 17, 25000]
        rng = np.random.default_rng(5)
        hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
        masters = [torch.from_numpy(h.copy()).cuda() for h in hosts]

        class Mixed(FixedPrecision):
            def round_tos(self):
                return [1, 3, 2]

        sync = ShardedWeightSync(masters, Mixed(len(counts), 32), transport="p2p")
        for _ in range(5):                      # both slots' graphs, replayed several times
            sync.launch_graphed(True)
        torch.cuda.synchronize()
        sync.check_barrier()
        ok = all(np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32),
                                h.view(np.uint32) & np.uint32(O.keep_mask(r)))
                 for i, (h, r) in enumerate(zip(hosts, [1, 3, 2])))
        norms = sync._norms()
        ok &= all(abs(n - O.l2_norm(h)) <= 1e-6 * O.l2_norm(h) for n, h in zip(norms, hosts))
        q.put((rank, ok, ""))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, traceback.format_exc()))


def test_p2p_graphed_step_two_processes_one_gpu():
    """ShardedWeightSync.launch_graphed: pack, device barrier, tail gather and
    gather-unpack captured in one CUDA graph per send slot."""
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_graphed_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, note in res:
        assert ok, (rank, note)


def _device_awp_main(rank, world, port, q, graphed):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2004_02297_b200 as adt
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        counts = [20 * 25, 50 * 20 * 25, 3 * 4096 + 17, 10 * 500, 9 * 4096]
        if world == 3:                           # some rank owns no piece
            counts = [37, 4100]
        L = len(counts)
        rng = np.random.default_rng(11)
        hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        masters = [torch.from_numpy(h.copy()).cuda() for h in hosts]
        kw = dict(threshold=-1e-3, interval=2, step_bits=8, initial_bits=8)
        octl = O.OracleController(L, **kw)
        sync = ShardedWeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**kw)), transport="p2p",
                                 awp_on_device=True, trace_ring=4)
        ok, notes, want = True, [], []
        for step in range(9):
            res = sync._step_device(step, step > 0, graphed=graphed)
            if step > 0:
                for i, h in enumerate(hosts):
                    octl.observe_layer(i, O.l2_norm(h))
                    want.append((step - 1, i, octl.bits[i]))
            torch.cuda.synchronize()
            rs = [octl.round_to(i) for i in range(L)] if step > 0 else [1] * L
            if sync.round_tos != rs:
                ok = False
                notes.append(f"step {step}: widths {sync.round_tos} != {rs}")
            for i, (h, r) in enumerate(zip(hosts, rs)):
                if not np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32),
                                      h.view(np.uint32) & np.uint32(O.keep_mask(r))):
                    ok = False
                    notes.append(f"step {step} layer {i} r={r} replica mismatch")
            for m, h in zip(masters, hosts):          # shrink 1%: delta < threshold -> escalations
                h *= np.float32(0.99)
                m.copy_(torch.from_numpy(h))
            del res
        rows = sync.drain_trace()
        if [(b, l, bits) for b, l, _, _, _, bits in rows] != want:
            ok = False
            notes.append(f"trace {rows[:3]} vs {want[:3]}")
        q.put((rank, ok, notes[:5], [r[2] for r in rows]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, False, [traceback.format_exc()], []))


@pytest.mark.parametrize("graphed,world", [(False, 2), (True, 2), (True, 8), (True, 3)])
def test_p2p_device_awp_processes_sharing_one_gpu(graphed, world):
    """ShardedWeightSync(p2p, awp_on_device): the decision on every rank's
    GPU from the gathered per-piece sums, escalated pieces re-packed by their
    owner and re-gathered by everyone — replicas, widths and trace rows vs the
    oracle, identical norms on both ranks."""
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_awp_main, args=(r, world, port, q, graphed)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    for rank, ok, notes, _ in res:
        assert ok, (rank, notes)
    assert all(r[3] == res[0][3] for r in res) and len(res[0][3]) > 0
