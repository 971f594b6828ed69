"""GPU parity: the sm_100a path vs the reference's golden vectors and the oracle.

Bar (BASELINE.json north_star): packed bytes and unpacked words bit-exact,
AWP widths identical, norms within 1e-6 relative (the reference's summation
order lives in OpenBLAS ddot and is not pinned; ours is fixed, so we also
assert run-to-run bit identity).
"""

import hashlib
import io
import math

import numpy as np
import pytest
import torch

from oracle import weightpack_oracle as O

pytestmark = pytest.mark.gpu

NORM_RTOL = 1e-6


@pytest.fixture(scope="module")
def adt():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2004_02297_b200 as adt
    return adt


def test_library_is_the_in_tree_build(adt):
    from paper_2004_02297_b200 import _lib
    lib = _lib.load()
    assert lib._name.endswith("paper_2004_02297_b200/libadt.so")
    from paper_2004_02297_b200 import engine
    assert engine.sm_count() >= 100


# ------------------------------------------------- golden (reference-run) vectors
def test_pack_matches_golden(adt, golden_codec):
    for c in golden_codec:
        x = c["words"].view(np.float32)
        want = c["payload"].tobytes()
        for fn in (lambda: adt.pack(x, c["r"]), lambda: adt.pack_vectorized(x, c["r"]),
                   lambda: adt.pack_parallel(x, c["r"], 3)):
            blk = fn()
            assert blk.payload == want, c["name"]
            assert blk.weight_count == c["words"].size


def test_unpack_matches_golden(adt, golden_codec):
    for c in golden_codec:
        blk = adt.PackedBlock(c["r"], c["words"].size, c["payload"].tobytes())
        got = adt.unpack(blk)
        assert isinstance(got, np.ndarray) and got.dtype == np.float32 and got.flags.writeable
        assert np.array_equal(got.view(np.uint32), c["unpacked"]), c["name"]


def test_device_payload_path(adt, golden_codec):
    for c in golden_codec[::7]:
        t = torch.from_numpy(c["words"].astype(np.uint32).view(np.float32).copy()).cuda()
        blk = adt.pack(t, c["r"])
        assert blk.on_device
        assert blk.payload_bytes() == c["payload"].tobytes()
        out = adt.unpack(blk)
        assert out.is_cuda
        assert np.array_equal(out.cpu().numpy().view(np.uint32), c["unpacked"])


def test_reference_kats(adt):
    # test_codec.py:66-147
    assert adt.pack([1.0], 3).payload == bytes([0x3F, 0x80, 0x00])
    assert adt.pack([-2.0], 1).payload == bytes([0xC0])
    assert adt.pack([np.float32(3.14159274)], 2).payload == bytes([0x40, 0x49])
    m = np.array([0x11223344, 0x55667788, 0x99AABBCC, 0xDDEEFF00], np.uint32).view(np.float32).reshape(2, 2)
    assert adt.pack(m, 1).payload == bytes([0x11, 0x55, 0x99, 0xDD])
    assert adt.unpack(adt.PackedBlock(1, 1, bytes([0x3F]))).tolist() == [0.5]
    assert adt.unpack(adt.PackedBlock(2, 1, bytes([0x40, 0x49]))).tolist() == [3.140625]
    snan = np.array([0x7F800001], np.uint32).view(np.float32)
    assert adt.unpack(adt.pack(snan, 3)).tolist() == [float("inf")]
    e = adt.pack([], 2)
    assert e.payload == b"" and e.weight_count == 0
    assert adt.unpack(e).size == 0


def test_errors_map_to_reference_types(adt):
    for bad in (0, 5, 2.5):
        with pytest.raises(ValueError):
            adt.pack([1.0], bad)
    with pytest.raises(ValueError):
        adt.pack_parallel([1.0], 2, 0)
    with pytest.raises(adt.MalformedBlock):
        adt.PackedBlock(2, 3, bytes(5))


def test_transposed_and_float64_inputs_follow_reference_cast(adt):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((33, 17))
    for x in (a, a.T, a.astype(np.float32).T):
        for r in (1, 3, 4):
            assert adt.pack(x, r).payload == O.pack_scalar(x, r)


# ------------------------------------------------------------- laws at scale
@pytest.mark.parametrize("r", [1, 2, 3, 4])
def test_mask_law_and_idempotence_1e6(adt, r):
    """test_acceptance.py:71-83 (criterion 1) and test_codec.py:163-171, on device."""
    rng = np.random.default_rng(7)
    words = np.concatenate([rng.integers(0, 1 << 32, 10**6, dtype=np.uint32),
                            np.array(O.SPECIAL_WORDS, np.uint32)])
    t = torch.from_numpy(words.view(np.float32).copy()).cuda()
    blk = adt.pack(t, r)
    assert blk.payload_bytes() == O.pack_vectorized(words.view(np.float32), r)
    back = adt.unpack(blk)
    want = torch.from_numpy((words & np.uint32(O.keep_mask(r))).view(np.int32).copy()).cuda()
    assert torch.equal(back.view(torch.int32), want)
    assert adt.pack(back, r) == blk


LENGTHS = [0, 1, 3, 4, 5, 15, 16, 17, 4095, 4096, 4097, 8191, 8193, 12289, 65537, 100003]


def test_multi_tensor_ragged_mixed_widths(adt):
    rng = np.random.default_rng(11)
    hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in LENGTHS]
    rs = [(i % 4) + 1 for i in range(len(hosts))]
    devs = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    packed, layout, ss = adt.pack_many(devs, rs, with_norms=True)
    assert all(o % 16 == 0 for o in layout.offsets)
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = layout.span(i)
        assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(h, r), (i, LENGTHS[i], r)
    outs = adt.unpack_many(packed, layout)
    for h, r, o in zip(hosts, rs, outs):
        assert np.array_equal(o.cpu().numpy().view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r)))
    blocks = adt.blocks_of(packed, layout)
    assert [b.weight_count for b in blocks] == LENGTHS


def test_multi_tensor_beyond_one_launch_table(adt):
    """> 256 layers forces several launches; results must not change."""
    rng = np.random.default_rng(5)
    counts = [int(c) for c in rng.integers(0, 9000, 300)]
    hosts = [(rng.standard_normal(n, dtype=np.float32) * np.float32(0.1)) for n in counts]
    rs = [int(x) for x in rng.integers(1, 5, len(counts))]
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    packed, layout, ss = adt.pack_many(devs, rs, with_norms=True)
    ss = ss.cpu().numpy()
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = layout.span(i)
        assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(h, r)
        assert ss[i] == pytest.approx(O.sumsq(h), rel=1e-12, abs=0)


# -------------------------------------------------------------------- norms
def test_norms_match_golden(adt, golden_norms):
    for x, want in golden_norms:
        got = adt.l2_norm(x)
        if want == 0.0:
            assert got == 0.0
        else:
            assert abs(got - want) <= NORM_RTOL * want


def test_fused_norm_bit_identical_across_runs_and_widths(adt):
    rng = np.random.default_rng(0)
    hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in (1000, 4096 * 37 + 5, 1 << 20)]
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    runs = []
    for rs in ([1, 2, 3], [4, 4, 4], [3, 1, 2]):
        _, _, ss = adt.pack_many(devs, rs, with_norms=True)
        runs.append(ss.cpu().numpy().tobytes())
    assert len(set(runs)) == 1
    ss = np.frombuffer(runs[0], np.float64)
    for h, s in zip(hosts, ss):
        assert math.sqrt(s) == pytest.approx(O.l2_norm(h), rel=1e-12)


# ---------------------------------------------------------------- container
def test_container_roundtrip_device_block(adt):
    t = torch.randn(1001, device="cuda")
    blk = adt.pack(t, 3)
    buf = io.BytesIO()
    n = adt.write_stream(buf, blk)
    assert n == 14 + 3003
    buf.seek(0)
    back = adt.read_stream(buf)
    assert back == blk
    assert buf.getvalue() == O.write_container(3, 1001, O.pack_vectorized(t.cpu().numpy(), 3))


# --------------------------------------------------------- pinned zero-copy
def test_unpack_from_pinned_host(adt):
    from paper_2004_02297_b200 import engine
    rng = np.random.default_rng(2)
    counts, rs = [5000, 4096, 77], [2, 3, 1]
    hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in counts]
    layout = adt.PackedLayout.plan(counts, rs)
    buf = np.zeros(layout.nbytes, np.uint8)
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = layout.span(i)
        buf[lo:hi] = np.frombuffer(O.pack_vectorized(h, r), np.uint8)
    pinned = torch.from_numpy(buf).pin_memory()
    outs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in counts]
    engine.unpack(engine.SegmentTable(outs, layout), pinned)
    torch.cuda.synchronize()
    for h, r, o in zip(hosts, rs, outs):
        assert np.array_equal(o.cpu().numpy().view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r)))


# ------------------------------------------------------- AWP flow (config 1)
def test_lenet_awp_walk_matches_reference(adt, golden_lenet):
    """200 batches of the seeded LeNet walk through
    WeightSync (fused norms, repack on escalation) vs the reference's run."""
    steps = int(golden_lenet["steps"])
    walk = list(O.lenet_walk(steps, seed=7))
    L = len(walk[0][1])
    cfg = adt.PrecisionConfig(threshold=-2e-3, interval=int(golden_lenet["interval"]), step_bits=8, initial_bits=8)
    ctl = adt.PrecisionController(L, cfg)
    masters = [torch.from_numpy(w.copy()).cuda() for w in walk[0][1]]
    sync = adt.WeightSync(masters, ctl)
    trace = []
    for t in range(steps):
        for m, w in zip(masters, walk[t][1]):
            m.copy_(torch.from_numpy(w))
        res = sync.step(batch=t)
        trace += res.trace
        assert res.round_tos == list(golden_lenet["widths"][t]), t
        lo_hi = [sync.layout.span(i) for i in range(L)]
        host_packed = sync.packed.cpu().numpy()
        for i in range(L):
            pay = host_packed[lo_hi[i][0]:lo_hi[i][1]].tobytes()
            assert hashlib.sha256(pay).digest() == golden_lenet["payload_sha"][t, i].tobytes(), (t, i)
            rep = sync.replicas[i].cpu().numpy()
            assert hashlib.sha256(rep.tobytes()).digest() == golden_lenet["unpacked_sha"][t, i].tobytes(), (t, i)
    for m, w in zip(masters, walk[steps][1]):
        m.copy_(torch.from_numpy(w))
    trace += sync.observe_final(batch=steps - 1)
    assert len(trace) == steps * L
    for k, (b, layer, norm, delta, counter, bits) in enumerate(trace):
        t, i = divmod(k, L)
        assert (b, layer) == (t, i)
        assert bits == golden_lenet["bits"][t, i] and counter == golden_lenet["counter"][t, i], (t, i)
        assert abs(norm - golden_lenet["norms"][t, i]) <= NORM_RTOL * golden_lenet["norms"][t, i]
        gd = golden_lenet["delta"][t, i]
        assert (delta is None and math.isnan(gd)) or abs(delta - gd) <= 1e-6 * max(abs(gd), 1e-3)



def test_graphed_step_matches_eager(adt):
    """WeightSync.launch_graphed (two CUDA graphs, finalize on a side branch)
    == eager launch: same packed bytes, replicas and norm bits."""
    g = torch.Generator(device="cuda").manual_seed(3)
    masters = [torch.randn(n, generator=g, device="cuda") * 0.1 for n in (64, 4096 * 5 + 3, 1 << 18, 10)]
    sched = adt.FixedPrecision(len(masters), 24)
    a = adt.WeightSync(masters, sched)
    a.launch(fused_norm=True)
    eager = (a.packed.clone(), [r.clone() for r in a.replicas], a.read_norms())
    b = adt.WeightSync(masters, sched)
    for _ in range(3):
        b.launch_graphed(fused_norm=True)
    torch.cuda.synchronize()
    for i in range(len(masters)):  # payload spans (the inter-layer pad is never written)
        lo, hi = a.layout.span(i)
        assert torch.equal(b.packed[lo:hi], eager[0][lo:hi])
    assert all(torch.equal(x, y) for x, y in zip(b.replicas, eager[1]))
    assert b.read_norms() == eager[2]


# ------------------------------------------- fused SGD + pack
def test_sgd_pack_matches_reference_update(adt, golden_sgd):
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    for i, c in enumerate(golden_sgd):
        r = (i % 4) + 1
        w = torch.from_numpy(c["w"].reshape(-1).copy()).cuda()
        v = torch.from_numpy(c["v"].reshape(-1).copy()).cuda()
        g = torch.from_numpy(c["g"].reshape(-1).copy()).cuda()
        lay = PackedLayout.plan([w.numel()], [r])
        packed = torch.zeros(lay.nbytes, dtype=torch.uint8, device="cuda")
        ss = torch.empty(1, dtype=torch.float64, device="cuda")
        engine.sgd_pack(engine.SgdTable([w], [v], [g], lay), *c["hp"], packed, ss)
        torch.cuda.synchronize()
        w1 = c["w1"].reshape(-1)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), w1.view(np.uint32)), i
        assert np.array_equal(v.cpu().numpy().view(np.uint32), c["v1"].reshape(-1).view(np.uint32)), i
        lo, hi = lay.span(0)
        assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(w1, r), i
        assert math.sqrt(float(ss.item())) == pytest.approx(O.l2_norm(w1), rel=1e-12)


def test_weightsync_update_walk_matches_reference_order(adt):
    """30 batches of momentum SGD with AWP through WeightSync.update (fused
    update + pack + norm, repack on escalation) vs the oracle in the
    reference's order: update -> norm -> observe -> pack at the new widths."""
    rng = np.random.default_rng(21)
    counts = [500, 25000, 4096 * 3 + 7, 5000]
    L = len(counts)
    hp = (0.05, 0.9, 5e-4)
    w_ref = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    v_ref = [np.zeros(n, np.float32) for n in counts]
    noise = [[rng.standard_normal(n, dtype=np.float32) * np.float32(0.002) for n in counts] for _ in range(30)]
    kw = dict(threshold=-2e-3, interval=3, step_bits=8, initial_bits=8)
    octl = O.OracleController(L, **kw)
    masters = [torch.from_numpy(w.copy()).cuda() for w in w_ref]
    sync = adt.WeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**kw)))
    sync.step(batch=0)
    for b in range(30):
        # gradients pulling the weights toward zero (weight-decay-like): the norms shrink -> AWP escalates
        grads = [np.float32(0.4) * w + noise[b][i] for i, w in enumerate(w_ref)]
        res = sync.update([torch.from_numpy(x).cuda() for x in grads], *hp, batch=b)
        for i in range(L):
            w_ref[i], v_ref[i] = O.sgd_step(w_ref[i], v_ref[i], grads[i], *hp)
        for i in range(L):
            octl.observe_layer(i, O.l2_norm(w_ref[i]))
        rs = [octl.round_to(i) for i in range(L)]
        assert res.round_tos == rs, b
        for i in range(L):
            assert np.array_equal(masters[i].cpu().numpy().view(np.uint32), w_ref[i].view(np.uint32)), (b, i)
            lo, hi = sync.layout.span(i)
            assert sync.packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(w_ref[i], rs[i]), (b, i)
            want = w_ref[i].view(np.uint32) & np.uint32(O.keep_mask(rs[i]))
            assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), (b, i)
        assert [row[5] for row in res.trace] == [octl.bits[i] for i in range(L)]
    assert max(sync.round_tos) > 1  # the walk exercised escalation


def test_single_layer_beyond_4gb_packed_offsets(adt):
    """A 1.5e9-weight layer at r = 3: payload offsets pass 4 GiB (64-bit tile
    addressing). Spot windows against the oracle; the mask law over all of it."""
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    n, r = 1_500_000_003, 3
    free, _ = torch.cuda.mem_get_info()
    if free < 24 * (1 << 30):
        pytest.skip("needs ~18 GB of free HBM")
    g = torch.Generator(device="cuda").manual_seed(9)
    bits = torch.randint(-(1 << 31), 1 << 31, (n,), dtype=torch.int32, device="cuda", generator=g)
    w = bits.view(torch.float32)
    lay = PackedLayout.plan([n], [r])
    packed = torch.empty(lay.nbytes, dtype=torch.uint8, device="cuda")
    engine.pack(engine.SegmentTable([w], lay), packed)
    out = torch.empty_like(w)
    engine.unpack(engine.SegmentTable([out], lay), packed)
    torch.cuda.synchronize()
    mask = torch.tensor(O.keep_mask(r) - (1 << 32), dtype=torch.int32, device="cuda")
    assert torch.equal(out.view(torch.int32), bits & mask)
    for start in (0, 4095, 1_431_655_760, n - 4100):   # 3*start crosses 2^32 at the third window
        hw = w[start:start + 4100].cpu().numpy()
        assert packed[3 * start:3 * (start + 4100)].cpu().numpy().tobytes() == O.pack_vectorized(hw, r)
    del bits, w, out, packed
    torch.cuda.empty_cache()


def test_concurrent_host_threads_on_separate_streams(adt):
    """include/adt.h: callable from several host threads on different streams
    (no hidden mutable state; per-stream norm scratch)."""
    import threading
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    rng = np.random.default_rng(31)
    jobs = []
    for t in range(4):
        counts = [int(x) for x in rng.integers(1, 20000, 6)]
        rs = [int(x) for x in rng.integers(1, 5, 6)]
        hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
        jobs.append((counts, rs, hosts))
    results, errors = [None] * len(jobs), []

    def work(i):
        try:
            counts, rs, hosts = jobs[i]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                devs = [torch.from_numpy(h).cuda(non_blocking=False) for h in hosts]
                lay = PackedLayout.plan(counts, rs)
                packed = torch.empty(lay.nbytes, dtype=torch.uint8, device="cuda")
                ss = torch.empty(len(counts), dtype=torch.float64, device="cuda")
                outs = [torch.empty_like(d) for d in devs]
                for _ in range(20):
                    engine.pack(engine.SegmentTable(devs, lay), packed, ss, s)
                    engine.unpack(engine.SegmentTable(outs, lay), packed, s)
                s.synchronize()
                results[i] = (packed.cpu().numpy(), [o.cpu().numpy() for o in outs], ss.cpu().numpy(), lay)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for (counts, rs, hosts), (packed, outs, ss, lay) in zip(jobs, results):
        for l, (h, r) in enumerate(zip(hosts, rs)):
            lo, hi = lay.span(l)
            assert packed[lo:hi].tobytes() == O.pack_vectorized(h, r)
            assert np.array_equal(outs[l].view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r)))
            assert math.sqrt(ss[l]) == pytest.approx(O.l2_norm(h), rel=NORM_RTOL)


def test_l2_norm_many_matches_per_layer_and_golden(adt, golden_norms):
    xs = [x for x, _ in golden_norms]
    got = adt.l2_norm_many(xs)
    for (x, want), g in zip(golden_norms, got):
        assert g == adt.l2_norm(x)
        assert g == pytest.approx(want, rel=NORM_RTOL, abs=0.0) if want else g == 0.0
    devs = [torch.from_numpy(np.asarray(x, np.float32)).cuda() for x in xs]
    assert adt.l2_norm_many(devs) == got


@pytest.mark.parametrize("graphed", [True, False])
def test_lenet_awp_walk_device_controller(adt, golden_lenet, graphed):
    """The same 200-batch LeNet walk with the AWP decision on the device
    (WeightSync(awp_on_device=True): one graph per step, no host read per
    step): identical widths, payloads, replicas and trace rows, read back in
    batches (a 16-step trace ring forces several automatic drains)."""
    steps = int(golden_lenet["steps"])
    walk = list(O.lenet_walk(steps, seed=7))
    L = len(walk[0][1])
    cfg = adt.PrecisionConfig(threshold=-2e-3, interval=int(golden_lenet["interval"]), step_bits=8, initial_bits=8)
    masters = [torch.from_numpy(w.copy()).cuda() for w in walk[0][1]]
    sync = adt.WeightSync(masters, adt.PrecisionController(L, cfg), awp_on_device=True, trace_ring=16,
                          graphed=graphed)
    cap = sync.capacity_layout
    for t in range(steps):
        for m, w in zip(masters, walk[t][1]):
            m.copy_(torch.from_numpy(w))
        sync.step(batch=t)
        if t % 7 == 0 or t == steps - 1:          # inspect some steps (each inspection synchronises)
            rs = sync.round_tos
            assert rs == list(golden_lenet["widths"][t]), t
            host_packed = sync.packed.cpu().numpy()
            for i in range(L):
                lo = cap.offsets[i]
                pay = host_packed[lo:lo + cap.counts[i] * rs[i]].tobytes()
                assert hashlib.sha256(pay).digest() == golden_lenet["payload_sha"][t, i].tobytes(), (t, i)
                rep = sync.replicas[i].cpu().numpy()
                assert hashlib.sha256(rep.tobytes()).digest() == golden_lenet["unpacked_sha"][t, i].tobytes(), (t, i)
    trace = sync.drain_trace()
    for m, w in zip(masters, walk[steps][1]):
        m.copy_(torch.from_numpy(w))
    trace += sync.observe_final(batch=steps - 1)
    assert len(trace) == steps * L
    for k, (b, layer, norm, delta, counter, bits) in enumerate(trace):
        t, i = divmod(k, L)
        assert (b, layer) == (t, i)
        assert bits == golden_lenet["bits"][t, i] and counter == golden_lenet["counter"][t, i], (t, i)
        assert abs(norm - golden_lenet["norms"][t, i]) <= NORM_RTOL * golden_lenet["norms"][t, i]
        gd = golden_lenet["delta"][t, i]
        assert (delta is None and math.isnan(gd)) or abs(delta - gd) <= 1e-6 * max(abs(gd), 1e-3)
    # the host controller mirrors the device state after the drain
    assert sync.schedule.round_tos() == sync.round_tos


def test_device_controller_groups_match_host_controller(adt):
    """Grouped layers (shared state, observed in layer order) and consecutive
    mode: device decisions and trace rows equal the host controller's bit for bit."""
    rng = np.random.default_rng(12)
    counts = [4096 + 3, 700, 9000, 50, 4096 * 2]
    groups = [0, 0, 1, 2, 1]
    kw = dict(threshold=-1e-3, interval=2, step_bits=6, initial_bits=8, max_bits=24, consecutive=True)
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    ma = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    mb = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    host_sync = adt.WeightSync(ma, adt.PrecisionController(len(counts), adt.PrecisionConfig(**kw), groups))
    dev_sync = adt.WeightSync(mb, adt.PrecisionController(len(counts), adt.PrecisionConfig(**kw), groups),
                              awp_on_device=True)
    want = []
    for t in range(40):
        f = (1.0 + rng.uniform(-0.004, 0.002, len(counts))).astype(np.float32)
        for i, (a, b) in enumerate(zip(ma, mb)):
            a.mul_(float(f[i]))
            b.mul_(float(f[i]))
        want += host_sync.step(batch=t).trace
        dev_sync.step(batch=t)
        if t % 10 == 9:
            assert dev_sync.round_tos == host_sync.round_tos, t
            for x, y in zip(host_sync.replicas, dev_sync.replicas):
                assert torch.equal(x, y), t
    got = dev_sync.drain_trace()
    assert got == want
    assert max(host_sync.round_tos) > 1


def test_device_controller_beyond_one_launch_table(adt):
    """300 layers (two launch chunks for every dyn kernel and the fixup) with
    escalations every other step: device AWP equals the host controller."""
    rng = np.random.default_rng(13)
    counts = [int(x) for x in rng.integers(1, 3000, 300)]
    kw = dict(threshold=-5e-4, interval=2, step_bits=8, initial_bits=8)
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    ma = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    mb = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    host_sync = adt.WeightSync(ma, adt.PrecisionController(len(counts), adt.PrecisionConfig(**kw)))
    dev_sync = adt.WeightSync(mb, adt.PrecisionController(len(counts), adt.PrecisionConfig(**kw)), awp_on_device=True)
    want = []
    for t in range(7):
        f = (1.0 - rng.uniform(0.0, 0.002, len(counts))).astype(np.float32)
        for i, (a, b) in enumerate(zip(ma, mb)):
            a.mul_(float(f[i]))
            b.mul_(float(f[i]))
        want += host_sync.step(batch=t).trace
        dev_sync.step(batch=t)
    assert dev_sync.drain_trace() == want
    assert dev_sync.round_tos == host_sync.round_tos and max(host_sync.round_tos) > 1
    for x, y in zip(host_sync.replicas, dev_sync.replicas):
        assert torch.equal(x, y)


def test_host_staging_chunks_and_round_trips(adt):
    """hostio: sizes across the small-copy threshold and several 64 MiB staging
    chunks (odd tails), both directions, then the drop-in host API on a
    multi-chunk layer against the C oracle."""
    from oracle import c_oracle as C
    from paper_2004_02297_b200 import hostio
    rng = np.random.default_rng(41)
    for nbytes in (17, (1 << 20) + 3, 3 * hostio.CHUNK + 12345):
        x = rng.integers(0, 256, nbytes, dtype=np.uint8)
        d = hostio.to_device(x)
        assert torch.equal(d.cpu(), torch.from_numpy(x))
        assert hostio.to_bytes(d) == x.tobytes()
    f = rng.standard_normal(2 * hostio.CHUNK // 4 + 777, dtype=np.float32)
    assert np.array_equal(hostio.to_numpy_f32(hostio.to_device(f)), f)
    w = rng.integers(0, 1 << 32, 40_000_003, dtype=np.uint32).view(np.float32)
    for r in (1, 3, 4):
        blk = adt.pack_vectorized(w, r)
        assert blk.payload == C.pack(w, r)
        back = adt.unpack(blk)
        assert back.flags.writeable and np.array_equal(back.view(np.uint32), w.view(np.uint32) & np.uint32(O.keep_mask(r)))


def test_measured_profile_shape(adt):
    """transfer.measured_profile: the reference's profile_report phases with
    measured device times (the Table-2 rows) — every phase present, positive,
    and the weight-stream byte ratio equal to the reference ledger arithmetic."""
    from paper_2004_02297_b200 import transfer
    rng = np.random.default_rng(3)
    counts = [20 * 25, 50 * 20 * 25, 500 * 800, 10 * 500]
    masters = [torch.from_numpy(rng.standard_normal(n, dtype=np.float32)).cuda() for n in counts]

    class W(adt.FixedPrecision):
        def round_tos(self):
            return [1, 2, 3, 4]

    sync = adt.WeightSync(masters, W(len(counts), 32))
    prof = transfer.measured_profile(sync)
    ph = prof["phases"]
    for key in ("pack", "unpack", "l2_norm", "to_worker"):
        assert key in ph
    assert ph["pack"]["device_s"] > 0 and ph["unpack"]["device_s"] > 0
    assert ph["to_worker"]["raw_fp32_h2d_s"] > ph["to_worker"]["packed_h2d_s"] > 0
    raw = sum(4 * n for n in counts)
    wire = sum(14 + n * r for n, r in zip(counts, [1, 2, 3, 4]))
    assert prof["weight_stream"]["raw_bytes"] == raw and prof["weight_stream"]["wire_bytes"] == wire
    assert prof["weight_stream"]["ratio"] == pytest.approx(raw / wire)


def test_trace_csv_byte_identical_across_reruns(adt):
    """test_acceptance.py:206-215: a rerun writes a byte-identical trace.csv
    (fixed-order reductions, no float atomics) — host and device AWP alike."""
    import io
    walk = list(O.lenet_walk(40, seed=11))
    L = len(walk[0][1])
    cfg = dict(threshold=-2e-3, interval=3, step_bits=8, initial_bits=8)

    def run(on_device):
        masters = [torch.from_numpy(w.copy()).cuda() for w in walk[0][1]]
        sync = adt.WeightSync(masters, adt.PrecisionController(L, adt.PrecisionConfig(**cfg)), awp_on_device=on_device)
        rows = []
        for t in range(40):
            for m, w in zip(masters, walk[t][1]):
                m.copy_(torch.from_numpy(w))
            rows += sync.step(batch=t).trace
        rows += sync.drain_trace() if on_device else []
        buf = io.StringIO()
        adt.write_trace_csv(buf, rows)
        return buf.getvalue()

    a, b, c = run(False), run(False), run(True)
    assert a == b == c and len(a.splitlines()) == 1 + 39 * L


def test_l2_norm_any_array_like_float64(adt):
    """precision.py:25-28 takes ANY array-like (np.asarray(float64)): float64,
    float16 and integer inputs go through the float64-input kernel and match
    the reference's float64 norm to 1e-12; float32 stays on the exact path."""
    rng = np.random.default_rng(12)
    x64 = rng.standard_normal(10 ** 6)
    ref = O.l2_norm(x64)
    assert abs(adt.l2_norm(x64) - ref) <= 1e-12 * ref
    assert abs(adt.l2_norm(torch.from_numpy(x64).cuda()) - ref) <= 1e-12 * ref
    assert abs(adt.l2_norm(x64.tolist()[:1000]) - O.l2_norm(x64[:1000])) <= 1e-12 * O.l2_norm(x64[:1000])
    ints = rng.integers(-1000, 1000, 12345)
    assert abs(adt.l2_norm(ints) - O.l2_norm(ints)) <= 1e-12 * O.l2_norm(ints)
    h = rng.standard_normal(5000).astype(np.float16)
    assert abs(adt.l2_norm(h) - O.l2_norm(h)) <= 1e-12 * O.l2_norm(h)
    assert adt.l2_norm(np.zeros(0)) == 0.0 and adt.l2_norm([3.0, 4.0]) == 5.0
    assert math.isnan(adt.l2_norm(np.array([1.0, np.nan])))
    big = rng.standard_normal(3 * 10 ** 7)               # many CTAs: fixed order, bit-identical reruns
    a, b = adt.l2_norm(big), adt.l2_norm(big)
    assert a == b and abs(a - O.l2_norm(big)) <= 1e-12 * a
    many = adt.l2_norm_many([x64, x64.astype(np.float32), ints])
    assert many[0] == adt.l2_norm(x64) and many[2] == adt.l2_norm(ints)
    assert abs(many[1] - O.l2_norm(x64.astype(np.float32))) <= 1e-12 * many[1]


def test_one_launch_small_step_matches_three_launch_step(adt):
    """adt_roundtrip (pack + norms, grid barrier, unpack, per-layer sums in one
    cooperative launch) gives the same packed bytes, replicas and bit-identical
    norms as pack -> finalize -> unpack, across many graph replays (the grid
    barrier is reused launch after launch), up to the one-tile-per-SM limit."""
    from paper_2004_02297_b200 import engine
    rng = np.random.default_rng(21)
    limit = engine.roundtrip_max_tiles()
    for counts, rs in (([20 * 25, 50 * 20 * 25, 500 * 800, 10 * 500], [1, 2, 3, 4]),
                       ([4096 * (limit - 2), 5000, 3], [3, 1, 2]),
                       ([4096 * limit + 1], [2])):          # one tile over the limit: the 3-launch step
        hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
        outs = []
        for fuse in (True, False):
            class Fixed(adt.FixedPrecision):
                def round_tos(self):
                    return list(rs)
            sync = adt.WeightSync([torch.from_numpy(h.copy()).cuda() for h in hosts], Fixed(len(counts), 32),
                                  fuse_small=fuse)
            for _ in range(300):
                sync.launch_graphed(fused_norm=True)
            norms = sync.read_norms()
            torch.cuda.synchronize()
            outs.append((sync._small, sync.packed[:sync.layout.nbytes].cpu().numpy(),
                         [r.cpu().numpy().view(np.uint32) for r in sync.replicas], norms, sync.layout))
        (small, pk_a, rep_a, n_a, lay), (_, pk_b, rep_b, n_b, _) = outs
        assert small == (sum((n + 4095) // 4096 for n in counts) <= limit)
        for i, (h, r) in enumerate(zip(hosts, rs)):
            lo, hi = lay.span(i)
            assert pk_a[lo:hi].tobytes() == pk_b[lo:hi].tobytes() == O.pack_vectorized(h, r)
            assert np.array_equal(rep_a[i], h.view(np.uint32) & np.uint32(O.keep_mask(r)))
            assert np.array_equal(rep_a[i], rep_b[i])
        assert n_a == n_b                                       # same fixed summation order
        for h, n in zip(hosts, n_a):
            assert abs(n - O.l2_norm(h)) <= 1e-6 * O.l2_norm(h)
