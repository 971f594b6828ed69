"""Property tests of the device codec, the reference's hypothesis laws
(test_codec.py:150-179) run against the sm_100a path with the oracle as the
checker: bytes identical to the scalar reference pack for any word pattern,
length and width; unpack(pack(x)) == x & truncation_mask(r) (mask law);
pack(unpack(pack(x))) == pack(x) (idempotence); len(payload) == n·r (size
law); output independent of worker_count."""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import weightpack_oracle as O

pytestmark = pytest.mark.gpu

words = st.integers(min_value=0, max_value=(1 << 32) - 1)


@pytest.fixture(scope="module")
def adt():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2004_02297_b200 as adt
    return adt


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(data=st.lists(words, max_size=300), r=st.integers(1, 4), workers=st.integers(1, 8))
def test_device_laws_on_arbitrary_words(adt, data, r, workers):
    x = np.array(data, dtype=np.uint32).view(np.float32)
    want = O.pack_scalar(x, r)
    dev = torch.from_numpy(x.copy()).cuda()
    blk = adt.pack_parallel(dev, r, workers)
    assert blk.weight_count == x.size and len(blk.payload_bytes()) == x.size * r
    assert blk.payload_bytes() == want
    back = adt.unpack(blk)
    got = back.cpu().numpy() if isinstance(back, torch.Tensor) else back
    assert np.array_equal(got.view(np.uint32), x.view(np.uint32) & np.uint32(O.keep_mask(r)))
    assert adt.pack_vectorized(back, r) == blk


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(n=st.integers(0, 3 * 4096 + 40), r=st.integers(1, 4), seed=st.integers(0, 2 ** 31))
def test_device_laws_across_tile_boundaries(adt, n, r, seed):
    x = np.random.default_rng(seed).integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32)
    blk = adt.pack(x, r)                      # host in -> host block, device kernels underneath
    assert blk.payload == O.pack_vectorized(x, r)
    assert np.array_equal(adt.unpack(blk).view(np.uint32), x.view(np.uint32) & np.uint32(O.keep_mask(r)))


@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(counts=st.lists(st.integers(0, 9000), min_size=1, max_size=12), seed=st.integers(0, 2 ** 31))
def test_multi_tensor_pack_unpack_norms(adt, counts, seed):
    rng = np.random.default_rng(seed)
    rs = [int(v) for v in rng.integers(1, 5, len(counts))]
    hosts = [(rng.standard_normal(n, dtype=np.float32) * np.float32(0.1)) for n in counts]
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    packed, lay, ss = adt.pack_many(devs, rs, with_norms=True)
    outs = adt.unpack_many(packed, lay)
    ss = ss.cpu().numpy()
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = lay.span(i)
        assert packed[lo:hi].cpu().numpy().tobytes() == O.pack_vectorized(h, r)
        assert np.array_equal(outs[i].cpu().numpy().view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r)))
        ref = O.l2_norm(h)
        assert abs(np.sqrt(ss[i]) - ref) <= 1e-6 * ref


@settings(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(counts=st.lists(st.integers(0, 20000), min_size=1, max_size=10), world=st.integers(1, 8),
       seed=st.integers(0, 2 ** 31))
def test_virtual_ranks_shard_pack_gather_unpack(adt, counts, world, seed):
    """Any layer set, widths and world size: every virtual rank packs its
    ShardPlan pieces (device kernel, norm tail fused) into its own send
    buffer; the rotated gather-unpack over all buffers rebuilds every replica
    as the reference would, and the rank-order norm combine matches."""
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    from paper_2004_02297_b200.sharded import ShardPlan
    rng = np.random.default_rng(seed)
    rs = [int(x) for x in rng.integers(1, 5, len(counts))]
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    plan = ShardPlan.plan(counts, rs, world)
    S = plan.send_bytes
    bufs = [torch.zeros(S, dtype=torch.uint8, device="cuda") for _ in range(world)]
    for q in range(world):
        mine = plan.pieces[q]
        if not mine:
            continue
        lay = PackedLayout(tuple(pc.hi - pc.lo for pc in mine), tuple(rs[pc.layer] for pc in mine),
                           tuple(pc.offset for pc in mine), plan.payload_cap)
        tail = bufs[q][plan.payload_cap:plan.payload_cap + 8 * plan.max_pieces].view(torch.float64)
        engine.pack(engine.SegmentTable([devs[pc.layer][pc.lo:pc.hi] for pc in mine], lay), bufs[q], tail)
    outs = [torch.full_like(d, float("nan")) for d in devs]
    views, cnt, rr, offs, srcs = [], [], [], [], []
    for q in range(world):
        for pc in plan.pieces[q]:
            views.append(outs[pc.layer][pc.lo:pc.hi])
            cnt.append(pc.hi - pc.lo)
            rr.append(rs[pc.layer])
            offs.append(pc.offset)
            srcs.append(q)
    if views:
        lay = PackedLayout(tuple(cnt), tuple(rr), tuple(offs), S)
        start = sum(len(plan.pieces[q]) for q in range(world // 2))
        engine.unpack_multi(engine.SegmentTable(views, lay, sources=srcs), [b.data_ptr() for b in bufs],
                            start_seg=start)
    torch.cuda.synchronize()
    for h, r, o in zip(hosts, rs, outs):
        assert np.array_equal(o.cpu().numpy().view(np.uint32), h.view(np.uint32) & np.uint32(O.keep_mask(r)))
    tails = [b[plan.payload_cap:plan.payload_cap + 8 * plan.max_pieces].view(torch.float64).cpu().tolist()
             for b in bufs]
    for h, s in zip(hosts, plan.combine_sumsq(tails)):
        ref = O.l2_norm(h) ** 2
        assert abs(s - ref) <= 1e-9 * max(ref, 1e-30)


# ------------------------------------------- full BASELINE sizes, size-independent laws
def _mask(r):
    return torch.tensor(O.keep_mask(r) - (1 << 32) if O.keep_mask(r) >= 1 << 31 else O.keep_mask(r),
                        dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("name,bits", [("alexnet", None), ("vgg16", 8), ("vgg16", 24), ("resnet50", 8),
                                       ("1b", 16), ("1b", 24)])
def test_full_size_sets_obey_the_laws(adt, name, bits):
    """BASELINE.json's configs at full size, checked on the device (the
    oracle is too slow there): for arbitrary 32-bit words the replicas equal
    words & truncation_mask(r) (mask law), re-packing the replicas gives the
    same bytes (idempotence), the payload is Σ n·r (size law); for N(0, 0.1²)
    weights the fused norms match a float64 torch reduction to 1e-9."""
    from paper_2004_02297_b200 import workloads
    counts = workloads.counts_of(name)
    rs = [(b + 7) // 8 for b in workloads.default_bits(name, bits)]
    g = torch.Generator(device="cuda").manual_seed(5)
    words = [torch.randint(-(1 << 31), 1 << 31, (n,), dtype=torch.int32, device="cuda", generator=g) for n in counts]
    packed, layout, _ = adt.pack_many([w.view(torch.float32) for w in words], rs)
    assert sum(hi - lo for lo, hi in (layout.span(i) for i in range(len(counts)))) == sum(
        n * r for n, r in zip(counts, rs))
    reps = adt.unpack_many(packed, layout)
    for w, rep, r in zip(words, reps, rs):
        assert torch.equal(rep.view(torch.int32), w & _mask(r))
    again, _, _ = adt.pack_many(reps, rs)
    for i in range(len(counts)):                 # payload spans (the 16-B alignment pad is not data)
        lo, hi = layout.span(i)
        assert torch.equal(again[lo:hi], packed[lo:hi]), i
    del words, reps, again, packed
    vals = [torch.randn(n, device="cuda", generator=g) * 0.1 for n in counts]
    _, _, ss = adt.pack_many(vals, rs, with_norms=True)
    ref = torch.stack([v.double().square().sum() for v in vals])
    assert torch.allclose(ss, ref, rtol=1e-9, atol=0.0)


@pytest.mark.parametrize("name,world", [("alexnet", 8), ("resnet50", 8), ("vgg16", 3)])
def test_full_size_virtual_ranks_gather_unpack(adt, name, world):
    """The sharded path at full size with every rank's send buffer on this
    GPU: each virtual rank packs its ShardPlan pieces with the norm tail
    fused, the rotated multi-source gather-unpack rebuilds every replica as
    words & mask, and the rank-order combine of the tails gives the layer
    norms (float64 torch reduction, 1e-9)."""
    from paper_2004_02297_b200 import engine, workloads
    from paper_2004_02297_b200.layout import PackedLayout
    from paper_2004_02297_b200.sharded import ShardPlan
    counts = workloads.counts_of(name)
    rs = [(b + 7) // 8 for b in workloads.default_bits(name)]
    g = torch.Generator(device="cuda").manual_seed(9)
    devs = [torch.randn(n, device="cuda", generator=g) * 0.1 for n in counts]
    plan = ShardPlan.plan(counts, rs, world)
    S = plan.send_bytes
    bufs = [torch.zeros(S, dtype=torch.uint8, device="cuda") for _ in range(world)]
    tails = []
    for q in range(world):
        mine = plan.pieces[q]
        tail = bufs[q][plan.payload_cap:plan.payload_cap + 8 * plan.max_pieces].view(torch.float64)
        tails.append(tail)
        if mine:
            lay = PackedLayout(tuple(pc.hi - pc.lo for pc in mine), tuple(rs[pc.layer] for pc in mine),
                               tuple(pc.offset for pc in mine), plan.payload_cap)
            engine.pack(engine.SegmentTable([devs[pc.layer][pc.lo:pc.hi] for pc in mine], lay), bufs[q], tail)
    outs = [torch.full_like(d, float("nan")) for d in devs]
    views, cnt, rr, offs, srcs = [], [], [], [], []
    for q in range(world):
        for pc in plan.pieces[q]:
            views.append(outs[pc.layer][pc.lo:pc.hi])
            cnt.append(pc.hi - pc.lo)
            rr.append(rs[pc.layer])
            offs.append(pc.offset)
            srcs.append(q)
    start = sum(len(plan.pieces[q]) for q in range(world // 2))
    engine.unpack_multi(engine.SegmentTable(views, PackedLayout(tuple(cnt), tuple(rr), tuple(offs), S), sources=srcs),
                        [b.data_ptr() for b in bufs], start_seg=start)
    for d, o, r in zip(devs, outs, rs):
        assert torch.equal(o.view(torch.int32), d.view(torch.int32) & _mask(r))
    sums = plan.combine_sumsq([t.cpu().tolist() for t in tails])
    ref = torch.stack([d.double().square().sum() for d in devs]).cpu()
    assert torch.allclose(torch.tensor(sums, dtype=torch.float64), ref, rtol=1e-9, atol=0.0)
