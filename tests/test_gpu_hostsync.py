"""The CPU-master path end to end on a B200 (the paper's setting,
PAPER.md:219-229): host FP32 masters -> adt_pack_host on the host cores ->
packed stream over PCIe while the rest is packed -> adt_unpack on the GPU.
Replicas must equal the reference's unpack(pack(W)) bit for bit, norms its
l2_norm, and the AWP walk must take the reference run's decisions."""

import hashlib
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


@pytest.mark.parametrize("ring,zero_copy", [(0, False), (0, True), (48 * (384 << 10), False)])
def test_replicas_and_norms_mixed_widths(adt, ring, zero_copy):
    rng = np.random.default_rng(3)
    counts = [20 * 25, 50 * 20 * 25, 4097, 0, 65536 * 3 + 11, 10 * 500, 3]
    rs = [1, 2, 3, 4, 4, 1, 3]
    hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    hosts[4][:12] = np.array(O.SPECIAL_WORDS, np.uint32).view(np.float32)

    class Fixed(adt.FixedPrecision):
        def round_tos(self):
            return list(rs)

    sync = adt.HostWeightSync(hosts, Fixed(len(counts), 32), ring_bytes=ring,
                              zero_copy_bytes=(1 << 30) if zero_copy else 0)
    assert sync.zero_copy == zero_copy
    for _ in range(3):                        # repeated transfers reuse the staging buffer
        for r_ in sync.replicas:
            r_.fill_(float("nan"))
        sync.launch(fused_norm=True)
        torch.cuda.synchronize()
        for i, (h, r) in enumerate(zip(hosts, rs)):
            want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
            assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), i
        if not ring:
            stream = sync.stream_bytes()
            for i, (h, r) in enumerate(zip(hosts, rs)):
                lo, hi = sync.layout.span(i)
                assert stream[lo:hi].tobytes() == O.pack_vectorized(h, r), i
    norms = sync.norms()
    for i, h in enumerate(hosts):
        if i == 4:
            assert math.isnan(norms[i])       # NaN payloads in the specials: the reference's norm is NaN too
            continue
        ref = O.l2_norm(h)
        assert abs(norms[i] - ref) <= NORM_RTOL * max(ref, 1e-30), i
    assert sync.h2d_bytes < 4 * sum(counts)


def _pinned_copy(h):
    t = torch.empty(h.size, dtype=torch.float32, pin_memory=True)
    t.numpy()[:] = h
    return t


def test_direct_full_width_layers_from_pinned_masters(adt):
    """ADT_H2D_DIRECT_FULL: r = 4 layers with page-locked masters are DMA'd
    straight into their replicas (no host pack, no device unpack); the other
    layers take the packed path. Replicas and norms equal the all-packed path
    bit for bit (norms: the direct layers' come from a device pass over the
    replicas, within 1e-12 of the host pass); pageable masters never go direct."""
    rng = np.random.default_rng(11)
    counts = [5000, 65536 * 2 + 7, 4097, 0, 300000, 65, 3]
    rs = [4, 1, 4, 4, 3, 4, 2]
    hosts = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in counts]
    hosts[2][:12] = np.array(O.SPECIAL_WORDS[:12], np.uint32).view(np.float32)
    hosts[2][:12][~np.isfinite(hosts[2][:12])] = 1.0  # keep this layer's norm finite
    pinned = [_pinned_copy(h) for h in hosts]

    class Fixed(adt.FixedPrecision):
        def round_tos(self):
            return list(rs)

    direct = adt.HostWeightSync(pinned, Fixed(len(counts), 32))
    packed = adt.HostWeightSync(pinned, Fixed(len(counts), 32), direct_full=False)
    pageable = adt.HostWeightSync(hosts, Fixed(len(counts), 32))
    for sync in (direct, packed, pageable):
        for _ in range(2):
            for r_ in sync.replicas:
                r_.fill_(float("nan"))
            sync.launch(fused_norm=True)
            torch.cuda.synchronize()
            for i, (h, r) in enumerate(zip(hosts, rs)):
                want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
                assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), i
    assert list(direct.direct[:len(counts)]) == [1, 0, 1, 0, 0, 1, 0]
    assert not packed.direct.any() and not pageable.direct.any()
    assert packed.norms() == pageable.norms()                          # bit-identical host sums
    for a, b, r in zip(direct.norms(), packed.norms(), rs):
        assert (a == b) if r != 4 else abs(a - b) <= 1e-12 * max(b, 1e-30)
    for i, h in enumerate(hosts):
        ref = O.l2_norm(h)
        assert abs(direct.norms()[i] - ref) <= NORM_RTOL * max(ref, 1e-30), i
    # flags = DIRECT_FULL alone: the direct layers' norms from the host pass, bit-equal to the packed path's
    from paper_2004_02297_b200 import _lib
    ss = np.zeros(len(counts), dtype=np.float64)
    flags_out = np.zeros(len(counts), dtype=np.uint8)
    _lib.check(_lib.load().adt_host_to_device_ex(
        direct._host_segs, direct.unpack_table.array, len(counts), direct._stage_ptr, direct.packed.data_ptr(),
        direct.layout.nbytes, ss.ctypes.data, 0, 0, _lib.H2D_DIRECT_FULL, flags_out.ctypes.data,
        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert list(flags_out) == [1, 0, 1, 0, 0, 1, 0]
    assert [math.sqrt(v) for v in ss] == packed.norms()
    # masters updated in place on the host: the next launch carries the new words
    for p_ in pinned:
        p_.mul_(2.0)
    direct.launch(fused_norm=True)
    torch.cuda.synchronize()
    for i, (p_, r) in enumerate(zip(pinned, rs)):
        want = p_.numpy().view(np.uint32) & np.uint32(O.keep_mask(r))
        assert np.array_equal(direct.replicas[i].cpu().numpy().view(np.uint32), want), i


@pytest.mark.parametrize("ring", [0, 48 * (320 << 10), 17 * (320 << 10)])
def test_large_set_in_many_copies(adt, ring):
    """A stream much larger than one copy batch: the DMA of early units overlaps
    the packing of later ones; every byte must still land once, in order."""
    rng = np.random.default_rng(8)
    counts = [5_000_000, 3_000_001, 777_777]
    rs = [3, 1, 2]
    hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in counts]

    class Fixed(adt.FixedPrecision):
        def round_tos(self):
            return list(rs)

    sync = adt.HostWeightSync(hosts, Fixed(len(counts), 32), min_copy_bytes=64 << 10, ring_bytes=ring,
                              slot_bytes=320 << 10)
    sync.launch(fused_norm=False)
    torch.cuda.synchronize()
    for i, (h, r) in enumerate(zip(hosts, rs)):
        want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
        assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), i
    dev = sync.packed.cpu().numpy()
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = sync.layout.span(i)
        assert dev[lo:hi].tobytes() == O.pack_vectorized(h, r)


@pytest.mark.parametrize("pinned,zero_copy", [(False, True), (True, True), (False, False)])
def test_lenet_awp_walk_host_masters(adt, golden_lenet, pinned, zero_copy):
    """SURVEY §8d config 1 through the CPU-master path: the host arrays are the
    masters (updated in place), norms come from the host pass, widths / trace
    rows / payloads / replicas equal the reference run's. pinned: page-locked
    masters, so every layer AWP has widened to 32 bits goes by direct DMA with
    its norm from the device (about half of the walk's layer-steps). zero_copy:
    the device unpack reads the packed stream from the pinned staging buffer
    (the default for a stream this small) instead of a staged copy."""
    steps = int(golden_lenet["steps"])
    walk = list(O.lenet_walk(steps, seed=7))
    L = len(walk[0][1])
    cfg = adt.PrecisionConfig(threshold=-2e-3, interval=int(golden_lenet["interval"]), step_bits=8, initial_bits=8)
    masters = [_pinned_copy(w.reshape(-1)).numpy().reshape(w.shape) if pinned else w.copy() for w in walk[0][1]]
    sync = adt.HostWeightSync(masters, adt.PrecisionController(L, cfg), zero_copy_bytes=(1 << 30) if zero_copy else 0)
    assert sync.zero_copy == zero_copy
    direct_steps = 0
    trace = []
    for t in range(steps):
        for m, w in zip(masters, walk[t][1]):
            m[...] = w
        res = sync.step(batch=t)
        trace += res.trace
        assert res.round_tos == list(golden_lenet["widths"][t]), t
        torch.cuda.synchronize()
        dev = sync.stream_bytes()
        for i in range(L):
            lo, hi = sync.layout.span(i)
            if sync.direct[i]:                 # sent as FP32 straight into the replica: no packed payload
                direct_steps += 1
            else:
                assert hashlib.sha256(dev[lo:hi].tobytes()).digest() == golden_lenet["payload_sha"][t, i].tobytes()
            rep = sync.replicas[i].cpu().numpy()
            assert hashlib.sha256(rep.tobytes()).digest() == golden_lenet["unpacked_sha"][t, i].tobytes()
    for m, w in zip(masters, walk[steps][1]):
        m[...] = w
    trace += sync.observe_final(batch=steps - 1)
    assert len(trace) == steps * L
    for k, (b, layer, norm, delta, counter, bits) in enumerate(trace):
        t, i = divmod(k, L)
        assert (b, layer) == (t, i)
        assert bits == golden_lenet["bits"][t, i] and counter == golden_lenet["counter"][t, i], (t, i)
        assert abs(norm - golden_lenet["norms"][t, i]) <= NORM_RTOL * golden_lenet["norms"][t, i]
    assert (direct_steps > 100) == pinned


def test_rejects_device_and_strided_masters(adt):
    with pytest.raises(TypeError):
        adt.HostWeightSync([torch.zeros(8, device="cuda")])
    with pytest.raises(ValueError):
        adt.HostWeightSync([np.zeros((4, 6), np.float32).T])


def test_tune_keeps_results(adt):
    """tune() / tune_threads() only pick the packer thread count and the copy
    batch: after them, transfers still produce the reference's replicas and
    bit-identical host norms (the sums never depend on the thread count)."""
    from paper_2004_02297_b200.hostsync import host_threads
    rng = np.random.default_rng(21)
    counts = [300000, 5000, 65536 * 2 + 3]
    rs = [1, 3, 2]
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]

    class Fixed(adt.FixedPrecision):
        def round_tos(self):
            return list(rs)

    sync = adt.HostWeightSync(hosts, Fixed(len(counts), 32))
    sync.launch(fused_norm=True)
    torch.cuda.synchronize()
    before = sync.norms()
    grid = sync.tune(batches=[0, 256 << 10], reps=1)
    assert f"{sync.threads}x{sync.min_copy_bytes >> 10}K" in grid and len(grid) >= 2
    timings = sync.tune_threads(reps=1)
    assert sync.threads in timings and all(1 <= t <= host_threads() for t in timings)
    for r_ in sync.replicas:
        r_.fill_(float("nan"))
    sync.launch(fused_norm=True)
    torch.cuda.synchronize()
    assert sync.norms() == before
    for i, (h, r) in enumerate(zip(hosts, rs)):
        want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
        assert np.array_equal(sync.replicas[i].cpu().numpy().view(np.uint32), want), i
