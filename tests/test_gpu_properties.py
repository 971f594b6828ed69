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
