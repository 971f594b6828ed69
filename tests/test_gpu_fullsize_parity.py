"""Byte-exact parity on the EXACT benchmarked inputs at full BASELINE sizes.

For every bench config (AlexNet mixed widths, VGG-16 at r = 1..4, ResNet-50's
161 tensors, the 1B set at r = 1 and 3) the product step (WeightSync: pack
with the norm fused, unpack) runs on bench.py's own inputs — N(0, 0.1²)
float32 from np.random.default_rng(0) — and on uniform 32-bit words, and:

* each layer's device payload hashes (sha256) to the C oracle's pack of the
  same words (oracle_pack: codec.py:116-130, per weight the top r bytes of
  the big-endian word) — a byte-order error consistent between pack and
  unpack cannot pass this;
* each replica hashes to words & truncation_mask(r) (codec.py:183-197);
* each fused norm is within 1e-6 of the oracle's float64 sum (precision.py:25-28).

ResNet-50 also runs block-level AWP (layer_groups) over a
shrinking walk at full size: widths, counters and payloads follow the oracle
controller fed the oracle's norms.
"""

import hashlib
import importlib.util
import math
import os

import numpy as np
import pytest
import torch

from oracle import c_oracle as C
from oracle import weightpack_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_inputs", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


@pytest.fixture(scope="module")
def adt():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2004_02297_b200 as adt
    return adt


def _sha(b) -> bytes:
    return hashlib.sha256(b).digest()


def _fixed(adt, rs):
    class Fixed(adt.FixedPrecision):
        def round_tos(self):
            return list(rs)
    return Fixed(len(rs), 32)


def _check(adt, hosts, rs, norms=True, tag=""):
    """One product step on `hosts` at widths `rs`; payload, replica and norm parity per layer."""
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    sync = adt.WeightSync(devs, _fixed(adt, rs))
    sync.launch(fused_norm=True)
    got_norms = sync.read_norms()
    torch.cuda.synchronize()
    packed = sync.packed[:sync.layout.nbytes].cpu().numpy()
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = sync.layout.span(i)
        assert _sha(packed[lo:hi].tobytes()) == _sha(C.pack(h, r)), (tag, i, r)
        want = h.view(np.uint32) & np.uint32(O.keep_mask(r))
        assert _sha(sync.replicas[i].cpu().numpy().tobytes()) == _sha(want.tobytes()), (tag, i, r)
        if norms:
            ref = math.sqrt(C.sumsq(h))
            assert abs(got_norms[i] - ref) <= 1e-6 * ref, (tag, i, got_norms[i], ref)
    del sync, devs


def _uniform(counts, seed=1):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in counts]


CASES = [("alexnet", None), ("vgg16", 8), ("vgg16", 16), ("vgg16", 24), ("vgg16", 32), ("resnet50", 8),
         ("resnet50", 24)]


@pytest.mark.parametrize("name,bits", CASES)
def test_bench_inputs_byte_exact(adt, name, bits):
    b = _bench()
    from paper_2004_02297_b200 import workloads
    counts = workloads.counts_of(name)
    rs = [(x + 7) // 8 for x in workloads.default_bits(name, bits)]
    _check(adt, b.host_weights(counts), rs, tag=f"{name} bench inputs")
    _check(adt, _uniform(counts), rs, norms=False, tag=f"{name} uniform words")


def test_resnet50_mixed_widths_uniform_words(adt):
    from paper_2004_02297_b200 import workloads
    counts = workloads.counts_of("resnet50")
    rs = [1 + i % 4 for i in range(len(counts))]
    _check(adt, _uniform(counts, seed=3), rs, norms=False, tag="resnet50 mixed")


@pytest.mark.parametrize("bits", [8, 24])
def test_1b_bench_inputs_byte_exact(adt, bits):
    b = _bench()
    from paper_2004_02297_b200 import workloads
    counts = workloads.counts_of("1b")
    rs = [(bits + 7) // 8] * len(counts)
    _check(adt, b.host_weights(counts), rs, tag=f"1b r={rs[0]}")


def _resnet_blocks():
    """layer_groups for ResNet-50's 161 tensors: the stem, each bottleneck block, the classifier."""
    groups = [0, 0, 0]
    g = 1
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for blk in range(blocks):
            groups += [g] * (12 if blk == 0 else 9)
            g += 1
    return groups + [g, g]


def test_resnet50_block_level_awp_full_size(adt):
    from paper_2004_02297_b200 import workloads
    counts = workloads.counts_of("resnet50")
    groups = _resnet_blocks()
    assert len(groups) == len(counts) == 161
    hosts = _bench().host_weights(counts)
    cfg = adt.PrecisionConfig(threshold=-1e-3, interval=2, step_bits=8, initial_bits=8)
    ctl = adt.PrecisionController(len(counts), cfg, layer_groups=groups)
    ref = O.OracleController(len(counts), threshold=-1e-3, interval=2, step_bits=8, initial_bits=8,
                             layer_groups=groups)
    devs = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    sync = adt.WeightSync(devs, ctl)
    rng = np.random.default_rng(2)
    expected_rows = []
    for t in range(7):
        # the reference's widths for batch t, from the oracle controller's state
        want_rs = [ref.round_to(i) for i in range(len(counts))]
        res = sync.step(batch=t)
        torch.cuda.synchronize()
        assert res.round_tos == want_rs, t
        packed = sync.packed[:sync.layout.nbytes].cpu().numpy()
        for i in range(t % 7, len(counts), 7):      # a spread of layers every step, every layer over the walk
            lo, hi = sync.layout.span(i)
            assert _sha(packed[lo:hi].tobytes()) == _sha(C.pack(hosts[i], want_rs[i])), (t, i)
        got = [(row[0], row[1], row[4], row[5]) for row in res.trace]
        assert got == expected_rows, t
        # update: the post-update masters of batch t, observed by the reference
        # (training.py:246-254) and fused into step t+1 here
        f = (1.0 + rng.uniform(-0.004, 0.001, size=len(counts))).astype(np.float32)
        expected_rows = []
        for i, h in enumerate(hosts):
            h *= f[i]
            devs[i].copy_(torch.from_numpy(h))
        for i, h in enumerate(hosts):
            bits = ref.observe_layer(i, math.sqrt(C.sumsq(h)))
            expected_rows.append((t, i, ref.counter[groups[i]], bits))
    packed = sync.packed[:sync.layout.nbytes].cpu().numpy()
    assert max(ctl.round_tos()) > 1                  # the walk escalated some blocks
