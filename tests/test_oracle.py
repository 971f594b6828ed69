"""Pin the CPU oracle against the reference's golden vectors and KATs (no GPU).

The fixtures under tests/golden/ were produced by running the reference
itself (tests/golden/make_golden.py). Everything here is CPU-only.
"""

import hashlib
import math

import numpy as np
import pytest

from oracle import weightpack_oracle as O


def test_pack_paths_match_golden(golden_codec):
    for c in golden_codec:
        x = c["words"].view(np.float32)
        want = c["payload"].tobytes()
        assert O.pack_scalar(x, c["r"]) == want, c["name"]
        assert O.pack_vectorized(x, c["r"]) == want, c["name"]
        assert O.pack_parallel(x, c["r"], 4) == want, c["name"]


def test_unpack_matches_golden(golden_codec):
    for c in golden_codec:
        got = O.unpack(c["payload"].tobytes(), c["words"].size, c["r"])
        assert np.array_equal(got.view(np.uint32), c["unpacked"]), c["name"]
        assert np.array_equal(c["unpacked"], c["words"] & np.uint32(O.keep_mask(c["r"])))


def test_reference_kats():
    # test_codec.py:66-98, 123-147
    assert O.pack_scalar([1.0], 3) == bytes([0x3F, 0x80, 0x00])
    assert O.pack_scalar([-2.0], 1) == bytes([0xC0])
    assert O.pack_scalar([np.float32(3.14159274)], 2) == bytes([0x40, 0x49])
    assert O.unpack(bytes([0x3F]), 1, 1).tolist() == [0.5]
    assert O.unpack(bytes([0x40, 0x49]), 1, 2).tolist() == [3.140625]
    assert [O.keep_mask(r) for r in (1, 2, 3, 4)] == [0xFF000000, 0xFFFF0000, 0xFFFFFF00, 0xFFFFFFFF]
    assert O.round_to_for_bits(14) == 2 and O.round_to_for_bits(17) == 3
    for bad in (0, 5, 2.5):
        with pytest.raises(ValueError):
            O.valid_round_to(bad)


def test_norms_match_golden(golden_norms):
    for x, want in golden_norms:
        got = O.l2_norm(x)
        assert got == pytest.approx(want, rel=1e-12, abs=0.0) or (got == want == 0.0)


def test_controller_matches_golden_traces(golden_awp):
    for run in golden_awp:
        L = run["norms"].shape[1]
        c = O.OracleController(L, layer_groups=run["groups"], **run["cfg"])
        k = 0
        for row in run["norms"]:
            for layer in range(L):
                b = c.observe_layer(layer, float(row[layer]))
                g = run["groups"][layer]
                d = c.delta[g]
                assert b == run["bits"][k], (run["name"], k)
                assert c.counter[g] == run["counter"][k], (run["name"], k)
                want_d = run["delta"][k]
                assert (d is None and math.isnan(want_d)) or d == want_d, (run["name"], k)
                k += 1


def test_lenet_walk_matches_golden(golden_lenet):
    """Replays config 1 with the oracle in the reference's ordering."""
    steps = int(golden_lenet["steps"])
    walk = list(O.lenet_walk(steps, seed=7))
    L = len(walk[0][1])
    c = O.OracleController(L, threshold=-2e-3, interval=int(golden_lenet["interval"]), step_bits=8, initial_bits=8)
    for t in range(0, steps):
        rs = [c.round_to(i) for i in range(L)]
        assert rs == list(golden_lenet["widths"][t])
        if t % 25 == 0:  # hashing every step is slow in pure numpy; sample
            for i, w in enumerate(walk[t][1]):
                p = O.pack_vectorized(w, rs[i])
                assert hashlib.sha256(p).digest() == golden_lenet["payload_sha"][t, i].tobytes()
                u = O.unpack(p, w.size, rs[i])
                assert hashlib.sha256(u.tobytes()).digest() == golden_lenet["unpacked_sha"][t, i].tobytes()
        for i, w in enumerate(walk[t + 1][1]):
            n = O.l2_norm(w)
            assert n == pytest.approx(golden_lenet["norms"][t, i], rel=1e-12)
            # feed the reference's own norm so the trace comparison is exact
            b = c.observe_layer(i, float(golden_lenet["norms"][t, i]))
            assert b == golden_lenet["bits"][t, i]
            assert c.counter[i] == golden_lenet["counter"][t, i]


def test_c_oracle_matches_golden(golden_codec, golden_norms):
    from oracle import c_oracle as C
    for c in golden_codec:
        x = c["words"].view(np.float32)
        assert C.pack(x, c["r"]) == c["payload"].tobytes(), c["name"]
        got = C.unpack(c["payload"].tobytes(), c["words"].size, c["r"])
        assert np.array_equal(got.view(np.uint32), c["unpacked"]), c["name"]
    for x, want in golden_norms:
        got = math.sqrt(C.sumsq(x))
        assert got == pytest.approx(want, rel=1e-12) or got == want == 0.0


def test_sgd_step_matches_reference_update(golden_sgd):
    for c in golden_sgd:
        w1, v1 = O.sgd_step(c["w"], c["v"], c["g"], *c["hp"])
        assert np.array_equal(w1.view(np.uint32), c["w1"].view(np.uint32))
        assert np.array_equal(v1.view(np.uint32), c["v1"].view(np.uint32))


def test_gather_and_update_matches_reference(golden_reduce_sgd):
    for c in golden_reduce_sgd:
        w1, v1 = O.gather_and_update_weights(c["w"], c["v"], list(c["g"]), c["counts"], *c["hp"])
        assert np.array_equal(w1.view(np.uint32), c["w1"].view(np.uint32))
        assert np.array_equal(v1.view(np.uint32), c["v1"].view(np.uint32))


def test_pairwise_tree_shape():
    # the association tree of net.py:186-200 for 5 leaves: ((a+b)+(c+d))+e
    leaves = [np.float32(x) for x in (1e8, 1.0, -1e8, 1.0, 3.0)]
    want = ((leaves[0] + leaves[1]) + (leaves[2] + leaves[3])) + leaves[4]
    assert O.pairwise_sum(leaves) == want
