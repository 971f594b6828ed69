"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

It imports the reference package `weightpack` from
/root/reference/pkg/src (codec + precision only; no matplotlib needed) and
writes, next to this script:

* golden_codec.npz  — pack payloads / unpacked words / norms for the
  reference tests' known-answer inputs (test_codec.py:14-27, 66-98, 123-147),
  SPECIAL_WORDS, and seeded random word sets at ragged lengths, r = 1..4.
* golden_awp.npz    — controller traces (delta, counter, bits) for the
  reference tests' seeded norm walks (test_precision.py:175-202,
  test_acceptance.py:126-155) plus consecutive-mode and grouped variants.
* golden_sgd.npz    — net.gather_and_update's weight/velocity step (net.py:236-246)
  for the fused SGD + pack kernel.
* golden_reduce_sgd.npz — net.gather_and_update with 1..16 weighted gradient
  contributions (pairwise_sum tree, net.py:186-257) for the fused
  gradient-reduce + SGD + pack kernel.
* golden_lenet.npz  — SURVEY.md §8d config 1: the LeNet weight set under a
  seeded multiplicative walk, 200 batches, driven in the reference's own
  order (training.py:209-254): pack every layer at the controller's widths
  (sha256 of each payload and of each unpacked array), then observe the
  post-update norms.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from weightpack import codec, precision  # noqa: E402  (the reference itself)

from oracle.weightpack_oracle import lenet_walk  # noqa: E402  (shared input generator)

SPECIAL_WORDS = [
    0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001,
    0xFFC01234, 0x00000001, 0x007FFFFF, 0x807FFFFF, 0x3F800000, 0xFF7FFFFF,
]
LENGTHS = [0, 1, 7, 8, 9, 15, 16, 17, 31, 33, 1003, 4095, 4096, 4097]


def random_words(n, seed):
    return np.random.default_rng(seed).integers(0, 1 << 32, size=n, dtype=np.uint32)


def codec_cases():
    cases = []
    f32 = lambda vals: np.asarray(vals, dtype=np.float32)
    cases.append(("one_r3", f32([1.0]).view(np.uint32), 3))
    cases.append(("minus_two_r1", f32([-2.0]).view(np.uint32), 1))
    cases.append(("pi_r2", f32([3.14159274]).view(np.uint32), 2))
    cases.append(("matrix_r1", np.array([0x11223344, 0x55667788, 0x99AABBCC, 0xDDEEFF00], np.uint32), 1))
    cases.append(("random37_r4", random_words(37, 0), 4))
    cases.append(("snan_r3", np.array([0x7F800001], np.uint32), 3))
    for r in (1, 2, 3, 4):
        cases.append((f"specials_r{r}", np.array(SPECIAL_WORDS * 3, np.uint32), r))
        for n in LENGTHS:
            cases.append((f"rand{n}_r{r}", random_words(n, n), r))
    out = {}
    for i, (name, words, r) in enumerate(cases):
        w = words.view(np.float32)
        block = codec.pack(w, r)
        assert codec.pack_vectorized(w, r) == block
        assert codec.pack_parallel(w, r, 3) == block
        restored = codec.unpack(block)
        out[f"c{i}_name"] = np.array(name)
        out[f"c{i}_words"] = words
        out[f"c{i}_r"] = np.array(r)
        out[f"c{i}_payload"] = np.frombuffer(block.payload, np.uint8)
        out[f"c{i}_unpacked"] = restored.view(np.uint32)
    out["ncases"] = np.array(len(cases))
    # norms of finite inputs (precision.py:25-28)
    norm_inputs = [
        np.array([3.0, 4.0], np.float32),
        np.array([], np.float32),
        np.full(1000, 0.1, np.float32),
        np.arange(6, dtype=np.float32),
        np.array([3.0e38, -3.0e38, 1e-45], np.float32),
    ]
    rng = np.random.default_rng(7)
    for n in (1, 17, 1003, 100_000):
        norm_inputs.append(rng.standard_normal(n, dtype=np.float32) * np.float32(0.1))
    for i, x in enumerate(norm_inputs):
        out[f"n{i}_x"] = x
        out[f"n{i}_norm"] = np.array(precision.l2_norm(x))
    out["nnorms"] = np.array(len(norm_inputs))
    return out


def drive(norm_seq, cfg, layer_groups=None):
    """Observe every (batch, layer) norm in the reference controller."""
    layers = len(norm_seq[0])
    c = precision.PrecisionController(layers, cfg, layer_groups)
    delta, counter, bits = [], [], []
    for row in norm_seq:
        for layer in range(layers):
            b = c.observe_batch(layer, row[layer])
            st = c.state(layer)
            delta.append(np.nan if st.last_delta is None else st.last_delta)
            counter.append(st.interval_counter)
            bits.append(b)
    return np.array(delta), np.array(counter), np.array(bits)


def awp_cases():
    out = {}
    runs = []
    for seed in (1, 2, 3):  # test_precision.py:175-202
        rng = np.random.default_rng(seed)
        norms = np.ones(4)
        seq = []
        for _ in range(120):
            norms = norms * (1.0 + rng.uniform(-0.012, 0.01, size=4))
            seq.append([float(v) for v in norms])
        runs.append((f"prec_seed{seed}", seq, dict(threshold=-2e-3, interval=5, step_bits=8, initial_bits=8), None))
    for run in range(20):  # test_acceptance.py:126-155
        rng = np.random.default_rng(1000 + run)
        interval = int(rng.integers(3, 9))
        norms = np.ones(5)
        seq = []
        for _ in range(200):
            norms = norms * (1.0 + rng.uniform(-0.015, 0.012, size=5))
            seq.append([float(v) for v in norms])
        runs.append((f"accept{run}", seq, dict(threshold=-2e-3, interval=interval, step_bits=8, initial_bits=8), None))
    # consecutive mode, a non-byte step (14 bits -> 2 bytes), zero norms, groups
    rng = np.random.default_rng(99)
    norms = np.ones(3)
    seq = []
    for _ in range(150):
        norms = norms * (1.0 + rng.uniform(-0.01, 0.006, size=3))
        seq.append([float(v) for v in norms])
    runs.append(("consecutive", seq, dict(threshold=-2e-3, interval=4, step_bits=8, initial_bits=8, consecutive=True), None))
    runs.append(("step6", seq, dict(threshold=-2e-3, interval=3, step_bits=6, initial_bits=8), None))
    runs.append(("zeros", [[0.0, 0.0, 1.0]] * 3 + [[0.0, 2.0, 0.0]] * 2, dict(threshold=-1e-3, interval=1, step_bits=8, initial_bits=8), None))
    gseq = [[v[0], v[0], v[1], v[2]] for v in seq]
    runs.append(("groups", gseq, dict(threshold=-2e-3, interval=4, step_bits=8, initial_bits=16, max_bits=24), [0, 0, 1, 2]))
    for i, (name, seq, kw, groups) in enumerate(runs):
        cfg = precision.PrecisionConfig(**kw)
        d, c, b = drive(seq, cfg, groups)
        out[f"a{i}_name"] = np.array(name)
        out[f"a{i}_norms"] = np.array(seq, dtype=np.float64)
        out[f"a{i}_cfg"] = np.array([cfg.threshold, cfg.interval, cfg.step_bits, cfg.initial_bits,
                                     cfg.max_bits, float(cfg.consecutive)], dtype=np.float64)
        out[f"a{i}_groups"] = np.array(groups if groups is not None else list(range(len(seq[0]))))
        out[f"a{i}_delta"], out[f"a{i}_counter"], out[f"a{i}_bits"] = d, c, b
    out["nruns"] = np.array(len(runs))
    return out


LENET_STEPS = 200
LENET_INTERVAL = 15


def lenet_case():
    """Reference ordering (training.py:209-254) over the seeded LeNet walk."""
    cfg = precision.PrecisionConfig(threshold=-2e-3, interval=LENET_INTERVAL, step_bits=8, initial_bits=8)
    walk = list(lenet_walk(LENET_STEPS, seed=7))
    L = len(walk[0][1])
    c = precision.PrecisionController(L, cfg)
    pay_sha, unp_sha, widths = [], [], []
    norms, delta, counter, bits = [], [], [], []
    for t in range(LENET_STEPS):
        ws = walk[t][1]
        rs = [c.current_round_to(i) for i in range(L)]
        widths.append(rs)
        row_p, row_u = [], []
        for i, w in enumerate(ws):
            blk = codec.pack_vectorized(w, rs[i])
            row_p.append(hashlib.sha256(blk.payload).digest())
            row_u.append(hashlib.sha256(codec.unpack(blk).tobytes()).digest())
        pay_sha.append(row_p)
        unp_sha.append(row_u)
        nxt = walk[t + 1][1]  # post-update master
        for i, w in enumerate(nxt):
            n = precision.l2_norm(w)
            b = c.observe_batch(i, n)
            st = c.state(i)
            norms.append(n)
            delta.append(np.nan if st.last_delta is None else st.last_delta)
            counter.append(st.interval_counter)
            bits.append(b)
    return {
        "steps": np.array(LENET_STEPS), "interval": np.array(LENET_INTERVAL),
        "widths": np.array(widths, np.int32),
        "payload_sha": np.frombuffer(b"".join(b"".join(r) for r in pay_sha), np.uint8).reshape(LENET_STEPS, L, 32),
        "unpacked_sha": np.frombuffer(b"".join(b"".join(r) for r in unp_sha), np.uint8).reshape(LENET_STEPS, L, 32),
        "norms": np.array(norms).reshape(LENET_STEPS, L), "delta": np.array(delta).reshape(LENET_STEPS, L),
        "counter": np.array(counter).reshape(LENET_STEPS, L), "bits": np.array(bits).reshape(LENET_STEPS, L),
    }


def sgd_cases():
    """net.gather_and_update (net.py:203-257) on a one-layer network with one
    gradient contribution: the weight/velocity update the fused kernel restates."""
    from weightpack import net
    out = {}
    rng = np.random.default_rng(5)
    cases = [((37, 41), 0.05, 0.9, 5e-4), ((128, 300), 1e-3, 0.9, 0.0), ((64, 65), 0.1, 0.0, 5e-4),
             ((10, 4099), 0.02, 0.5, 1e-2)]
    for i, (shape, lr, mom, wd) in enumerate(cases):
        w = (rng.standard_normal(shape) * 0.1).astype(np.float32)
        v = (rng.standard_normal(shape) * 0.01).astype(np.float32)
        g = (rng.standard_normal(shape) * 0.05).astype(np.float32)
        network = net.Network([net.Layer(w.copy(), np.zeros(shape[1], np.float32))])
        state = net.SgdState(vel_weights=[v.copy()], vel_biases=[np.zeros(shape[1], np.float32)])
        grads = net.GradientSet(weight_grads=[g.copy()], bias_grads=[np.zeros(shape[1], np.float32)], sample_count=1)
        cfg = net.SgdConfig(learning_rate=lr, momentum=mom, weight_decay=wd)
        net.gather_and_update(network, [grads], cfg, state, lr)
        out.update({f"s{i}_w": w, f"s{i}_v": v, f"s{i}_g": g, f"s{i}_hp": np.array([lr, mom, wd]),
                    f"s{i}_w1": network.layers[0].weights, f"s{i}_v1": state.vel_weights[0]})
    out["ncases"] = np.array(len(cases))
    return out


REDUCE_CASES = [
    # (shape, sample counts per contribution, lr, momentum, weight_decay)
    ((37, 41), [64], 0.05, 0.9, 5e-4),
    ((64, 130), [32, 32], 0.02, 0.9, 5e-4),
    ((33, 257), [17, 33, 50], 0.1, 0.9, 0.0),
    ((50, 100), [1, 2, 3, 4, 5], 0.01, 0.5, 1e-3),
    ((8, 4099), [64] * 8, 0.05, 0.9, 5e-4),
    ((12, 345), [3, 64, 7, 1, 100, 9, 12, 5, 64, 2, 31, 8, 4, 64, 1, 77], 0.03, 0.9, 5e-4),
    ((5, 9), [7, 7, 7, 7, 7, 7, 7], 0.2, 0.0, 0.0),
]


def reduce_sgd_cases():
    """net.gather_and_update (net.py:203-257) with several gradient
    contributions: sample-count weighting, the pairwise_sum association tree
    (net.py:186-200), the division by the total count, then the momentum step
    — what the fused reduce + SGD + pack kernel (gradient return path,
    SURVEY.md §8f item 4) restates."""
    from weightpack import net
    out = {}
    rng = np.random.default_rng(9)
    for i, (shape, counts, lr, mom, wd) in enumerate(REDUCE_CASES):
        w = (rng.standard_normal(shape) * 0.1).astype(np.float32)
        v = (rng.standard_normal(shape) * 0.01).astype(np.float32)
        gs = [(rng.standard_normal(shape) * 0.05).astype(np.float32) for _ in counts]
        zb = np.zeros(shape[1], np.float32)
        network = net.Network([net.Layer(w.copy(), zb.copy())])
        state = net.SgdState(vel_weights=[v.copy()], vel_biases=[zb.copy()])
        contribs = [net.GradientSet(weight_grads=[g.copy()], bias_grads=[zb.copy()], sample_count=c)
                    for g, c in zip(gs, counts)]
        cfg = net.SgdConfig(learning_rate=lr, momentum=mom, weight_decay=wd)
        net.gather_and_update(network, contribs, cfg, state, lr)
        out.update({f"r{i}_w": w, f"r{i}_v": v, f"r{i}_g": np.stack(gs), f"r{i}_counts": np.array(counts, np.int64),
                    f"r{i}_hp": np.array([lr, mom, wd]),
                    f"r{i}_w1": network.layers[0].weights, f"r{i}_v1": state.vel_weights[0]})
    out["ncases"] = np.array(len(REDUCE_CASES))
    return out


def format_cases():
    """Text formats next to the path, rendered by the reference itself: the
    bench-codec table and CSV (bench.py:89-104) and the AWP trace CSV
    (training.py:304-321) for fixed rows (None deltas, inf, nan, -0.0)."""
    import io
    import json
    from weightpack import bench, training
    rows = [("scalar", 1000, 1, 1, 0.0123456789, 1.23e9), ("vectorized", 1048576, 2, 1, 0.25, 16777216.0),
            ("parallel", 1000000, 3, 8, 1.5e-05, 2.6666e11), ("unpack", 7, 4, 1, 3.3e-6, 9.1e9),
            ("scalar", 2097152, 1, 1, 0.1, 8.0e7), ("vectorized", 2097152, 1, 1, 0.2, 4.0e7)]
    csv_io = io.StringIO()
    bench.write_bench_csv(csv_io, rows)
    trace = [(0, 0, 1.2345678901234567, None, 0, 8), (1, 0, 1.2, -0.02799999999999997, 1, 8),
             (1, 1, 0.0, float("inf"), 0, 16), (2, 1, float("nan"), float("nan"), 0, 16), (3, 2, -0.0, 0.0, 2, 32)]
    tr_io = io.StringIO()
    training.write_trace_csv(tr_io, trace)
    return {"bench_rows": rows, "bench_table": bench.render_bench_table(rows), "bench_csv": csv_io.getvalue(),
            "bench_warnings": bench.slow_vector_warnings(rows),
            "trace_rows": [[None if (isinstance(v, float) and v != v) else v for v in r] for r in trace],
            "trace_nan_cells": [[isinstance(v, float) and v != v for v in r] for r in trace],
            "trace_csv": tr_io.getvalue()}


def main():
    import json
    with open(os.path.join(HERE, "golden_formats.json"), "w") as f:
        json.dump(format_cases(), f, indent=1, allow_nan=True)
    np.savez_compressed(os.path.join(HERE, "golden_reduce_sgd.npz"), **reduce_sgd_cases())
    np.savez_compressed(os.path.join(HERE, "golden_sgd.npz"), **sgd_cases())
    np.savez_compressed(os.path.join(HERE, "golden_codec.npz"), **codec_cases())
    np.savez_compressed(os.path.join(HERE, "golden_awp.npz"), **awp_cases())
    np.savez_compressed(os.path.join(HERE, "golden_lenet.npz"), **lenet_case())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
