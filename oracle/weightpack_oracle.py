"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A NumPy / pure-Python restatement of the reference `weightpack` package's
ADT codec and AWP controller (the hot path named in BASELINE.json). Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference
leg may import this module, and only as the checker or the timed CPU
reference — never as the product path. The product path
(`paper_2004_02297_b200`) runs CUDA kernels and fails loudly without them.

Pinning: every function here is checked against golden vectors produced by
running the reference itself (`tests/golden/make_golden.py`, which imports
`/root/reference/pkg/src/weightpack` in the build container), and against the
reference tests' known-answer vectors (`tests/test_oracle.py`).

Citations are to `/root/reference/pkg/src/weightpack/<file>:<line>`.
"""

from __future__ import annotations

import math
import struct
from concurrent.futures import ThreadPoolExecutor

import numpy as np

WORD_BYTES = 4
STREAM_HEADER = struct.Struct("<4sBBQ")  # codec.py:35 (magic, version, r, count)
STREAM_MAGIC = b"ADT1"  # codec.py:33
GROUP = 8  # codec.py:31 — weights per shuffle group

# Bit patterns with special float semantics (test_codec.py:14-27).
SPECIAL_WORDS = [
    0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001,
    0xFFC01234, 0x00000001, 0x007FFFFF, 0x807FFFFF, 0x3F800000, 0xFF7FFFFF,
]


# --------------------------------------------------------------------- codec
def valid_round_to(r) -> int:
    """codec.py:52-57 — integer-valued r in [1, 4] else ValueError."""
    ri = int(r)
    if ri != r or ri < 1 or ri > 4:
        raise ValueError(f"round_to must be an integer in [1, 4], got {r!r}")
    return ri


def round_to_for_bits(bits: int) -> int:
    """codec.py:60-67 — ceil(bits / 8) for bits in [1, 32]."""
    if bits < 1 or bits > 32:
        raise ValueError(f"bits must be in [1, 32], got {bits}")
    return (int(bits) + 7) // 8


def keep_mask(r: int) -> int:
    """codec.py:70-73 — the high r*8 bits a round trip preserves."""
    r = valid_round_to(r)
    return (0xFFFFFFFF >> (32 - 8 * r)) << (32 - 8 * r)


def as_words(x) -> np.ndarray:
    """codec.py:110-113 — cast to float32 (RNE), flatten row-major, view u32."""
    return np.ascontiguousarray(x, dtype=np.float32).reshape(-1).view(np.uint32)


def pack_scalar(x, r: int) -> bytes:
    """codec.py:116-130 — one weight at a time, top r big-endian bytes."""
    r = valid_round_to(r)
    out = bytearray()
    for w in as_words(x).tolist():
        out += w.to_bytes(4, "big")[:r]
    return bytes(out)


def _pack_words(words: np.ndarray, r: int) -> bytes:
    """codec.py:133-146 — groups of 8 words: big-endian byte view, gather the
    first r bytes of each word's 4; leftover (< 8) words one at a time."""
    n = words.size
    body = n - n % GROUP
    parts = []
    if body:
        be = np.ascontiguousarray(words[:body]).astype(">u4").view(np.uint8)
        cols = np.array([4 * j + k for j in range(GROUP) for k in range(r)], dtype=np.intp)
        parts.append(be.reshape(-1, 4 * GROUP)[:, cols].tobytes())
    for w in words[body:].tolist():
        parts.append(w.to_bytes(4, "big")[:r])
    return b"".join(parts)


def pack_vectorized(x, r: int) -> bytes:
    """codec.py:149-153 — the path the reference training loop uses."""
    r = valid_round_to(r)
    return _pack_words(as_words(x), r)


def pack_parallel(x, r: int, workers: int) -> bytes:
    """codec.py:156-180 — contiguous chunks floor(n*i/W) packed by threads into
    disjoint spans; byte-identical for every worker count."""
    r = valid_round_to(r)
    if workers < 1:
        raise ValueError(f"worker_count must be >= 1, got {workers}")
    words = as_words(x)
    n = words.size
    if workers == 1 or n < workers:
        return _pack_words(words, r)
    cuts = [n * i // workers for i in range(workers + 1)]
    out = bytearray(n * r)
    mv = memoryview(out)

    def job(i):
        lo, hi = cuts[i], cuts[i + 1]
        mv[lo * r:hi * r] = _pack_words(words[lo:hi], r)

    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(job, range(workers)))
    return bytes(out)


def unpack(payload: bytes, n: int, r: int) -> np.ndarray:
    """codec.py:183-197 — kept bytes become the word's MSBs, low bytes zero;
    returns a fresh float32 array (NaN payloads preserved, never canonicalised)."""
    r = valid_round_to(r)
    if len(payload) != n * r:
        raise ValueError(f"payload holds {len(payload)} bytes, expected {n * r}")
    be = np.zeros((n, 4), dtype=np.uint8)
    be[:, :r] = np.frombuffer(payload, dtype=np.uint8).reshape(n, r)
    return be.reshape(-1).view(">u4").astype(np.uint32).view(np.float32)


def write_container(r: int, n: int, payload: bytes) -> bytes:
    """codec.py:200-205 — '<4sBBQ' header (ADT1, v1, r, count) + payload."""
    return STREAM_HEADER.pack(STREAM_MAGIC, 1, r, n) + payload


# ----------------------------------------------------------------- precision
def l2_norm(x) -> float:
    """precision.py:25-28 — sqrt of the float64 sum of squares over all entries."""
    a = np.asarray(x, dtype=np.float64).reshape(-1)
    return float(math.sqrt(float(a @ a))) if a.size else 0.0


def sumsq(x) -> float:
    """float64 sum of squares (exact per-term for float32 inputs)."""
    a = np.asarray(x, dtype=np.float64).reshape(-1)
    return float(a @ a) if a.size else 0.0


def change_rate(curr: float, prev: float) -> float:
    """precision.py:31-39 — (curr - prev) / prev, with the zero-prev cases."""
    if prev > 0.0:
        return (curr - prev) / prev
    return 0.0 if curr == 0.0 else math.inf


class OracleController:
    """precision.py:77-148 (Alg. 1) as flat per-group lists.

    observe(group, norm) follows precision.py:125-141 step by step:
    first observation records only; otherwise delta = change_rate, counter += 1
    when delta < threshold (else reset only in `consecutive` mode); then, even
    on the first observation, a full counter escalates bits (clamped) and
    resets; finally prev_norm = norm.
    """

    def __init__(self, num_layers, threshold=-2e-3, interval=50, step_bits=8,
                 initial_bits=8, max_bits=32, consecutive=False, layer_groups=None):
        groups = list(range(num_layers)) if layer_groups is None else list(layer_groups)
        self.groups = groups
        ids = sorted(set(groups))
        self.bits = {g: initial_bits for g in ids}
        self.counter = {g: 0 for g in ids}
        self.prev = {g: None for g in ids}
        self.delta = {g: None for g in ids}
        self.threshold, self.interval = threshold, interval
        self.step_bits, self.max_bits, self.consecutive = step_bits, max_bits, consecutive

    def observe(self, group, norm):
        if self.prev[group] is None:
            self.delta[group] = None
        else:
            d = change_rate(norm, self.prev[group])
            self.delta[group] = d
            if d < self.threshold:
                self.counter[group] += 1
            elif self.consecutive:
                self.counter[group] = 0
        if self.counter[group] == self.interval:
            self.bits[group] = min(self.bits[group] + self.step_bits, self.max_bits)
            self.counter[group] = 0
        self.prev[group] = norm
        return self.bits[group]

    def observe_layer(self, layer, norm):
        return self.observe(self.groups[layer], norm)

    def round_to(self, layer):
        return round_to_for_bits(self.bits[self.groups[layer]])


# ------------------------------------------------------------ workloads (8d)
def lenet_shapes():
    """Caffe LeNet weight tensors (430,500 weights)."""
    return [(20, 1, 5, 5), (50, 20, 5, 5), (500, 800), (10, 500)]


def lenet_walk(steps=200, seed=7):
    """Config 1: W0 ~ N(0, 0.1^2) float32, then per step a
    per-layer multiplicative factor f32(1 + U(-0.015, 0.012)) (mirrors
    test_acceptance.py:138-142). Yields (step, [layer arrays]) for t = 0..steps."""
    rng = np.random.default_rng(seed)
    ws = [(rng.standard_normal(int(np.prod(s)), dtype=np.float32) * np.float32(0.1)) for s in lenet_shapes()]
    yield 0, ws
    for t in range(1, steps + 1):
        f = (1.0 + rng.uniform(-0.015, 0.012, size=len(ws))).astype(np.float32)
        ws = [w * f[i] for i, w in enumerate(ws)]
        yield t, ws


# ------------------------------------------------- SGD step
def sgd_step(w, v, g, lr, momentum, weight_decay):
    """net.py:236-246, weight half of gather_and_update for one averaged
    gradient: float32 arrays, rounding after every operation.
    Returns (new weights, new velocity)."""
    f = np.float32
    w = np.array(w, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    g = np.array(g, dtype=np.float32, copy=True)
    if weight_decay:
        g += f(weight_decay) * w
    v *= f(momentum)
    v += g
    w -= f(lr) * v
    return w, v


# ------------------------------------ gradient return
def pairwise_sum(arrays):
    """net.py:186-200: adjacent pairing, level by level (the association tree
    depends only on the list length); an odd leftover is carried up as is."""
    if not arrays:
        raise ValueError("pairwise_sum of no arrays")
    level = list(arrays)
    while len(level) > 1:
        carry = level[-1:] if len(level) % 2 else []
        level = [a + b for a, b in zip(level[0::2], level[1::2])] + carry
    return level[0]


def combine_gradients(grads, sample_counts):
    """net.py:229-231: sum_c f32(count_c) * g_c over the pairwise tree, then
    / f32(total) — float32 with rounding after every operation."""
    f = np.float32
    total = sum(int(c) for c in sample_counts)
    g = pairwise_sum([np.asarray(x, dtype=np.float32) * f(c) for x, c in zip(grads, sample_counts)])
    g = np.array(g, dtype=np.float32, copy=True)
    g /= f(total)
    return g


def gather_and_update_weights(w, v, grads, sample_counts, lr, momentum, weight_decay):
    """net.py:203-246, weight half of gather_and_update with several worker
    contributions. Returns (new weights, new velocity)."""
    return sgd_step(w, v, combine_gradients(grads, sample_counts), lr, momentum, weight_decay)
