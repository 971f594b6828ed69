"""The host (CPU) half of the CPU-master path: adt_pack_host, the paper's
Bitpack stage on the host cores. Runs without a
GPU: bytes against the oracle (codec.py:116-180 semantics) and the reference
golden vectors, fused norms against precision.l2_norm's float64 value, and
independence from the thread count and from the SIMD / store path."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import weightpack_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hostpack():
    from paper_2004_02297_b200 import hostsync
    return hostsync


COUNTS = [0, 1, 63, 64, 65, 1000, 65535, 65536, 65537, 140003]


@pytest.mark.parametrize("r", [1, 2, 3, 4])
@pytest.mark.parametrize("align", [16, 64])
def test_bytes_and_norms_match_oracle(hostpack, r, align):
    rng = np.random.default_rng(r)
    hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in COUNTS]
    hosts[3][:12] = np.array(O.SPECIAL_WORDS, dtype=np.uint32).view(np.float32)
    packed, lay, ss = hostpack.pack_host(hosts, [r] * len(COUNTS), align=align)
    for i, h in enumerate(hosts):
        lo, hi = lay.span(i)
        assert packed[lo:hi].tobytes() == O.pack_vectorized(h, r), (i, r)
    finite = [np.where(np.isfinite(h), h, np.float32(1)) for h in hosts]
    packed, lay, ss = hostpack.pack_host(finite, [r] * len(COUNTS), align=align)
    for h, s in zip(finite, ss):
        ref = O.l2_norm(h) ** 2
        assert abs(s - ref) <= 1e-12 * max(ref, 1e-300), (s, ref)


def test_mixed_widths_and_golden(hostpack, golden_codec):
    for case in golden_codec:
        packed, lay, _ = hostpack.pack_host([case["words"].view(np.float32)], [case["r"]])
        assert np.array_equal(packed[:lay.payload_end], case["payload"]), case["name"]
    rng = np.random.default_rng(11)
    counts = [5000, 64 * 1000 + 7, 3, 70000]
    rs = [3, 1, 4, 2]
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    packed, lay, ss = hostpack.pack_host(hosts, rs)
    for i, (h, r) in enumerate(zip(hosts, rs)):
        lo, hi = lay.span(i)
        assert packed[lo:hi].tobytes() == O.pack_vectorized(h, r)
        assert abs(np.sqrt(ss[i]) - O.l2_norm(h)) <= 1e-12 * O.l2_norm(h)


def test_thread_count_does_not_change_results(hostpack):
    rng = np.random.default_rng(5)
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in (300001, 65536 * 3 + 5, 17)]
    outs = [hostpack.pack_host(hosts, [3, 2, 1], threads=t) for t in (1, 2, 0)]
    spans = [outs[0][1].span(i) for i in range(len(hosts))]      # payloads (pad bytes are not data)
    for packed, _, ss in outs[1:]:
        for lo, hi in spans:
            assert np.array_equal(packed[lo:hi], outs[0][0][lo:hi])
        assert np.array_equal(ss, outs[0][2])          # fixed unit order: bit-identical sums


def test_rejects_copies_and_bad_widths(hostpack):
    a = np.zeros((4, 6), np.float32)
    with pytest.raises(ValueError):
        hostpack.pack_host([a.T], [2])                 # would pack a transposed copy
    with pytest.raises(TypeError):
        hostpack.pack_host([np.zeros(8)], [2])          # float64: the caller casts (codec.py:110-113)
    with pytest.raises(ValueError):
        hostpack.pack_host([np.zeros(8, np.float32)], [5])


_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
from paper_2004_02297_b200 import hostsync, _lib
rng = np.random.default_rng(9)
hosts = [rng.integers(0, 1 << 32, n, dtype=np.uint32).view(np.float32) for n in (70001, 64, 130)]
packed, lay, ss = hostsync.pack_host(hosts, [3, 4, 1])
pay = b"".join(packed[slice(*lay.span(i))].tobytes() for i in range(len(hosts)))
print(json.dumps({"simd": _lib.load().adt_host_simd(), "bytes": pay.hex(), "ss": ss.tolist()}))
"""


@pytest.mark.parametrize("env", [{"ADT_HOST_SCALAR": "1"}, {"ADT_HOST_NT": "0"}])
def test_scalar_and_regular_store_paths_agree(env):
    runs = []
    for e in ({}, env):
        p = subprocess.run([sys.executable, "-c", _SCRIPT % ROOT], env=dict(os.environ, **e),
                           capture_output=True, text=True, timeout=120)
        assert p.returncode == 0, p.stderr[-2000:]
        runs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert runs[0]["bytes"] == runs[1]["bytes"]
    assert np.allclose(runs[0]["ss"], runs[1]["ss"], rtol=1e-12, atol=0) or \
        all(np.isnan(a) == np.isnan(b) for a, b in zip(runs[0]["ss"], runs[1]["ss"]))
    if "ADT_HOST_SCALAR" in env:
        assert runs[1]["simd"] == 0


def test_concurrent_callers_share_the_pool(hostpack):
    """Several host threads call adt_pack_host at once (ctypes drops the GIL):
    calls queue on the one worker pool and every result equals the
    single-threaded one (bytes and bit-identical sums), whatever each call's
    thread count and whether the workers were spinning or asleep."""
    import threading
    import time
    rng = np.random.default_rng(12)
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in (500, 25000, 400000, 5000, 70001)]
    rs = [1, 2, 3, 4, 1]
    want_p, lay, want_ss = hostpack.pack_host(hosts, rs, threads=1)
    spans = [lay.span(i) for i in range(len(hosts))]
    bad = []

    def caller(t):
        for it in range(12):
            p, _, ss = hostpack.pack_host(hosts, rs, threads=1 + (3 * it + t) % 8)
            if any(not np.array_equal(p[a:b], want_p[a:b]) for a, b in spans) or not np.array_equal(ss, want_ss):
                bad.append((t, it))
            if it % 4 == 3:
                time.sleep(0.002)                      # the workers fall asleep before the next call

    ths = [threading.Thread(target=caller, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not bad
