"""Where the drop-in per-layer API's wall time goes (bench.py e2e_dropin):
host->device, device->host and the codec calls on AlexNet's weight tensors.

    python scripts/dropin_breakdown.py
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import hostio

COUNTS = [34848, 307200, 663552, 884736, 589824, 37748736, 16777216, 4096000]
RS = [1, 2, 3, 4, 1, 2, 3, 4]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    rng = np.random.default_rng(0)
    host = [rng.standard_normal(n, dtype=np.float32) * np.float32(0.1) for n in COUNTS]
    dev = [torch.from_numpy(h).cuda() for h in host]
    blocks = [adt.pack_vectorized(h, r) for h, r in zip(host, RS)]
    packed_dev = [torch.frombuffer(bytearray(b.payload), dtype=torch.uint8).cuda() for b in blocks]
    raw = sum(h.nbytes for h in host)
    pk = sum(len(b.payload) for b in blocks)
    rows = [
        ("to_device fp32 (all layers)", raw, lambda: [hostio.to_device(h) for h in host]),
        ("to_device packed payloads", pk, lambda: [hostio.to_device(np.frombuffer(b.payload, np.uint8)) for b in blocks]),
        ("to_bytes packed", pk, lambda: [hostio.to_bytes(p) for p in packed_dev]),
        ("to_numpy_f32", raw, lambda: [hostio.to_numpy_f32(d) for d in dev]),
        ("pageable torch H2D fp32", raw, lambda: [torch.from_numpy(h).cuda() for h in host]),
        ("np.empty + touch fp32", raw, lambda: [np.empty(h.size, np.float32).fill(0) for h in host]),
        ("pack_vectorized", raw + pk, lambda: [adt.pack_vectorized(h, r) for h, r in zip(host, RS)]),
        ("unpack", pk + raw, lambda: [adt.unpack(b) for b in blocks]),
        ("l2_norm", raw, lambda: [adt.l2_norm(h) for h in host]),
    ]
    print(f"cpus {os.cpu_count()} affinity {len(os.sched_getaffinity(0))}")
    for name, nbytes, fn in rows:
        ms = timed(fn)
        print(f"{name:<32} {ms:8.2f} ms  {nbytes / ms / 1e6:8.2f} GB/s over {nbytes / 1e6:.0f} MB")


if __name__ == "__main__" and "--trace" not in sys.argv:
    main()


def trace_to_device(n=37748736):
    """Per-chunk timeline of hostio.to_device on one large layer."""
    host = np.random.default_rng(1).standard_normal(n, dtype=np.float32)
    for _ in range(3):
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        raw_out = out.view(torch.uint8)
        bufs = hostio._Stage(out.device).__enter__()
        stream = torch.cuda.current_stream()
        t = [time.perf_counter()]
        log = []
        for k, pos in enumerate(range(0, host.nbytes, hostio.CHUNK)):
            m = min(hostio.CHUNK, host.nbytes - pos)
            buf, done = bufs[k & 1]
            a = time.perf_counter()
            done.synchronize()
            b = time.perf_counter()
            hostio._parallel_memmove(buf.data_ptr(), host.ctypes.data + pos, m)
            c = time.perf_counter()
            raw_out[pos:pos + m].copy_(buf[:m], non_blocking=True)
            done.record(stream)
            d = time.perf_counter()
            log.append(f"chunk {k}: wait {1e3 * (b - a):.2f} memmove {1e3 * (c - b):.2f} issue {1e3 * (d - c):.2f}")
        a = time.perf_counter()
        stream.synchronize()
        log.append(f"final sync {1e3 * (time.perf_counter() - a):.2f}; total {1e3 * (time.perf_counter() - t[0]):.2f} ms")
    print("\n".join(log))


if __name__ == "__main__" and "--trace" in sys.argv:
    trace_to_device()
