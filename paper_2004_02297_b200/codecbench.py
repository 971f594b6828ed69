"""`bench-codec`: the reference's codec micro-benchmark (bench.py, cli.py:97-119)
on the B200 codec.

Same contract as the reference: before any timing, every pack path is checked
byte-for-byte against `pack` on a fresh random input (uniform 32-bit patterns,
NaN/Inf included, bench.py:23-26) and `unpack` against the truncation-mask
law; a mismatch aborts the bench (exit 1). Timings are the best of N repeats
against the raw input size, in the reference's table and CSV formats
(BENCH_HEADER, bench.py:17, 89-104).

The reference's rows time host NumPy input -> `bytes` payload; here those
paths run the device kernels with the host<->device copies the host API
implies (scalar / vectorized / parallel all launch the same multi-tensor
kernel). Two rows are added per (size, round_to): `device` (pack of a CUDA
tensor into a device payload) and `device_unpack` — the codec itself without
the PCIe copies, timed with CUDA events.
"""

from __future__ import annotations

import time
from typing import IO

import numpy as np

from . import codec

BENCH_HEADER = ("path", "size", "round_to", "workers", "seconds", "bytes_per_s")
LARGE_INPUT_WEIGHTS = 1 << 20  # bench.py:20 — 4 MiB of float32


def random_weights(size: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform 32-bit patterns as float32 (NaN/Inf included), bench.py:23-26."""
    return rng.integers(0, 2 ** 32, size=size, dtype=np.uint32).view(np.float32)


def equivalence_precheck(size: int, round_tos, workers, rng: np.random.Generator) -> None:
    """bench.py:29-43. Raises AssertionError naming the first path that differs."""
    x = random_weights(size, rng)
    words = x.view(np.uint32)
    for r in round_tos:
        want = codec.pack(x, r)
        candidates = [("pack_vectorized", codec.pack_vectorized(x, r), f"round_to={r}")]
        candidates += [("pack_parallel", codec.pack_parallel(x, r, n), f"round_to={r}, workers={n}")
                       for n in workers]
        for name, got, where in candidates:
            if got != want:
                raise AssertionError(f"{name} mismatch at {where}")
        if not np.array_equal(codec.unpack(want).view(np.uint32), words & np.uint32(codec.truncation_mask(r))):
            raise AssertionError(f"unpack mismatch at round_to={r}")


def _host_seconds(fn, repeats: int) -> float:
    """Best wall-clock seconds of `repeats` calls (bench.py:46-51)."""
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return min(times)


def _device_seconds(fn, repeats: int) -> float:
    """Best CUDA-event seconds of `repeats` calls on device-resident data."""
    import torch
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        fn()
        stop.record()
        stop.synchronize()
        times.append(start.elapsed_time(stop) / 1e3)
    return min(times)


def run_bench(sizes, round_tos, workers, repeats: int, rng: np.random.Generator) -> list[tuple]:
    """Rows (path, size, round_to, workers, seconds, bytes_per_s) in the
    reference's order (bench.py:53-71), then `device`, `device_unpack`."""
    import torch
    rows = []

    def add(path, size, r, w, fn, timer, nbytes):
        secs = timer(fn, repeats)
        rows.append((path, size, r, w, secs, nbytes / secs))

    for size in sizes:
        x = random_weights(size, rng)
        on_dev = torch.from_numpy(x.copy()).cuda()
        for r in round_tos:
            add("scalar", size, r, 1, lambda: codec.pack(x, r), _host_seconds, x.nbytes)
            add("vectorized", size, r, 1, lambda: codec.pack_vectorized(x, r), _host_seconds, x.nbytes)
            for n in workers:
                add("parallel", size, r, n, lambda: codec.pack_parallel(x, r, n), _host_seconds, x.nbytes)
            host_block = codec.pack_vectorized(x, r)
            add("unpack", size, r, 1, lambda: codec.unpack(host_block), _host_seconds, x.nbytes)
            add("device", size, r, 1, lambda: codec.pack(on_dev, r), _device_seconds, x.nbytes)
            dev_block = codec.pack(on_dev, r)
            add("device_unpack", size, r, 1, lambda: codec.unpack(dev_block), _device_seconds, x.nbytes)
    return rows


def slow_vector_warnings(rows) -> list[str]:
    """bench.py:74-87: a soft warning wherever the vectorized pack lost to the
    scalar one on an input of at least LARGE_INPUT_WEIGHTS weights."""
    by_key = {}
    for path, size, r, _, secs, _ in rows:
        by_key.setdefault((size, r), {})[path] = secs
    msgs = []
    for path, size, r, _, secs, _ in rows:
        ref = by_key[(size, r)].get("scalar")
        if path == "vectorized" and size >= LARGE_INPUT_WEIGHTS and ref is not None and secs > ref:
            msgs.append("warning: vectorized pack slower than scalar at size=%d round_to=%d (%.4fs vs %.4fs)"
                        % (size, r, secs, ref))
    return msgs


def render_bench_table(rows) -> str:
    """The reference's text table (bench.py:89-98): columns padded to their
    widest cell, two-space gutters, a dashed rule under the header, trailing
    blanks stripped."""
    cells = [list(BENCH_HEADER)]
    for path, size, r, w, secs, bps in rows:
        cells.append([path, "%d" % size, "%d" % r, "%d" % w, "%.6f" % secs, "%.3f GB/s" % (bps / 1e9)])
    width = [max(len(c) for c in col) for col in zip(*cells)]
    fmt = lambda row: "  ".join(c + " " * (n - len(c)) for c, n in zip(row, width)).rstrip()  # noqa: E731
    out = [fmt(cells[0]), "  ".join("-" * n for n in width)] + [fmt(row) for row in cells[1:]]
    return "\n".join(out) + "\n"


def write_bench_csv(stream: IO[str], rows) -> None:
    """The reference's CSV (bench.py:101-104): header, then one row per
    timing with the float fields written as repr()."""
    lines = [",".join(BENCH_HEADER)]
    lines += [",".join([path, str(size), str(r), str(w), repr(secs), repr(bps)]) for path, size, r, w, secs, bps in rows]
    stream.write("\n".join(lines) + "\n")
