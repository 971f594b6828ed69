"""CPU-master path for small and mid-size sets on the GPU box's host: the
worker pool's spin-before-sleep (ADT_HOST_SPIN_US), the work-unit size
(ADT_HOST_UNIT; 0 = the set-dependent default) and zero-copy unpack from the
pinned staging buffer (HostWeightSync(zero_copy_bytes=)), against a raw FP32
pinned H2D of the same masters. Each variant runs in its own process (the
knobs are read once per process). Wall clock per step, as bench.py's e2e:
launch + 16-B read-back + stream sync; median of many steps.

    python scripts/small_host_probe.py            # every variant
    python scripts/small_host_probe.py child ...  # one variant (internal)
"""

import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETS = (("lenet", 8, 400), ("resnet50", 8, 100), ("alexnet", None, 30))
VARIANTS = (  # (spin_us, unit, zero_copy_bytes)
    (0, 65536, 0),            # round-2 pool: futex wake, 64K units, staged copy
    (200, 0, 0),              # spin 200 us, set-dependent units, staged copy
    (200, 0, 2 << 20),        # ... zero copy for streams <= 2 MiB (the default)
    (0, 0, 2 << 20),
)


def child(spin, unit, zc):
    import numpy as np
    import torch

    from paper_2004_02297_b200 import hostsync, workloads
    from paper_2004_02297_b200.codec import bits_to_round_to
    from paper_2004_02297_b200.precision import FixedPrecision

    rng = np.random.default_rng(0)
    s = torch.cuda.current_stream()
    for name, bits, steps in SETS:
        counts = workloads.counts_of(name)
        rs = [bits_to_round_to(b) for b in workloads.default_bits(name, bits)]
        pinned = []
        for n in counts:
            t = torch.empty(n, dtype=torch.float32, pin_memory=True)
            t.numpy()[:] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.1)
            pinned.append(t.numpy())

        class Fixed(FixedPrecision):
            def round_tos(self):
                return list(rs)

        sync = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32), zero_copy_bytes=zc)
        tail_dev = sync.replicas[-1][-4:]
        tail = torch.empty(4, dtype=torch.float32, pin_memory=True)

        def one():
            sync.launch(fused_norm=True)
            tail.copy_(tail_dev, non_blocking=True)
            s.synchronize()

        flat = torch.empty(sum(counts), dtype=torch.float32, pin_memory=True)
        dflat = torch.empty(sum(counts), dtype=torch.float32, device="cuda")

        def raw():
            dflat.copy_(flat, non_blocking=True)
            tail.copy_(dflat[-4:], non_blocking=True)
            s.synchronize()

        def med(fn):
            for _ in range(10):
                fn()
            ts = []
            for _ in range(steps):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            return float(np.median(ts)) * 1e6, float(np.min(ts)) * 1e6

        e, emin = med(one)
        r, rmin = med(raw)
        print(f"{name:9s} spin={spin:5d} unit={unit:6d} zc={zc >> 20:3d}MiB zero_copy={int(sync.zero_copy)} "
              f"e2e {e:9.1f} us (min {emin:9.1f})  raw FP32 {r:9.1f} us (min {rmin:9.1f})  ratio {r / e:5.2f}",
              flush=True)
        del sync


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "breakdown":
        return
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        return
    for spin, unit, zc in VARIANTS:
        env = dict(os.environ, ADT_HOST_SPIN_US=str(spin), ADT_HOST_UNIT=str(unit))
        subprocess.run([sys.executable, os.path.abspath(__file__), "child", str(spin), str(unit), str(zc)],
                       env=env, check=False)


if __name__ == "__main__":
    main()


def breakdown():
    """Where a LeNet step's wall time goes: host pack alone (threads 1..all),
    launch() until it returns, the whole step, the staged copy + unpack alone,
    and a raw FP32 copy, all wall clock (median of 400)."""
    import ctypes

    import numpy as np
    import torch

    from paper_2004_02297_b200 import _lib, engine, hostsync, workloads
    from paper_2004_02297_b200.layout import PackedLayout
    from paper_2004_02297_b200.precision import FixedPrecision

    lib = _lib.load()
    rng = np.random.default_rng(0)
    counts = workloads.counts_of("lenet")
    rs = [1] * len(counts)
    pinned = []
    for n in counts:
        t = torch.empty(n, dtype=torch.float32, pin_memory=True)
        t.numpy()[:] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.1)
        pinned.append(t.numpy())
    s = torch.cuda.current_stream()

    def med(fn, steps=400):
        for _ in range(20):
            fn()
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return f"{np.median(ts) * 1e6:8.1f} us (min {np.min(ts) * 1e6:7.1f})"

    lay = PackedLayout.plan(counts, rs, align=64)
    stage = torch.empty(lay.nbytes + 64, dtype=torch.uint8, pin_memory=True)
    base = (-stage.data_ptr()) % 64
    ss = np.zeros(len(counts))
    segs = _lib.segment_array([(p.ctypes.data, p.size, o, r) for p, o, r in zip(pinned, lay.offsets, rs)])
    for th in (1, 2, 4, 8, 16):
        print(f"pack_host threads={th:2d}: " + med(lambda: lib.adt_pack_host(segs, len(counts), stage.data_ptr() + base,
                                                                             ss.ctypes.data, th)), flush=True)

    class Fixed(FixedPrecision):
        def round_tos(self):
            return list(rs)

    for zc in (0, 1 << 30):
        sync = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32), zero_copy_bytes=zc)
        tail = torch.empty(4, dtype=torch.float32, pin_memory=True)

        def launch_only():
            sync.launch(fused_norm=True)

        def step():
            sync.launch(fused_norm=True)
            tail.copy_(sync.replicas[-1][-4:], non_blocking=True)
            s.synchronize()

        def launch_then_sync():
            t0 = time.perf_counter()
            sync.launch(fused_norm=True)
            t1 = time.perf_counter()
            s.synchronize()
            return t1 - t0

        print(f"zero_copy={int(sync.zero_copy)} launch() returns: " + med(lambda: (launch_only(), s.synchronize())[0]),
              flush=True)
        print(f"zero_copy={int(sync.zero_copy)} step (launch + 16 B read-back + sync): " + med(step), flush=True)
        lt = [launch_then_sync() for _ in range(400)]
        print(f"zero_copy={int(sync.zero_copy)} host part of launch(): {np.median(lt) * 1e6:8.1f} us", flush=True)
        del sync
    host_packed = stage[base:base + lay.nbytes]
    dev_packed = torch.empty(lay.nbytes, dtype=torch.uint8, device="cuda")
    reps = [torch.empty(n, dtype=torch.float32, device="cuda") for n in counts]
    table = engine.SegmentTable(reps, lay)

    def copy_unpack():
        dev_packed.copy_(host_packed, non_blocking=True)
        engine.unpack(table, dev_packed)
        s.synchronize()

    def zc_unpack():
        engine.unpack(table, host_packed)
        s.synchronize()

    flat = torch.empty(sum(counts), dtype=torch.float32, pin_memory=True)
    dflat = torch.empty(sum(counts), dtype=torch.float32, device="cuda")

    def raw():
        dflat.copy_(flat, non_blocking=True)
        s.synchronize()

    def empty_sync():
        s.synchronize()

    print("staged copy + unpack + sync: " + med(copy_unpack))
    print("zero-copy unpack + sync:     " + med(zc_unpack))
    print("raw FP32 copy + sync:        " + med(raw))
    print("stream sync alone:           " + med(empty_sync))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "breakdown":
    breakdown()
