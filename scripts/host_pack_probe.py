"""Host packer and CPU-master pipeline on the GPU box's host:
adt_pack_host throughput by thread count and width (NT vs regular stores),
then HostWeightSync (host pack || packed H2D -> unpack) vs a raw pinned FP32
H2D of the same masters, for the AlexNet mixed set and VGG-16 at r = 1..4.

    python scripts/host_pack_probe.py
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2004_02297_b200 import hostsync, workloads
from paper_2004_02297_b200.codec import bits_to_round_to
from paper_2004_02297_b200.precision import FixedPrecision


def best(fn, reps=5):
    fn()
    b = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        b = min(b, time.perf_counter() - t0)
    return b


def cudart_copy(dev_u8, host_u8, nbytes):
    dev_u8[:nbytes].copy_(host_u8[:nbytes], non_blocking=True)


def main():
    print(f"host threads {hostsync.host_threads()} simd {hostsync._lib.load().adt_host_simd()} "
          f"NT {os.environ.get('ADT_HOST_NT', '1')} prefetch {os.environ.get('ADT_HOST_PF', '8192')} B "
          f"hint {'L2' if os.environ.get('ADT_HOST_PF_HINT', '1') != '0' else 'L1'}")
    rng = np.random.default_rng(0)
    w = rng.standard_normal(1 << 26, dtype=np.float32)          # 256 MiB
    for r in (1, 2, 3, 4):
        for th in ((1, 16) if os.environ.get("PROBE_QUICK") else (1, 4, 8, 16)):
            dt = best(lambda: hostsync.pack_host([w], [r], threads=th, align=64))
            print(f"pack_host r={r} threads={th:2d}: {dt * 1e3:7.2f} ms  read {w.nbytes / dt / 1e9:6.1f} GB/s  "
                  f"(read+write {w.size * (4 + r) / dt / 1e9:6.1f} GB/s)")
    for name, bits in (("alexnet", None), ("vgg16", 8), ("vgg16", 16), ("vgg16", 24), ("vgg16", 32)):
        counts = workloads.counts_of(name)
        rs = [bits_to_round_to(b) for b in workloads.default_bits(name, bits)]
        host = [rng.standard_normal(n, dtype=np.float32) for n in counts]

        class Fixed(FixedPrecision):
            def round_tos(self):
                return list(rs)

        sync = hostsync.HostWeightSync(host, Fixed(len(counts), 32), ring_bytes=0)
        s = torch.cuda.current_stream()

        def step_of(sy):
            def f():
                sy.launch(fused_norm=True)
                s.synchronize()
            return f

        adt_step = step_of(sync)
        pinned = []
        for h in host:
            t = torch.empty(h.size, dtype=torch.float32, pin_memory=True)
            t.numpy()[:] = h
            pinned.append(t.numpy())
        dsync = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32))
        t_direct = best(step_of(dsync))
        print(f"   {name}: pinned masters, direct_full ({int(dsync.direct[:len(counts)].sum())} layers direct) "
              f"{t_direct * 1e3:.2f} ms")
        del dsync
        for slot in (384 << 10, 2 << 20, 8 << 20):
            ring = max(48 << 20, 20 * slot)
            rsync = hostsync.HostWeightSync(host, Fixed(len(counts), 32), ring_bytes=ring, slot_bytes=slot)
            print(f"   {name}: ring {ring >> 20} MiB, {slot >> 10} KiB slots: {best(step_of(rsync)) * 1e3:.2f} ms")
            del rsync

        flat = torch.empty(sum(counts), dtype=torch.float32).pin_memory()
        dev = torch.empty_like(flat, device="cuda")

        def raw():
            dev.copy_(flat, non_blocking=True)
            s.synchronize()

        t_adt, t_raw = best(adt_step), best(raw)
        lib = hostsync._lib.load()
        L = len(counts)

        def pack_only():                       # the host pass alone, into the pinned staging buffer
            lib.adt_pack_host(sync._host_segs, L, sync._stage_ptr, sync.sumsq.ctypes.data, 0)

        dev_packed = sync.packed

        def dma_only():                        # the packed stream's copy alone
            cudart_copy(dev_packed, sync.staging, sync.layout.nbytes)
            s.synchronize()

        t_pack, t_dma = best(pack_only), best(dma_only)
        print(f"   {name}: host pack alone {t_pack * 1e3:.2f} ms ({sum(counts) * 4 / t_pack / 1e9:.1f} GB/s of masters), "
              f"packed DMA alone {t_dma * 1e3:.2f} ms ({sync.layout.nbytes / t_dma / 1e9:.1f} GB/s)")
        n = sum(counts)
        print(f"{name} r={sorted(set(rs))}: HostWeightSync {t_adt * 1e3:7.2f} ms ({sync.h2d_bytes / 1e6:.0f} MB over "
              f"PCIe) vs raw FP32 pinned H2D {t_raw * 1e3:7.2f} ms ({4 * n / 1e6:.0f} MB): "
              f"{t_raw / t_adt:.2f}x")
        del sync, flat, dev, pinned


if __name__ == "__main__":
    main()
