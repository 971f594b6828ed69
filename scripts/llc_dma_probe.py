"""Does the H2D DMA read cache-hot pinned lines from the host's last-level
cache, or always from DRAM? (Decides whether a cache-resident staging ring
can take the packed stream off host DRAM in the CPU-master path.)

For a small pinned buffer (SLOT bytes), repeated N times:
  hot   — the CPU rewrites the buffer with regular stores right before each copy
  cold  — each copy reads a different slice of a 1 GiB pinned buffer
each measured alone and while host threads stream a separate 1 GiB array
(adt_pack_host, r = 1, NT stores) to load host DRAM. If hot copies keep their
rate under DRAM load while cold ones drop, the DMA is served from the LLC.

    python scripts/llc_dma_probe.py
"""

import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2004_02297_b200 import hostsync


def main():
    s = torch.cuda.current_stream()
    big = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    big.numpy()[:] = 1
    load_src = np.random.default_rng(0).standard_normal(1 << 28, dtype=np.float32)   # 1 GiB
    dev = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for slot_mb in (2, 8, 32):
        slot = slot_mb << 20
        hot = torch.empty(slot, dtype=torch.uint8, pin_memory=True)
        hv = hot.numpy()
        n = max(8, (256 << 20) // slot)

        def run(kind):                                   # copy time only (the fill is outside the clock)
            dt = 0.0
            for i in range(n):
                if kind == "hot":
                    hv[:] = i & 0xFF                     # regular stores: lines now in the CPU caches
                    src = hot
                else:
                    off = (i * slot) % ((1 << 30) - slot)
                    src = big[off:off + slot]
                t0 = time.perf_counter()
                dev[:slot].copy_(src, non_blocking=True)
                s.synchronize()
                dt += time.perf_counter() - t0
            return n * slot / dt / 1e9

        def cpu_only():
            t0 = time.perf_counter()
            for i in range(n):
                hv[:] = i & 0xFF
            return n * slot / (time.perf_counter() - t0) / 1e9

        stop = threading.Event()

        def loader():
            while not stop.is_set():
                hostsync.pack_host([load_src], [1], threads=max(1, hostsync.host_threads() - 2), align=64)

        base = {k: run(k) for k in ("hot", "cold")}
        fill = cpu_only()
        th = threading.Thread(target=loader)
        th.start()
        time.sleep(0.2)
        loaded = {k: run(k) for k in ("hot", "cold")}
        stop.set()
        th.join()
        print(f"slot {slot_mb:3d} MiB: CPU fill alone {fill:6.1f} GB/s | copy of a hot slot {base['hot']:6.1f} GB/s, "
              f"cold copy {base['cold']:6.1f} GB/s | under DRAM load: hot {loaded['hot']:6.1f}, "
              f"cold {loaded['cold']:6.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
