"""A/B: HostWeightSync through a pinned ring of large slots vs one staging
buffer as large as the stream (AlexNet mixed widths, VGG-16 r=1), wall clock
per step (launch + 16-B read-back + sync), median of 30.

    python scripts/ring_probe.py
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


def main():
    rng = np.random.default_rng(0)
    s = torch.cuda.current_stream()
    for name, bits in (("alexnet", None), ("vgg16", 8)):
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

        # more slots than host threads (each packer fills a whole chunk)
        rings = ((0, 0, 0), (24 << 20, 1 << 20, 0), (48 << 20, 2 << 20, 0), (96 << 20, 4 << 20, 0),
                 (20 * (384 << 10), 384 << 10, 0), (48 * (384 << 10), 384 << 10, 0))
        if os.environ.get("PROBE_THREADS"):          # packer threads with the staging buffer instead
            rings = tuple((0, 0, t) for t in (4, 6, 8, 10, 12, 14, 0))
        for ring, slot, th in rings:
            kw = dict(ring_bytes=ring, slot_bytes=slot) if ring else {}
            kw["threads"] = th
            sync = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32), **kw)
            tail = torch.empty(4, dtype=torch.float32, pin_memory=True)

            def one():
                sync.launch(fused_norm=True)
                tail.copy_(sync.replicas[-1][-4:], non_blocking=True)
                s.synchronize()

            for _ in range(5):
                one()
            ts = []
            for _ in range(30):
                t0 = time.perf_counter()
                one()
                ts.append(time.perf_counter() - t0)
            print(f"{name:8s} ring {ring >> 20:4d} MiB slot {slot >> 20:2d} MiB threads {th or 'all'}: "
                  f"{np.median(ts) * 1e3:7.3f} ms "
                  f"(min {np.min(ts) * 1e3:7.3f})", flush=True)
            del sync


if __name__ == "__main__":
    main()
