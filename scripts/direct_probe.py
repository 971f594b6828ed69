"""A/B of HostWeightSync's direct full-width path (ADT_H2D_DIRECT_FULL): with and
without the fused host norm pass, by host thread count, vs the all-packed path.

    python scripts/direct_probe.py
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


def best(fn, reps=7):
    fn()
    b = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        b = min(b, time.perf_counter() - t0)
    return b


def main():
    rng = np.random.default_rng(0)
    s = torch.cuda.current_stream()
    for name, bits in (("alexnet", None), ("vgg16", 32), ("vgg16", 8)):
        counts = workloads.counts_of(name)
        rs = [bits_to_round_to(b) for b in workloads.default_bits(name, bits)]

        class Fixed(FixedPrecision):
            def round_tos(self):
                return list(rs)

        pinned = []
        for n in counts:
            t = torch.empty(n, dtype=torch.float32, pin_memory=True)
            t.numpy()[:] = rng.standard_normal(n, dtype=np.float32)
            pinned.append(t.numpy())
        for direct in (True, False):
            for th in ((16, 8) if direct else (16,)):
                sy = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32), direct_full=direct, threads=th)
                for norm in (True, False):
                    def f():
                        sy.launch(fused_norm=norm)
                        s.synchronize()
                    print(f"{name} r={sorted(set(rs))} direct={direct} threads={th:2d} norm={norm}: "
                          f"{best(f) * 1e3:7.2f} ms", flush=True)
                del sy
        flat = torch.empty(sum(counts), dtype=torch.float32).pin_memory()
        dev = torch.empty_like(flat, device="cuda")

        def raw():
            dev.copy_(flat, non_blocking=True)
            s.synchronize()
        print(f"{name}: raw FP32 pinned H2D {best(raw) * 1e3:7.2f} ms", flush=True)
        del pinned, flat, dev


if __name__ == "__main__":
    main()
