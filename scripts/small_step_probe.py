"""Latency-bound sets (LeNet): the one-launch step (adt_roundtrip, cooperative
or plain grid) vs the three-launch step (pack -> finalize || unpack), each as
one CUDA-graph replay per step: back to back (K steps between two events) and
cold (L2 flushed before each step, each step between its own events).

    python scripts/small_step_probe.py            (ADT_RT_COOP=0 for the plain-grid variant)
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import workloads


def main():
    counts = workloads.counts_of("lenet")
    rng = np.random.default_rng(0)
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    scratch = torch.ones(2 * l2 // 4, device="cuda")
    sink = torch.empty((), device="cuda")
    for fuse in (True, False):
        for r in (1, 4):
            class Fixed(adt.FixedPrecision):
                def round_tos(self):
                    return [r] * len(counts)
            sync = adt.WeightSync([torch.from_numpy(h).cuda() for h in hosts], Fixed(len(counts), 32),
                                  fuse_small=fuse)
            for _ in range(50):
                sync.launch_graphed(True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(1000):
                sync.launch_graphed(True)
            b.record()
            b.synchronize()
            warm = a.elapsed_time(b)
            cold = []
            for _ in range(200):
                torch.sum(scratch, dim=0, out=sink)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sync.launch_graphed(True)
                e1.record()
                e1.synchronize()
                cold.append(e0.elapsed_time(e1) * 1e3)
            cold.sort()
            print(f"fuse_small={fuse} (one launch: {sync._small}) r={r}: back-to-back {warm:.3f} us/step, "
                  f"cold median {cold[len(cold) // 2]:.2f} us, p10 {cold[len(cold) // 10]:.2f} us "
                  f"[ADT_RT_COOP={os.environ.get('ADT_RT_COOP', '1')}]")


if __name__ == "__main__":
    main()
