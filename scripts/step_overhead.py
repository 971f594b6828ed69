"""Wall-clock cost of one AWP step through the public API (WeightSync.step:
pack with fused norm -> unpack -> 8·L-byte norm read -> PrecisionController
observe -> [repack]) vs the device time of the same step's kernels.

    python scripts/step_overhead.py [lenet resnet50 alexnet]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import workloads


def main(names):
    dev = torch.device("cuda", 0)
    for name in names:
        counts = workloads.counts_of(name)
        L = len(counts)
        masters = [torch.randn(n, device=dev) * 0.1 for n in counts]
        cfg = adt.PrecisionConfig(threshold=-2e-3, interval=50, step_bits=8, initial_bits=8)
        sync = adt.WeightSync(masters, adt.PrecisionController(L, cfg))
        for b in range(20):
            sync.step(batch=b)
        torch.cuda.synchronize()
        steps = 200
        t0 = time.perf_counter()
        for b in range(20, 20 + steps):
            sync.step(batch=b)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / steps * 1e6
        # host-side controller alone
        norms = [1.0 + 1e-4 * i for i in range(L)]
        t0 = time.perf_counter()
        for b in range(steps):
            sync.schedule.observe_all(norms, batch=b)
        ctl = (time.perf_counter() - t0) / steps * 1e6
        # device time of the same kernels (graphed, back to back)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sync.launch_graphed(True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(steps):
            sync.launch_graphed(True)
        e.record()
        e.synchronize()
        dev_us = a.elapsed_time(e) / steps * 1e3
        # the same step with the AWP decision on the device: no host read per step
        dsync = adt.WeightSync(masters, adt.PrecisionController(L, cfg), awp_on_device=True)
        for b in range(20):
            dsync.step(batch=b)
        dsync.drain_trace()
        t0 = time.perf_counter()
        for b in range(20, 20 + steps):
            dsync.step(batch=b)
        torch.cuda.synchronize()
        dwall = (time.perf_counter() - t0) / steps * 1e6
        rows = dsync.drain_trace()
        assert len(rows) == steps * L
        print(f"{name:10s} layers {L:4d}  step() wall {wall:8.1f} us   controller {ctl:7.1f} us   "
              f"device (graphed) {dev_us:7.1f} us   awp_on_device step() {dwall:7.1f} us")


if __name__ == "__main__":
    main(sys.argv[1:] or ["lenet", "resnet50", "alexnet"])
