"""Break the e2e step (bench.py run_e2e_weightsync) into its parts on the box:
flat pinned H2D alone, the step graph + norm read alone, and both."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import workloads
from paper_2004_02297_b200.grads import bucket_offsets
from paper_2004_02297_b200.precision import FixedPrecision


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for name in ("resnet50", "alexnet", "lenet"):
    counts = workloads.counts_of(name)
    rs = [(b + 7) // 8 for b in workloads.default_bits(name)]
    offs, total = bucket_offsets(counts)
    fh = torch.zeros(total).pin_memory()
    fd = torch.empty(total, device="cuda")
    masters = [fd[o:o + n] for o, n in zip(offs, counts)]

    class Fixed(FixedPrecision):
        def round_tos(self):
            return list(rs)
    sync = adt.WeightSync(masters, Fixed(len(masters), 32))
    h2d = lambda: fd.copy_(fh, non_blocking=True)  # noqa: E731
    stepg = lambda: (sync.launch_graphed(fused_norm=True), sync.read_norms())  # noqa: E731
    both = lambda: (h2d(), stepg())  # noqa: E731
    print(f"{name:9s} H2D {timed(h2d):.3f} ms  step+norms {timed(stepg):.3f} ms  both {timed(both):.3f} ms")
