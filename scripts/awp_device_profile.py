"""A few awp_on_device steps of one weight set, for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --csv python scripts/awp_device_profile.py resnet50"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
counts = workloads.counts_of(name)
masters = [torch.randn(n, device="cuda") * 0.1 for n in counts]
cfg = adt.PrecisionConfig(threshold=-2e-3, interval=50, step_bits=8, initial_bits=8)
sync = adt.WeightSync(masters, adt.PrecisionController(len(counts), cfg), awp_on_device=True, graphed=False)
for b in range(6):
    sync.step(batch=b)
torch.cuda.synchronize()
print(len(sync.drain_trace()), "rows")
