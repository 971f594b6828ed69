"""Small exercise of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): ragged multi-tensor pack (+norm) / unpack at r = 1..4, norm-only,
finalize on a side stream, fused SGD + pack, gather-unpack from several
sources, zero-copy unpack from pinned host memory.

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import engine
from paper_2004_02297_b200.layout import PackedLayout


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    counts = [0, 1, 5, 4095, 4097, 12289, 3]
    rs = [1, 2, 3, 4, 3, 2, 1]
    hosts = [rng.standard_normal(n, dtype=np.float32) for n in counts]
    devs = [torch.from_numpy(h).cuda() for h in hosts]
    packed, lay, ss = adt.pack_many(devs, rs, with_norms=True)
    outs = adt.unpack_many(packed, lay)
    norms = torch.empty(len(counts), dtype=torch.float64, device="cuda")
    engine.sumsq(engine.SegmentTable(devs, lay), norms)
    # side-stream finalize
    parts = torch.empty(max(1, engine.SegmentTable(devs, lay).npartials), dtype=torch.float64, device="cuda")
    t = engine.SegmentTable(devs, lay)
    engine.pack(t, packed, None, partials=parts)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    engine.finalize(t, parts, norms, side)
    torch.cuda.synchronize()
    # fused SGD + pack
    v = [torch.zeros_like(d) for d in devs]
    g = [torch.randn_like(d) for d in devs]
    engine.sgd_pack(engine.SgdTable(devs, v, g, lay), 0.01, 0.9, 5e-4, packed, norms)
    # gather-unpack from two sources
    a, b = packed.clone(), packed.clone()
    engine.unpack_multi(engine.SegmentTable(outs, lay, sources=[i % 2 for i in range(len(counts))]),
                        [a.data_ptr(), b.data_ptr()])
    # zero-copy from pinned host
    engine.unpack(engine.SegmentTable(outs, lay), packed.cpu().pin_memory())
    torch.cuda.synchronize()
    # fused gradient reduce + SGD + pack (gradient return path), 1, 3 and 8 contributions
    from paper_2004_02297_b200.grads import GradBucket
    for nc in (1, 3, 8):
        buckets = [GradBucket(counts, sample_count=c + 1).load([torch.randn_like(d) for d in devs])
                   for c in range(nc)]
        table = engine.ReduceSgdTable(devs, v, [buckets[0].byte_offset(l) for l in range(len(counts))], lay)
        engine.reduce_sgd_pack(table, [b.flat.data_ptr() for b in buckets], [b.sample_count for b in buckets],
                               0.01, 0.9, 5e-4, packed, norms)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
