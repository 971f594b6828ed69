"""The p2p gather-unpack kernel (adt_unpack_multi) with every source on this
GPU: P virtual ranks' send buffers (ShardPlan of the AlexNet mixed-width set)
unpacked into the full replica, vs the single-source unpack of the same
stream. On one GPU this isolates the multi-source kernel's own cost; on an
NVLink box the only difference is where (P-1)/P of the bytes come from.

    python scripts/unpack_multi_probe.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2004_02297_b200 import engine, workloads
from paper_2004_02297_b200.layout import PackedLayout
from paper_2004_02297_b200.sharded import ShardPlan


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    counts = workloads.counts_of("alexnet")
    bits = workloads.default_bits("alexnet")
    rs = [(b + 7) // 8 for b in bits]
    outs = [torch.empty(n, dtype=torch.float32, device="cuda") for n in counts]
    algo = sum((4 + r) * n for n, r in zip(counts, rs))
    print(f"AlexNet mixed widths, unpack algorithmic bytes {algo / 1e6:.1f} MB")
    for world in (1, 2, 4, 8):
        plan = ShardPlan.plan(counts, rs, world)
        bufs = [torch.randint(0, 255, (plan.send_bytes,), dtype=torch.uint8, device="cuda") for _ in range(world)]
        views, cnt, rr, offs, srcs = [], [], [], [], []
        for q in range(world):
            for pc in plan.pieces[q]:
                views.append(outs[pc.layer][pc.lo:pc.hi])
                cnt.append(pc.hi - pc.lo)
                rr.append(rs[pc.layer])
                offs.append(pc.offset)
                srcs.append(q)
        table = engine.SegmentTable(views, PackedLayout(tuple(cnt), tuple(rr), tuple(offs), plan.send_bytes),
                                    sources=srcs)
        ptrs = [b.data_ptr() for b in bufs]
        gathered = torch.cat(bufs)                    # the nccl transport's receive buffer
        flat = engine.SegmentTable(views, PackedLayout(tuple(cnt), tuple(rr),
                                                       tuple(o + q * plan.send_bytes for o, q in zip(offs, srcs)),
                                                       plan.send_bytes * world))
        start = sum(len(plan.pieces[q]) for q in range(world // 2))
        t_multi = timed(lambda: engine.unpack_multi(table, ptrs))
        t_rot = timed(lambda: engine.unpack_multi(table, ptrs, start_seg=start))
        t_flat = timed(lambda: engine.unpack(flat, gathered))
        print(f"P={world}: pieces {len(cnt):3d}  unpack_multi {t_multi * 1e3:7.1f} us ({algo / t_multi / 1e6:6.0f} GB/s)"
              f"  rotated {t_rot * 1e3:7.1f} us  single-source unpack {t_flat * 1e3:7.1f} us "
              f"({algo / t_flat / 1e6:6.0f} GB/s)")


if __name__ == "__main__":
    main()
