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
    # device-resident AWP: dyn pack/unpack, observe, fixup with escalations every step (interval 1)
    nz = [d for d in devs if d.numel()]
    cfg = adt.PrecisionConfig(threshold=10.0, interval=1, step_bits=8, initial_bits=8)
    ws = adt.WeightSync(nz, adt.PrecisionController(len(nz), cfg), awp_on_device=True, graphed=False, trace_ring=2)
    for b in range(5):
        ws.step(batch=b)
    ws.gather_and_update([GradBucket([d.numel() for d in nz], sample_count=3).load([torch.randn_like(d) for d in nz])],
                         lr=0.01, batch=5)
    ws.drain_trace()
    # peer barrier: two virtual ranks on two streams
    flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    states = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for r in (1, 0):
        engine.peer_barrier([f.data_ptr() for f in flags], r, states[r], stream=streams[r])
    # multi-rank device-AWP kernels on local buffers: combine, dyn gather-unpack, fixup pieces / gather
    lay4 = PackedLayout.plan([d.numel() for d in nz], [4] * len(nz))
    tab = engine.SegmentTable(nz, lay4)
    outs4 = [torch.empty_like(d) for d in nz]
    otab = engine.SegmentTable(outs4, lay4, sources=[0] * len(nz))
    buf = torch.zeros(lay4.nbytes, dtype=torch.uint8, device="cuda")
    w = torch.full((len(nz),), 2, dtype=torch.uint8, device="cuda")
    engine.pack_dyn(tab, buf, w)
    engine.unpack_multi_dyn(otab, [buf.data_ptr()], w)
    esc = torch.tensor([1, 0] + [0] * len(nz), dtype=torch.int32, device="cuda")
    w3 = torch.full((len(nz),), 3, dtype=torch.uint8, device="cuda")
    engine.awp_fixup_pieces(tab, engine.SegmentTable(outs4, lay4), list(range(len(nz))), buf, esc, w3)
    engine.awp_fixup_gather(otab, list(range(len(nz))), [buf.data_ptr()], esc, w3)
    tails = torch.rand(2 * len(nz), dtype=torch.float64, device="cuda")
    pl = torch.tensor(list(range(len(nz))) * 2, dtype=torch.int32, device="cuda")
    engine.awp_combine(tails, pl, len(nz), torch.empty(len(nz), dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    # r02: peer-abort guard (a lone barrier times out, then every guarded kernel is a no-op),
    # float64-input norm, one-launch small step, CPU-master transfer (staging and ring)
    lone = torch.zeros(2, dtype=torch.int32, device="cuda")
    lone_flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(2)]
    engine.peer_barrier([f.data_ptr() for f in lone_flags], 0, lone, timeout_s=0.01)
    engine.unpack_multi(engine.SegmentTable(outs, lay, sources=[0] * len(counts)), [a.data_ptr()], abort=lone[1:2])
    engine.copy_multi(torch.zeros(32, dtype=torch.uint8, device="cuda"), [a.data_ptr()], 0, 32, abort=lone[1:2])
    engine.reduce_sgd_pack(table, [b.flat.data_ptr() for b in buckets], [b.sample_count for b in buckets],
                           0.01, 0.9, 5e-4, packed, norms, abort=lone[1:2])
    x64 = torch.randn(100003, dtype=torch.float64, device="cuda")
    engine.sumsq_f64(x64, torch.empty(1, dtype=torch.float64, device="cuda"))
    small = adt.WeightSync([d.clone() for d in nz], fuse_small=True)
    for _ in range(3):
        small.launch(fused_norm=True)
    hosts_nz = [h for h in hosts if h.size]
    for ring, zc in ((0, 1 << 30), (0, 0), (24 * (320 << 10), 0)):    # zero-copy, staged, ring
        hs = adt.HostWeightSync([h.copy() for h in hosts_nz], ring_bytes=ring, slot_bytes=320 << 10,
                                zero_copy_bytes=zc)
        hs.launch(fused_norm=True)
    # drop-in per-call host API: small arrays (one staged round trip) and a large one
    for n in (1, 300, 4097, 300000):
        w = rng.standard_normal(n, dtype=np.float32)
        for r in (1, 3, 4):
            blk = adt.pack_vectorized(w, r)
            adt.unpack(blk)
        adt.l2_norm(w)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
