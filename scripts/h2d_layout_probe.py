import sys, time, torch
sys.path.insert(0, '.')
from paper_2004_02297_b200 import workloads
from paper_2004_02297_b200.grads import bucket_offsets
for name in ("resnet50", "alexnet"):
    counts = workloads.counts_of(name)
    offs, total = bucket_offsets(counts)
    fh = torch.zeros(total).pin_memory(); fd = torch.empty(total, device="cuda")
    hs = [torch.zeros(n).pin_memory() for n in counts]; ds = [torch.empty(n, device="cuda") for n in counts]
    def flat(): fd.copy_(fh, non_blocking=True)
    def per(): [d.copy_(h, non_blocking=True) for d, h in zip(ds, hs)]
    for f, lab in ((flat, "flat"), (per, "per-layer")):
        for _ in range(3): f()
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(20): f()
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
        print(name, lab, f"{dt*1e3:.3f} ms", f"{4*total/dt/1e9:.1f} GB/s")
