"""The paper's CPU-master setting as a training loop: the
FP32 master weights live in HOST memory and are updated by the CPU; every
batch they are packed on the host at each layer's AWP width, only the packed
bytes cross PCIe, the GPU unpacks them into the replicas its workers compute
on, and the workers' gradients come back to the host uncompressed
 for the momentum step.

    host:  masters (pinned float32) --HostWeightSync.step: pack (AWP widths, norms fused)-->
    link:  packed bytes (Σ n·r instead of 4·Σ n) --> GPU: unpack -> replicas
    GPU:   simulated workers' forward/backward on the replicas (torch/cuBLAS),
           sample-count-weighted gradient combine
    link:  combined FP32 gradients back (4·Σ n)
    host:  momentum SGD on the masters (torch CPU ops, in place), norms of the
           updated masters -> AWP (fused into the next batch's pack)

    python examples/train_mlp_cpu_master.py --steps 300
    python examples/train_mlp_cpu_master.py --steps 300 --fp32     # the uncompressed baseline

Prints one JSON line: loss, accuracy, final widths, weight bytes vs FP32 and
the wall seconds of each phase (weight transfer, GPU compute, gradient
return, host update).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200.precision import FixedPrecision

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from train_mlp_adt import blobs, forward_backward  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="256,2048,2048,10")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--interval", type=int, default=50)            # the reference's PrecisionConfig defaults
    ap.add_argument("--threshold", type=float, default=-2e-3)
    ap.add_argument("--fp32", action="store_true", help="no truncation (FixedPrecision 32 bits)")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--update-threads", type=int, default=0,
                    help="torch CPU threads for the host update (0 = torch's default); the host packer "
                         "shares the same cores")
    args = ap.parse_args(argv)
    torch.manual_seed(args.seed)
    if args.update_threads:
        torch.set_num_threads(args.update_threads)
    dev = torch.device("cuda")
    sizes = [int(s) for s in args.sizes.split(",")]
    shapes = list(zip(sizes[:-1], sizes[1:]))
    L = len(shapes)
    x_all, y_all = blobs(args.steps * args.batch + 2048, sizes[0], sizes[-1], args.seed)
    x_all, y_all = torch.from_numpy(x_all).to(dev), torch.from_numpy(y_all).to(dev)
    rng = np.random.default_rng(args.seed)
    # host masters and optimizer state, page-locked (the DMA reads full-width layers in place)
    masters = [torch.from_numpy(rng.normal(0.0, 0.1, s).astype(np.float32)).pin_memory() for s in shapes]
    vel = [torch.zeros_like(m) for m in masters]
    biases = [torch.zeros(s[1], device=dev) for s in shapes]
    vel_b = [torch.zeros_like(b) for b in biases]
    sched = FixedPrecision(L, 32) if args.fp32 else adt.PrecisionController(
        L, adt.PrecisionConfig(threshold=args.threshold, interval=args.interval, step_bits=8, initial_bits=8))
    sync = adt.HostWeightSync(masters, sched)
    sync.tune(reps=2)                                     # setup: packer threads / copy batch for this host
    reps = [r.view(s) for r, s in zip(sync.replicas, shapes)]
    grad_dev = [torch.empty(s, device=dev) for s in shapes]
    worker_g = [[torch.empty(s, device=dev) for s in shapes] for _ in range(args.workers)]
    grad_host = [torch.empty(s, dtype=torch.float32).pin_memory() for s in shapes]
    wire = raw = 0
    losses, trace = [], []
    t = {"weights_to_gpu": 0.0, "gpu_compute": 0.0, "grads_to_host": 0.0, "host_update": 0.0}
    stream = torch.cuda.current_stream()
    t_start = time.perf_counter()
    for b in range(args.steps):
        t0 = time.perf_counter()
        res = sync.step(batch=b)                          # pack (norms of the updated masters) -> H2D -> unpack
        stream.synchronize()
        t1 = time.perf_counter()
        trace += res.trace
        wire += sum(n * r for n, r in zip(sync.counts, res.round_tos))
        raw += 4 * sum(sync.counts)
        xb = x_all[b * args.batch:(b + 1) * args.batch]
        yb = y_all[b * args.batch:(b + 1) * args.batch]
        chunks = torch.chunk(torch.arange(len(yb), device=dev), args.workers)
        counts = [len(c) for c in chunks]
        bias_grads = []
        for k, idx in enumerate(chunks):
            loss, gb = forward_backward(reps, biases, xb[idx], yb[idx], worker_g[k])
            bias_grads.append(gb)
            losses.append(loss)
        total = sum(counts)
        for i in range(L):                                # sample-count-weighted combine (net.py:229-231)
            torch.mul(worker_g[0][i], counts[0] / total, out=grad_dev[i])
            for k in range(1, args.workers):
                grad_dev[i].add_(worker_g[k][i], alpha=counts[k] / total)
            g = sum(gb[i] * n for gb, n in zip(bias_grads, counts)) / total
            vel_b[i].mul_(0.9).add_(g)                    # biases travel raw and step on the GPU
            biases[i].sub_(args.lr * vel_b[i])
        stream.synchronize()
        t2 = time.perf_counter()
        for gd, gh in zip(grad_dev, grad_host):           # gradients return uncompressed
            gh.copy_(gd, non_blocking=True)
        stream.synchronize()
        t3 = time.perf_counter()
        with torch.no_grad():                             # momentum SGD on the host masters, in place
            for m, v, g in zip(masters, vel, grad_host):
                g.add_(m, alpha=5e-4)
                v.mul_(0.9).add_(g)
                m.sub_(v, alpha=args.lr)
        t4 = time.perf_counter()
        t["weights_to_gpu"] += t1 - t0
        t["gpu_compute"] += t2 - t1
        t["grads_to_host"] += t3 - t2
        t["host_update"] += t4 - t3
    trace += sync.observe_final(batch=args.steps - 1)
    secs = time.perf_counter() - t_start
    res = sync.step(batch=args.steps, observe=False)      # replicas of the final masters for evaluation
    stream.synchronize()
    with torch.no_grad():
        xe, ye = x_all[-2048:], y_all[-2048:]
        h = xe
        for i, (w, bb) in enumerate(zip(reps, biases)):
            h = torch.addmm(bb, h, w)
            h = torch.relu(h) if i + 1 < L else h
        acc = float((h.argmax(1) == ye).float().mean())
    out = {"steps": args.steps, "workers": args.workers, "mode": "fp32" if args.fp32 else "awp",
           "weights": sum(sync.counts), "first_loss": float(np.mean(losses[:args.workers])),
           "final_loss": float(np.mean(losses[-args.workers:])), "val_accuracy": acc,
           "final_bits": [sched.current_bits(i) for i in range(L)] if not args.fp32 else [32] * L,
           "weight_bytes_vs_fp32": wire / raw if raw else None, "trace_rows": len(trace), "seconds": secs,
           "phase_seconds": t, "host_threads": sync.threads, "update_threads": torch.get_num_threads()}
    print(json.dumps(out))
    return out


if __name__ == "__main__":
    main()
