"""Data-parallel MLP training with ADT + AWP on one B200 — the caller of the path.

The reference's training loop (/root/reference/pkg/src/weightpack/training.py:
187-273) packs the master weights at each layer's AWP width, lets every
simulated worker compute gradients on its truncated copy, combines the
workers' gradients (net.gather_and_update) and feeds the post-update norms to
the controller. The same loop here, with the B200 path doing all of the
weight traffic:

* the workers' forward/backward run on the replicas (the truncated copies the
  unpack produced) — cuBLAS GEMMs via torch, written straight into each
  worker's gradient bucket;
* `WeightSync.gather_and_update` combines the contributions (sample-count
  weights, the reference's pairwise tree), steps the FP32 masters, packs them
  at the AWP widths with the norms fused, unpacks the replicas, and — with
  `--awp-on-device` — takes the AWP decision on the GPU (no host round trip);
* biases travel raw and take a plain momentum step.

    python examples/train_mlp_adt.py --steps 400 --workers 4
    python examples/train_mlp_adt.py --steps 400 --fp32          # the uncompressed baseline

Prints one JSON line: final loss and accuracy, and the weight-stream bytes
sent relative to FP32 (Σ n·r / Σ 4n over the run).
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
from paper_2004_02297_b200.grads import GradBucket
from paper_2004_02297_b200.precision import FixedPrecision


def blobs(n: int, features: int, classes: int, seed: int):
    """Gaussian clusters (the reference's synthetic dataset shape, dataset.py)."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, 0.35, size=(classes, features)).astype(np.float32)
    y = rng.integers(0, classes, n)
    x = centers[y] + rng.normal(0.0, 1.0, size=(n, features)).astype(np.float32)
    return x.astype(np.float32), y.astype(np.int64)


def forward_backward(ws, bs, x, y, grads_w):
    """Mean cross-entropy of a ReLU MLP on (x, y); weight gradients written
    into grads_w (the worker's bucket views); returns (loss, bias grads)."""
    acts = [x]
    h = x
    for i, (w, b) in enumerate(zip(ws, bs)):
        z = torch.addmm(b, h, w)
        h = torch.relu(z) if i + 1 < len(ws) else z
        acts.append(h)
    logits = acts[-1]
    logp = torch.log_softmax(logits, dim=1)
    loss = -logp[torch.arange(len(y), device=x.device), y].mean()
    delta = torch.softmax(logits, dim=1)
    delta[torch.arange(len(y), device=x.device), y] -= 1.0
    delta /= len(y)
    gb = [None] * len(ws)
    for i in range(len(ws) - 1, -1, -1):
        torch.mm(acts[i].t(), delta, out=grads_w[i])
        gb[i] = delta.sum(0)
        if i:
            delta = (delta @ ws[i].t()) * (acts[i] > 0)
    return float(loss), gb


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,512,512,10")
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--interval", type=int, default=50)
    ap.add_argument("--threshold", type=float, default=1e-3,
                    help="AWP T: a layer's counter grows when its norm's relative change is below T")
    ap.add_argument("--fp32", action="store_true", help="no truncation (FixedPrecision 32 bits)")
    ap.add_argument("--awp-on-device", action="store_true")
    ap.add_argument("--seed", type=int, default=7)
    args = ap.parse_args(argv)
    torch.manual_seed(args.seed)
    dev = torch.device("cuda")
    sizes = [int(s) for s in args.sizes.split(",")]
    x_all, y_all = blobs(args.steps * args.batch + 2048, sizes[0], sizes[-1], args.seed)
    x_all, y_all = torch.from_numpy(x_all).to(dev), torch.from_numpy(y_all).to(dev)
    rng = np.random.default_rng(args.seed)
    shapes = list(zip(sizes[:-1], sizes[1:]))
    masters = [torch.from_numpy(rng.normal(0.0, 0.1, s).astype(np.float32)).to(dev) for s in shapes]
    biases = [torch.zeros(s[1], device=dev) for s in shapes]
    vel_b = [torch.zeros_like(b) for b in biases]
    L = len(masters)
    if args.fp32:
        sched = FixedPrecision(L, 32)
    else:
        sched = adt.PrecisionController(L, adt.PrecisionConfig(threshold=args.threshold, interval=args.interval,
                                                               step_bits=8, initial_bits=8))
    sync = adt.WeightSync(masters, sched, awp_on_device=args.awp_on_device and not args.fp32)
    sync.step(batch=0)                                   # replicas of W0 at the initial widths
    reps = [r.view(s) for r, s in zip(sync.replicas, shapes)]
    buckets = [GradBucket(shapes, dev) for _ in range(args.workers)]
    wire, raw, losses = 0, 0, []
    trace = []
    t0 = time.perf_counter()
    for b in range(args.steps):
        xb = x_all[b * args.batch:(b + 1) * args.batch]
        yb = y_all[b * args.batch:(b + 1) * args.batch]
        chunks = torch.chunk(torch.arange(len(yb), device=dev), args.workers)
        bias_grads = []
        for k, idx in enumerate(chunks):
            loss, gb = forward_backward(reps, biases, xb[idx], yb[idx], buckets[k].views)
            buckets[k].sample_count = len(idx)
            bias_grads.append((gb, len(idx)))
            losses.append(loss)
        res = sync.gather_and_update(buckets, args.lr, 0.9, 5e-4, batch=b)
        if not sync.awp_on_device:                       # widths the next batch's weights travel at
            wire += sum(n * r for n, r in zip(sync.counts, res.round_tos))
            raw += 4 * sum(sync.counts)
            trace += res.trace
        total = sum(n for _, n in bias_grads)
        for i in range(L):                               # biases: raw, plain momentum step
            g = sum(gb[i] * n for gb, n in bias_grads) / total
            vel_b[i].mul_(0.9).add_(g)
            biases[i].sub_(args.lr * vel_b[i])
    if sync.awp_on_device:
        trace = sync.drain_trace()
        wire = sum(sync.counts[layer] * ((bits + 7) // 8) for _, layer, _, _, _, bits in trace)
        raw = 4 * sum(sync.counts[layer] for _, layer, *_ in trace)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    with torch.no_grad():
        xe, ye = x_all[-2048:], y_all[-2048:]
        h = xe
        for i, (w, bb) in enumerate(zip(reps, biases)):
            h = torch.addmm(bb, h, w)
            h = torch.relu(h) if i + 1 < L else h
        acc = float((h.argmax(1) == ye).float().mean())
    out = {"steps": args.steps, "workers": args.workers, "mode": "fp32" if args.fp32 else
           ("awp_on_device" if sync.awp_on_device else "awp"),
           "first_loss": float(np.mean(losses[:args.workers])), "final_loss": float(np.mean(losses[-args.workers:])),
           "val_accuracy": acc,
           "final_bits": [sched.current_bits(i) for i in range(L)] if not args.fp32 else [32] * L,
           "weight_bytes_vs_fp32": wire / raw if raw else None, "seconds": secs}
    print(json.dumps(out))
    return out


if __name__ == "__main__":
    main()
