"""Data-parallel MLP training, one rank per GPU, with ShardedWeightSync — the
multi-GPU caller of the path.

The reference simulates its data-parallel workers in one process
(/root/reference/pkg/src/weightpack/training.py:187-273); here each worker is a
torchrun rank. Every step, on every rank:

* forward/backward on this rank's slice of the batch, using its replica (the
  truncated weights the last unpack produced), gradients written straight into
  its GradBucket;
* `ShardedWeightSync.update`: one fused kernel reads every rank's gradients for
  this rank's master shard (peer memory over NVLink, or an all-to-all), combines
  them with the reference's weighting and pairwise tree, momentum-steps the
  shard, packs it at the AWP widths with its norm fused; the packed shards are
  exchanged and every rank unpacks all of them into its replica; the AWP
  decision (same inputs everywhere) picks the next widths;
* biases travel raw: gathered and combined in rank order.

With the same seed, data split and widths, the run is the one
examples/train_mlp_adt.py simulates with --workers = world size.

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/train_mlp_dp.py --steps 400

Prints one JSON line on rank 0. ADT_EXAMPLE_BACKEND=gloo lets ranks share one
GPU (test hook; p2p transport).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np
import torch
import torch.distributed as dist

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200.grads import GradBucket
from paper_2004_02297_b200.sharded import ShardedWeightSync
from train_mlp_adt import blobs, forward_backward


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,512,512,10")
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--batch", type=int, default=256, help="global batch, split over the ranks")
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--interval", type=int, default=50)
    ap.add_argument("--threshold", type=float, default=1e-3)
    ap.add_argument("--transport", default="auto", choices=("auto", "p2p", "nccl"))
    ap.add_argument("--awp-on-device", action="store_true",
                    help="AWP decision on every GPU (p2p transport): a step has no host round trip")
    ap.add_argument("--seed", type=int, default=7)
    args = ap.parse_args(argv)
    backend = os.environ.get("ADT_EXAMPLE_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group(backend, device_id=dev) if backend == "nccl" else dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    try:
        return _train(args, rank, world, dev)
    finally:
        dist.destroy_process_group()


def _train(args, rank, world, dev):
    torch.manual_seed(args.seed)
    sizes = [int(s) for s in args.sizes.split(",")]
    x_all, y_all = blobs(args.steps * args.batch + 2048, sizes[0], sizes[-1], args.seed)
    x_all, y_all = torch.from_numpy(x_all).to(dev), torch.from_numpy(y_all).to(dev)
    rng = np.random.default_rng(args.seed)
    shapes = list(zip(sizes[:-1], sizes[1:]))
    masters = [torch.from_numpy(rng.normal(0.0, 0.1, s).astype(np.float32)).to(dev) for s in shapes]
    biases = [torch.zeros(s[1], device=dev) for s in shapes]
    vel_b = [torch.zeros_like(b) for b in biases]
    L = len(masters)
    sched = adt.PrecisionController(L, adt.PrecisionConfig(threshold=args.threshold, interval=args.interval,
                                                           step_bits=8, initial_bits=8))
    sync = ShardedWeightSync(masters, sched, transport=args.transport, awp_on_device=args.awp_on_device)
    sync.step(batch=0)                                   # replicas of W0 at the initial widths
    reps = [r.view(s) for r, s in zip(sync.replicas, shapes)]
    bucket = GradBucket(shapes, dev)
    losses, wire, raw = [], 0, 0
    t0 = time.perf_counter()
    for b in range(args.steps):
        xb = x_all[b * args.batch:(b + 1) * args.batch]
        yb = y_all[b * args.batch:(b + 1) * args.batch]
        parts = torch.chunk(torch.arange(len(yb), device=dev), world)   # the simulated workers' split
        idx = parts[rank]
        loss, gb = forward_backward(reps, biases, xb[idx], yb[idx], bucket.views)
        counts = [len(p) for p in parts]
        bucket.sample_count = counts[rank]
        res = sync.update(bucket, counts, args.lr, 0.9, 5e-4, batch=b)
        if not sync.awp_on_device:                       # widths the next batch's weights travel at
            wire += sum(n * r for n, r in zip(sync.counts, res.round_tos))
            raw += 4 * sum(sync.counts)
        # biases: every rank's bias gradients, combined in rank order (as the
        # single-process example sums its workers'), then a plain momentum step
        flat_gb = torch.cat([g.reshape(-1) for g in gb])
        every = [torch.empty_like(flat_gb) for _ in range(world)]
        dist.all_gather(every, flat_gb)
        total = sum(counts)
        for i, s in enumerate(shapes):
            o = sum(t[1] for t in shapes[:i])
            g = sum(e[o:o + s[1]] * n for e, n in zip(every, counts)) / total
            vel_b[i].mul_(0.9).add_(g)
            biases[i].sub_(args.lr * vel_b[i])
        losses.append(loss)
    if sync.awp_on_device:                               # trace rows -> widths (refreshes sched)
        trace = sync.drain_trace()
        wire = sum(sync.counts[layer] * ((bits + 7) // 8) for _, layer, _, _, _, bits in trace)
        raw = 4 * sum(sync.counts[layer] for _, layer, *_ in trace)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    # every rank must hold bit-identical replicas and biases
    digest = torch.tensor([float(torch.cat([r.reshape(-1) for r in sync.replicas] + biases).double().sum())],
                          device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    digests = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(digests, digest)
    step_losses = torch.tensor(losses, dtype=torch.float64, device=digest.device)
    every_loss = [torch.zeros_like(step_losses) for _ in range(world)]
    dist.all_gather(every_loss, step_losses)
    with torch.no_grad():
        xe, ye = x_all[-2048:], y_all[-2048:]
        h = xe
        for i, (w, bb) in enumerate(zip(reps, biases)):
            h = torch.addmm(bb, h, w)
            h = torch.relu(h) if i + 1 < L else h
        acc = float((h.argmax(1) == ye).float().mean())
    out = {"steps": args.steps, "ranks": world, "transport": sync.transport,
           "mode": "awp_on_device" if sync.awp_on_device else "awp",
           "first_loss": float(np.mean([float(e[0]) for e in every_loss])),
           "final_loss": float(np.mean([float(e[-1]) for e in every_loss])),
           "val_accuracy": acc, "final_bits": [sched.current_bits(i) for i in range(L)],
           "weight_bytes_vs_fp32": wire / raw, "replicas_identical": len({float(d) for d in digests}) == 1,
           "seconds": secs}
    if rank == 0:
        print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    main()
