#!/usr/bin/env python
"""Benchmark: ADT pack+unpack GB/s (% of HBM peak) and weight-sync ms/iter.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config alexnet]

One STEP = one weight-distribution pass of the whole synthetic weight set:
  N = 1: pack every layer at its AWP width with the l2-norm fused (one launch)
         + unpack every layer into the FP32 replica (one launch);
  N > 1: each rank packs its shard (norm fused), ncclAllGather of the packed
         bytes, every rank unpacks the full set (sharded.ShardedWeightSync).
value = algorithmic bytes of all ranks / time = (Σ(4+r)n + N·Σ(r+4)n) / t,
which at N = 1 is the pack+unpack round trip 2·Σ(4+r)n / t.

Default workload: BASELINE.json configs[1] — AlexNet's 8 weight tensors
(61,090,496 weights) at widths 8/16/24/32/8/16/24/32 bits by layer index,
N(0, 0.1²) synthetic FP32 weights generated on the device (seed 0).
The working set (244 MB FP32 + 149 MB packed + 244 MB replica) exceeds the
126 MB L2, so no explicit flush is needed between steps.

`--impl reference` times the reference CPU implementation (the oracle port of
weightpack's pack_parallel / unpack / l2_norm, oracle/weightpack_oracle.py)
on the host cores, rank 0 only, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADT pack+unpack GB/s (% HBM peak); weight-sync ms/iter at 1/2/4/8 GPUs"
UNIT = "GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="alexnet", choices=["lenet", "alexnet", "vgg16", "resnet50", "1b"])
    ap.add_argument("--bits", type=int, default=None, help="uniform width (default: the config's widths)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--quiet-extra", action="store_true", help="skip per-kernel event timing")
    ap.add_argument("--no-norm", action="store_true", help="A/B only: pack without the fused l2-norm")
    ap.add_argument("--eager", action="store_true", help="launch each step eagerly instead of from CUDA graphs")
    ap.add_argument("--no-h2d", action="store_true", help="skip the pinned host->device comparison")
    ap.add_argument("--no-sgd", action="store_true", help="skip the fused SGD+pack comparison")
    ap.add_argument("--no-reduce", action="store_true",
                    help="skip the fused gradient-reduce + SGD + pack comparison (gradient return path)")
    ap.add_argument("--reduce-contribs", type=int, default=8, help="worker contributions for that comparison")
    ap.add_argument("--no-awp-step", action="store_true",
                    help="skip the per-step wall time of the AWP step (host vs device controller)")
    ap.add_argument("--l2", choices=["auto", "flush", "none"], default="auto",
                    help="flush L2 before every timed step (auto: when the FP32 masters are < 1.5x L2)")
    ap.add_argument("--transport", choices=["auto", "nccl", "p2p"], default="auto",
                    help="N > 1: fused peer-read gather-unpack over CUDA IPC (p2p; auto picks it when every "
                         "rank's GPU is a peer), or ncclAllGather of the packed bytes (nccl)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(args):
    from paper_2004_02297_b200 import workloads
    from paper_2004_02297_b200.codec import bits_to_round_to
    counts = workloads.counts_of(args.config)
    bits = workloads.default_bits(args.config, args.bits)
    return counts, bits, [bits_to_round_to(b) for b in bits]


def workload_name(args, bits):
    b = "/".join(str(x) for x in bits) if len(set(bits)) > 1 else str(bits[0])
    return f"{args.config} weight set, per-layer widths {b} bits"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML
    polling thread (every ~5 ms, plus one synchronous sample on entry and on
    exit, so even a millisecond-long region has samples); falls back to
    `nvidia-smi -lms 50` when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []            # (sm_mhz, max_mhz, set of reason names)
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()

    def _nvml_sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        masks = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        self.samples.append((float(sm), float(mx), {n for n, m in zip(self.NAMES, masks) if bits & m}))

    def _poll(self):
        while not self._stop.wait(0.005):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            try:
                phys = torch.cuda._get_nvml_device_index(self.idx)
            except Exception:
                phys = self.idx
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(phys))
            self._nvml_sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]),
                                     {n for n, v in zip(self.NAMES, parts[2:6]) if v.lower().startswith("active")}))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._stop.set()
            self.thread.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = sorted(x[0] for x in self.samples)
        reasons = sorted(set().union(*(x[2] for x in self.samples)))
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.samples[-1][1], "reasons": reasons,
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# -------------------------------------------------------- reference (CPU)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
L2_BYTES_B200 = 126 << 20          # for the config text only; the flush decision reads the device


def reference_package():
    """The UNMODIFIED reference package `weightpack`, pip-installed into
    baseline/_ref by __graft_entry__.build() (git-ignored, shipped to the GPU
    box with the snapshot). None when it is absent (then the oracle port of the
    same calls, oracle/weightpack_oracle.py, stands in and says so)."""
    if not os.path.isdir(os.path.join(REF_DIR, "weightpack")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import weightpack
    return weightpack


def reference_parallel_pack_GBps(wp, layers, rs, reps=2):
    """The reference's own threaded packer, codec.pack_parallel (codec.py:156-180)
    with one worker per host thread, in place of pack_vectorized in the same
    step (unpack + l2_norm unchanged): the host-thread-parallel form of the
    reference path, reported beside the training-path number. None without
    baseline/_ref."""
    if wp is None:
        return None
    th = reference_threads()
    byts = 2 * sum((4 + r) * w.size for w, r in zip(layers, rs))
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        blocks = [wp.pack_parallel(w, r, th) for w, r in zip(layers, rs)]
        for b in blocks:
            wp.unpack(b)
        for w in layers:
            wp.l2_norm(w)
        best = min(best, time.perf_counter() - t0)
    return {"value": byts / best / 1e9, "unit": UNIT, "pack": f"codec.pack_parallel(w, r, {th})",
            "seconds_per_pass": best}


def reference_step(wp, layers, rs, workers=1):
    """One step of the reference's own CPU path, the calls its training loop
    makes per batch (training.py:209-213 pack every layer once with
    codec.pack_vectorized, :214-225 unpack every block once per worker,
    :246-250 l2_norm of every layer; codec.py:149-153, 183-197,
    precision.py:25-28)."""
    if wp is not None:
        blocks = [wp.pack_vectorized(w, r) for w, r in zip(layers, rs)]
        for _ in range(workers):
            for b in blocks:
                wp.unpack(b)
        for w in layers:
            wp.l2_norm(w)
        return
    from oracle import weightpack_oracle as O
    payloads = [O.pack_vectorized(w, r) for w, r in zip(layers, rs)]
    for _ in range(workers):
        for p, w, r in zip(payloads, layers, rs):
            O.unpack(p, w.size, r)
    for w in layers:
        O.l2_norm(w)


def host_weights(counts, limit=None):
    """The bench inputs, generated on the host so both arms see identical bits:
    N(0, 0.1²) float32 per layer from np.random.default_rng(0) (net.py:98).
    limit: keep only the first `limit` weights of each layer (a bounded sample)."""
    import numpy as np
    rng = np.random.default_rng(0)
    out = []
    for n in counts:
        w = rng.standard_normal(n, dtype=np.float32)
        w *= np.float32(0.1)
        out.append(w if limit is None or n <= limit else np.ascontiguousarray(w[:limit]))
    return out


FULL_REFERENCE_WEIGHTS = 1 << 28   # above this the reference CPU path runs on a per-layer sample


def reference_sample(counts):
    """(per-layer limit or None, text): the whole workload unless it is too big
    for a CPU pass of a few seconds (the 1B set)."""
    if sum(counts) <= FULL_REFERENCE_WEIGHTS:
        return None, f"the whole workload ({sum(counts)} weights)"
    lim = 1 << 22
    return lim, f"first min(n, {lim}) weights of each layer ({sum(min(n, lim) for n in counts)} weights)"


def reference_kind(wp):
    return ("reference", "weightpack 0.1.0 from baseline/_ref: codec.pack_vectorized + codec.unpack + "
            "precision.l2_norm per layer (training.py:209-254)") if wp is not None else \
           ("port", "oracle/weightpack_oracle.py port of pack_vectorized + unpack + l2_norm "
            "(baseline/_ref missing)")


THREADS_NOTE = ("cores = the host threads the reference path may use: its NumPy codec calls "
                "(pack_vectorized, unpack) run on one thread, OpenBLAS ddot (l2_norm) on up to all of them")


def reference_threads():
    """Host threads the reference path may use: NumPy's codec ops are
    single-threaded; OpenBLAS's ddot (l2_norm) uses up to the affinity count."""
    return len(os.sched_getaffinity(0))


def run_cpu_baseline(counts, rs, budget_s=10.0, min_reps=2):
    """cpu_baseline of our arm: the same reference step the reference arm
    times, on the same inputs, repeated until `budget_s` of CPU work (at least
    `min_reps` passes); value = algorithmic bytes / mean pass time."""
    wp = reference_package()
    lim, sample = reference_sample(counts)
    layers = host_weights(counts, lim)
    byts = 2 * sum((4 + r) * w.size for w, r in zip(layers, rs))
    times = []
    while len(times) < min_reps or sum(times) < budget_s:
        t0 = time.perf_counter()
        reference_step(wp, layers, rs)
        times.append(time.perf_counter() - t0)
    kind, what = reference_kind(wp)
    mean = sum(times) / len(times)
    return {"value": byts / mean / 1e9, "unit": UNIT, "cores": reference_threads(), "kind": kind,
            "sample": f"{sample}; {what}; mean of {len(times)} passes ({sum(times):.1f} s)",
            "threads_note": THREADS_NOTE, "seconds_per_pass": mean, "host_cpus": os.cpu_count(),
            "with_pack_parallel": reference_parallel_pack_GBps(wp, layers, rs)}


def bench_config(args, counts, bits, rs, world=1, transport=None):
    """`config` of the JSON line — identical in both arms for the same flags."""
    flush = args.l2 == "flush" or (args.l2 == "auto" and 4 * sum(counts) < 3 * L2_BYTES_B200 // 2)
    return {"workload": workload_name(args, bits), "weights": sum(counts), "layers": len(counts),
            "widths_bits": list(bits),
            "packed_payload_bytes": sum(n * r for n, r in zip(counts, rs)),
            "algorithmic_bytes_per_step": (1 + world) * sum((4 + r) * n for n, r in zip(counts, rs)),
            "data_seed": 0,
            "l2": ("GPU arm: L2 flushed before every timed step (read of a 2x L2 buffer outside the events)"
                   if flush else "inputs larger than L2: FP32 masters > 1.5x the 126 MB L2 "
                                 "(master + packed + replica several x L2); no flush"),
            "parallelism": f"dp{world}" if world > 1 else "single"}


def main_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))    # N workers: one pack, N unpacks (training.py:214-225)
    counts, bits, rs = workload(args)
    wp = reference_package()
    lim, sample = reference_sample(counts)
    layers = host_weights(counts, lim)
    byts = (1 + world) * sum((4 + r) * w.size for w, r in zip(layers, rs))
    for _ in range(args.warmup):
        reference_step(wp, layers, rs, world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reference_step(wp, layers, rs, world)
    dt = (time.perf_counter() - t0) / args.steps
    value = byts / dt / 1e9
    kind, what = reference_kind(wp)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic N(0,0.1^2) float32 from np.random.default_rng(0), host arrays",
        "config": bench_config(args, counts, bits, rs, world=world),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": reference_threads(), "kind": kind,
                         "sample": f"{sample}; {what}; each step one pass" + (f" with {world} worker unpacks" if world > 1 else ""),
                         "threads_note": THREADS_NOTE, "host_cpus": os.cpu_count(),
                         "with_pack_parallel": reference_parallel_pack_GBps(wp, layers, rs)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def main_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ADT_BENCH_BACKEND=gloo (test hook): ranks may share one GPU; only the
    # p2p transport runs there (NCCL refuses two ranks on one device).
    backend = os.environ.get("ADT_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # communicator lines for the driver's rank check (NCCL's INIT log) and one
        # line per rank of our own, whichever transport carries the weights
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        print(f"[bench] rank {rank} of world {dist.get_world_size()} (local rank {local}, {backend}) on "
              f"{torch.cuda.get_device_name(dev)} pci {torch.cuda.get_device_properties(dev).pci_bus_id}",
              file=sys.stderr, flush=True)

    import paper_2004_02297_b200 as adt
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    from paper_2004_02297_b200.precision import FixedPrecision

    counts, bits, rs = workload(args)
    L = len(counts)
    host = host_weights(counts)                    # identical bits to the reference arm's inputs
    masters = [torch.from_numpy(h).to(dev) for h in host]
    del host
    flat_masters = None
    if world > 1:
        # one flat master store (layers at 16-B aligned offsets, the gradient
        # bucket layout): each rank's owned pieces are then one contiguous range
        from paper_2004_02297_b200.grads import bucket_offsets
        offs, total = bucket_offsets(counts)
        flat_masters = torch.zeros(max(total, 4), device=dev)
        for o, m in zip(offs, masters):
            flat_masters[o:o + m.numel()].copy_(m)
        masters = [flat_masters[o:o + n] for o, n in zip(offs, counts)]
    replicas = [torch.empty_like(m) for m in masters]

    class Fixed(FixedPrecision):
        def round_tos(self):
            return list(rs)

    sched = Fixed(L, 32)
    stream = torch.cuda.current_stream()

    # The timed step is the product's own step: WeightSync.launch (N = 1) or
    # ShardedWeightSync.launch (N > 1) — pack with the norm fused, [gather],
    # unpack. `mid` events split pack from unpack for the per-kernel numbers.
    if world == 1:
        sync = adt.WeightSync(masters, sched, replicas)
        pack_bytes = sum((4 + r) * n for n, r in zip(counts, rs))
        unpack_bytes = pack_bytes
    else:
        from paper_2004_02297_b200.sharded import ShardedWeightSync
        sync = ShardedWeightSync(masters, sched, replicas, transport=args.transport)
        plan = sync.plan
        pack_bytes = sum((pc.hi - pc.lo) * (4 + plan.round_tos[pc.layer]) for pc in plan.pieces[rank])
        unpack_bytes = sum((4 + r) * n for n, r in zip(counts, rs))
    # ours per step: pack, unpack, norm finalize (small sets: the one adt_roundtrip launch);
    # p2p adds the peer barrier and the norm-tail gather
    small = world == 1 and getattr(sync, "_small", False)
    kernels_per_step = 1 if small else 2 + (0 if args.no_norm else 1)
    if world > 1 and getattr(sync, "transport", "") == "p2p":
        kernels_per_step += 1 + (0 if args.no_norm else 1)
    elif world > 1:                               # nccl: one unpack per gathered chunk
        kernels_per_step += sum(t is not None for t in sync._chunk_tables) - 1
    fused = not args.no_norm
    run_step = sync.launch if args.eager else sync.launch_graphed

    for _ in range(args.warmup):
        run_step(fused)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    K = args.steps
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = args.l2 == "flush" or (args.l2 == "auto" and 4 * sum(counts) < 3 * l2 // 2)
    if flush:
        # Small sets (the FP32 masters fit in the 126 MB L2): before every timed
        # step, read a 2xL2 scratch buffer (outside the events) so the step
        # starts with a cold L2 holding only clean lines; each step is timed
        # by its own event pair and split at the pack/unpack boundary.
        scratch = torch.ones(2 * l2 // 4, dtype=torch.float32, device=dev)
        sink = torch.empty((), dtype=torch.float32, device=dev)
        def flushed(split):
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
            for k in range(K):
                torch.sum(scratch, dim=0, out=sink)
                ev[k][0].record(stream)
                if split:
                    sync.launch_graphed(fused, mid_event=ev[k][1])
                else:
                    run_step(fused)
                ev[k][2].record(stream)
            torch.cuda.synchronize()
            return ev

        if world == 1 and not args.quiet_extra:       # capture the split graphs outside the timed passes
            sync.launch_graphed(fused, mid_event=torch.cuda.Event(enable_timing=True))
            run_step(fused)
            torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            step_ms = [a.elapsed_time(c) for a, _, c in flushed(False)]
        flushed_split = None
        if world == 1 and not args.quiet_extra:   # second pass: pack | unpack split (two graphs)
            ev = flushed(True)
            flushed_split = ([a.elapsed_time(b) for a, b, _ in ev], [b.elapsed_time(c) for _, b, c in ev])
    else:
        # pass 1 (the reported value): K whole steps back to back, one graph each
        with ClockSampler(local) as clocks:
            e_start.record(stream)
            for k in range(K):
                run_step(fused)
            e_end.record(stream)
            torch.cuda.synchronize()
    # pass 2 (per-kernel split for the roofline). N = 1: each phase of the step
    # (pack | finalize||unpack) replayed back to back from a graph of 20 copies,
    # two events around each replay batch (no launch latency, no event nodes
    # between kernels). N > 1 (eager): an event between the pack (+ gather) and
    # the unpack of each step.
    pk_list, up_list = [], []
    if flush:
        if flushed_split is not None:
            pk_list, up_list = flushed_split
    elif not args.quiet_extra:
        if world == 1 and not args.eager:
            a_ms, b_ms = sync.phase_ms(fused, reps=20, rounds=max(1, min(K, 200) // 20))
            pk_list, up_list = [a_ms], [b_ms]
        else:
            for _ in range(K):
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(stream)
                sync.launch(fused, mid_event=e1)
                e2.record(stream)
                torch.cuda.synchronize()
                pk_list.append(e0.elapsed_time(e1))
                up_list.append(e1.elapsed_time(e2))
    if world > 1:
        sync.check_barrier()
        dist.barrier()
    ms = sum(step_ms) / K if flush else e_start.elapsed_time(e_end) / K
    if world > 1:
        t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_bytes = (sum((4 + r) * n for n, r in zip(counts, rs))            # pack: every weight once (sharded)
                   + world * sum((4 + r) * n for n, r in zip(counts, rs)))  # unpack: every rank, full set
    value = total_bytes / (ms * 1e-3) / 1e9

    pk = up = None
    if pk_list:
        pk = sum(pk_list) / len(pk_list)
        up = sum(up_list) / len(up_list)
    hbm, peak_kind = peaks()
    roofline = None
    if small:
        # the step IS one kernel (adt_roundtrip): its duration is the step's
        dom, dur, byts = "adt_roundtrip_kernel", ms, total_bytes
        roofline = {"bound": "hbm", "achieved": byts / (dur * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": byts / (dur * 1e-3) / 1e9 / hbm, "traffic": traffic_of(dom, args), "kernel": dom,
                    "peak_source": f"{peak_kind} hbm_gbs (burst copy)", "step_kernels": 1,
                    "split_two_kernel_path": {"pack_ms": pk, "unpack_ms": up} if pk is not None else None}
    elif pk is not None:
        if world == 1:
            dom, dur, byts = ("adt_unpack_kernel", up, unpack_bytes) if up >= pk else ("adt_pack_kernel", pk, pack_bytes)
        else:
            dom, dur, byts = "adt_unpack_kernel", up, unpack_bytes
        achieved = byts / (dur * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic_of(dom, args), "kernel": dom, "peak_source": f"{peak_kind} hbm_gbs (burst copy)",
                    "pack_ms": pk, "unpack_ms": up,
                    "pack_GBps": pack_bytes / (pk * 1e-3) / 1e9, "unpack_GBps": unpack_bytes / (up * 1e-3) / 1e9}

    if roofline is not None:
        roofline["frac_spec"] = roofline["achieved"] / SPEC_HBM_GBPS
        if roofline.get("traffic"):
            dram = roofline["traffic"] / (dur * 1e-3) / 1e9
            roofline["dram_GBps"] = dram
            roofline["dram_frac"] = dram / hbm
        if world == 1 and not args.quiet_extra and not small:
            l2b = torch.cuda.get_device_properties(dev).L2_cache_size
            if 4 * (8 * sum(counts) + sync.layout.nbytes) > 2 * l2b:
                roofline["cold"] = run_cold_roofline(sync, pack_bytes, unpack_bytes, hbm, not args.no_norm)
            else:
                roofline["cold"] = {"note": "not applicable: four copies of the set fit in L2 (latency-bound set)"}

    # ---- e2e through the public API with host buffers (pinned H2D in the timed region)
    e2e = e2e_dropin = e2e_fp32_h2d = None
    if not args.no_e2e and world == 1:
        e2e_fp32_h2d = run_e2e_weightsync(args, masters, rs, dev)
        e2e = run_e2e_host_master(args, host_weights(counts), rs, dev)
        e2e_dropin = run_e2e(args, masters, rs, dev)
    elif not args.no_e2e and world > 1:
        e2e = run_e2e_sharded(args, sync, counts, rs, dev, backend, flat_masters)

    h2d = None
    if not args.no_h2d and world == 1:
        h2d = run_h2d(sync)
    sgd = None
    if not args.no_sgd and world == 1:
        sgd = run_sgd_compare(masters, rs, dev)
    awp = None
    if not args.no_awp_step and world == 1:
        awp = run_awp_step(masters)
    red = None
    if not args.no_reduce and world == 1:
        red = run_reduce_compare(masters, rs, dev, args.reduce_contribs)
    fp32_gather = None
    if world > 1:
        fp32_gather = run_fp32_allgather(counts, world, dev) if backend == "nccl" else None
    exchange = None
    if world > 1:
        # SURVEY §8e report: packed bytes each rank receives from its peers per
        # step and the bus rate over the whole step (nccl-tests busbw convention),
        # and the same step at 32 bits over the same transport: the target is
        # sync(P, widths) / sync_fp32(P) = Σ n·r / 4 Σ n
        payload = sum(n * r for n, r in zip(counts, rs))
        per_rank = payload - sync.plan.rank_payload_bytes(rank)
        fp32_ms = run_fp32_sync(sync, masters, replicas, K, dev, backend, args)
        exchange = {"packed_bytes_total": payload, "bytes_received_per_rank": per_rank,
                    "busbw_GBps": payload * (world - 1) / world / (ms * 1e-3) / 1e9,
                    "pack_ms": pk, "gather_unpack_ms": up, "sync_ms": ms,
                    "fp32_sync_ms": fp32_ms, "transport": sync.transport,
                    "target_ratio": payload / (4 * sum(counts)),
                    "achieved_ratio": (ms / fp32_ms) if fp32_ms else None}
    dp = None
    if world > 1 and not args.no_reduce:
        dp = run_dp_update(sync, counts, world, dev, backend)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(counts, rs)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic N(0,0.1^2) float32 from np.random.default_rng(0), copied to the device",
            "config": bench_config(args, counts, bits, rs, world=world),
            "setup": {"fused_norm": not args.no_norm, "transport": getattr(sync, "transport", "local"),
                      "l2_flushed": flush, "graphed": not args.eager},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_dropin": e2e_dropin,
            "e2e_device_pack": e2e_fp32_h2d,
            "gpu_launches": kernels_per_step * K, "clocks": clocks.summary(),
            "sync_ms_per_iter": ms, "host_to_device": h2d, "fp32_allgather": fp32_gather, "exchange": exchange,
            "fused_sgd_pack": sgd, "fused_reduce_sgd_pack": red, "dp_update": dp, "awp_step": awp,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


SPEC_HBM_GBPS = 8000.0     # B200 HBM3e nominal (DGX figure; B200_PROFILING.md), for frac_spec


def _graph_ms(fns, reps=10, rounds=5):
    """Median over `rounds` replays of one CUDA graph holding `reps` copies of
    the sequence `fns` -> device ms per copy (events only around the replay)."""
    import torch
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            for f in fns:
                f()
    g.replay()
    out = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return sorted(out)[len(out) // 2]


def run_cold_roofline(sync, pack_bytes, unpack_bytes, hbm, fused_norm=True):
    """SURVEY §8d cold-L2 per-kernel figures, by rotation: K independent
    copies of the step's buffers (masters, packed stream, replicas; K = 4, or
    2 when a copy is over 1 GB) and one CUDA graph of `reps` x K launches that
    cycles through them — pack(0), pack(1), ..., pack(K-1), pack(0), ... Every
    launch reads inputs last touched K-1 launches (>= 3 x its own traffic, well
    over the 126 MB L2) earlier, i.e. from DRAM, and the write-backs of the
    previous launches' outputs land inside the timed region: steady-state
    streaming, nothing left in L2 for free. Same for the unpack. Median of 5
    replays; per-launch ms = replay time / (reps x K)."""
    import torch
    from paper_2004_02297_b200 import engine
    dev = sync.device
    lay = sync.layout
    foot = 4 * sum(lay.counts) * 2 + lay.nbytes
    K = 4 if foot < (1 << 30) else 2
    sets = []
    for k in range(K):
        masters = [m.clone() for m in sync.masters]
        reps = [torch.empty_like(m) for m in sync.masters]
        packed = torch.empty_like(sync.packed)
        parts = torch.empty_like(sync._partials)
        sets.append((engine.SegmentTable(masters, lay), engine.SegmentTable(reps, lay), packed, parts))
    for ptab, utab, packed, parts in sets:           # every packed copy holds a real stream
        engine.pack(ptab, packed, None, torch.cuda.current_stream(), partials=parts)
    reps_per = max(2, 8 // K)

    def packs():                                     # current stream: the capture stream inside _graph_ms
        for ptab, _, packed, parts in sets:
            engine.pack(ptab, packed, None, torch.cuda.current_stream(), partials=parts if fused_norm else None)

    def unpacks():
        for _, utab, packed, _ in sets:
            engine.unpack(utab, packed, torch.cuda.current_stream())

    p = _graph_ms([packs], reps=reps_per) / K
    u = _graph_ms([unpacks], reps=reps_per) / K
    pg, ug = pack_bytes / (p * 1e-3) / 1e9, unpack_bytes / (u * 1e-3) / 1e9
    del sets
    torch.cuda.empty_cache()
    # Size-matched copy ceiling: one streaming kernel moving the pack's byte
    # volume (pack_bytes / 2 read + the same written), same rotation (K
    # source/destination pairs, one launch each): what a plain copy reaches on
    # a stream of this size, launch ramp and drain included.
    half = max(16, pack_bytes // 2 // 16 * 16)
    pairs = [(torch.empty(half // 4, dtype=torch.float32, device=dev),
              torch.empty(half // 4, dtype=torch.float32, device=dev)) for _ in range(K)]
    for a, b in pairs:
        a.fill_(1)

    def copies():                                    # an SM streaming kernel (inside a CUDA graph a
        for a, b in pairs:                           # copy_ becomes a copy-engine memcpy node: ~3 TB/s)
            torch.neg(a, out=b)

    c = _graph_ms([copies], reps=reps_per) / K
    cg = 2 * half / (c * 1e-3) / 1e9
    del pairs
    torch.cuda.empty_cache()
    return {"pack_ms": p, "unpack_ms": u, "pack_GBps": pg, "unpack_GBps": ug, "pack_frac": pg / hbm,
            "unpack_frac": ug / hbm, "frac": min(pg, ug) / hbm, "frac_spec": min(pg, ug) / SPEC_HBM_GBPS,
            "size_matched_copy_GBps": cg, "frac_of_size_matched_copy": min(pg, ug) / cg,
            "method": f"rotation over {K} buffer sets, CUDA graph of {reps_per * K} launches, median of 5 replays; "
                      f"size-matched copy: torch float32 elementwise kernel (neg) reading and writing {half} B each, "
                      f"same rotation"}


def traffic_of(kernel, args):
    """dram bytes per launch from a committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(args.config, {}).get(kernel)
    except Exception:
        return None


def _time_ms(fn, reps):
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_h2d(sync, reps=10):
    """The paper's CPU-master setting: weights cross from
    pinned host memory to the GPU. Compares, on the same layer set,
      raw FP32 H2D (4n bytes, one contiguous copy) — the uncompressed baseline,
      packed H2D memcpy (Σn·r bytes) + unpack       — ADT, two steps,
      zero-copy unpack reading mapped pinned memory — ADT, one kernel (K5).
    The host packed stream is the device pack's output copied to pinned
    memory beforehand (setup, untimed)."""
    import torch
    from paper_2004_02297_b200 import engine
    lay = sync.layout
    host_packed = torch.empty(lay.nbytes, dtype=torch.uint8, pin_memory=True)
    host_packed.copy_(sync.packed[:lay.nbytes])
    dev_packed = torch.empty(lay.nbytes, dtype=torch.uint8, device=sync.device)
    # the FP32 baseline gets the same advantage as the packed stream: one
    # contiguous pinned buffer, one copy (not one copy per layer)
    host_fp32 = torch.cat([m.reshape(-1) for m in sync.masters]).cpu().pin_memory()
    dev_fp32 = torch.empty_like(host_fp32, device=sync.device)
    table = engine.SegmentTable(sync.replicas, lay)

    def raw():
        dev_fp32.copy_(host_fp32, non_blocking=True)

    def copy_unpack():
        dev_packed.copy_(host_packed, non_blocking=True)
        engine.unpack(table, dev_packed)

    def zero_copy():
        engine.unpack(table, host_packed)

    t_raw, t_cu, t_zc = _time_ms(raw, reps), _time_ms(copy_unpack, reps), _time_ms(zero_copy, reps)
    raw_b, pk_b = lay.raw_bytes, lay.total_payload_bytes
    return {"raw_fp32_ms": t_raw, "adt_copy_unpack_ms": t_cu, "adt_zero_copy_unpack_ms": t_zc,
            "raw_fp32_GBps": raw_b / t_raw / 1e6, "packed_bytes": pk_b, "raw_bytes": raw_b,
            "payload_ratio": raw_b / pk_b, "speedup_vs_fp32": t_raw / min(t_cu, t_zc)}


def run_sgd_compare(dev_masters, rs, dev, reps=20):
    """momentum-SGD step fused with pack + norm (adt_sgd_pack,
    one pass: read W, v, g; write W, v, packed) vs the unfused sequence
    (the same update as four in-place torch kernels, then adt_pack with the
    norm). Algorithmic bytes per weight: fused 20 + r; unfused 24 + r."""
    import torch
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.layout import PackedLayout
    lay = PackedLayout.plan([m.numel() for m in dev_masters], rs)
    w = [m.clone() for m in dev_masters]
    v = [torch.zeros_like(m) for m in dev_masters]
    g = [torch.randn_like(m) * 0.01 for m in dev_masters]
    packed = torch.empty(lay.nbytes, dtype=torch.uint8, device=dev)
    ss = torch.empty(len(w), dtype=torch.float64, device=dev)
    fused_t = engine.SgdTable(w, v, g, lay)
    pack_t = engine.SegmentTable(w, lay)
    lr, mu, wd = 1e-4, 0.9, 5e-4

    def fused():
        engine.sgd_pack(fused_t, lr, mu, wd, packed, ss)

    def unfused():
        for wi, vi, gi in zip(w, v, g):
            gi2 = gi.add(wi, alpha=wd)   # g + wd*W (alpha-scaled add)
            vi.mul_(mu).add_(gi2)
            wi.sub_(vi, alpha=lr)
        engine.pack(pack_t, packed, ss)

    tf, tu = _time_ms(fused, reps), _time_ms(unfused, reps)
    n = sum(lay.counts)
    pb = lay.total_payload_bytes
    return {"fused_ms": tf, "unfused_ms": tu, "speedup": tu / tf,
            "fused_GBps": (20 * n + pb) / (tf * 1e-3) / 1e9,
            "note": "fused: adt_sgd_pack (update + pack + norm, 20+r B/weight); unfused: torch in-place update "
                    "kernels + adt_pack"}


def run_awp_step(dev_masters, steps=200):
    """Wall-clock cost of one full AWP step through the public API
    (WeightSync.step: pack + fused norm, unpack, observe, re-pack on
    escalation) on this weight set: the AWP decision on the host (one 8·L-byte
    read + Python Algorithm 1 per step) vs on the device (awp_on_device=True:
    one graph replay per step, trace rows drained at the end)."""
    import torch
    import paper_2004_02297_b200 as adt
    L = len(dev_masters)
    cfg = adt.PrecisionConfig(threshold=-2e-3, interval=50, step_bits=8, initial_bits=8)
    out = {}
    for name, on_dev in (("host_controller_us", False), ("device_controller_us", True)):
        masters = [m.clone() for m in dev_masters]
        sync = adt.WeightSync(masters, adt.PrecisionController(L, cfg), awp_on_device=on_dev)
        for b in range(10):
            sync.step(batch=b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(10, 10 + steps):
            sync.step(batch=b)
        if on_dev:
            sync.drain_trace()
        torch.cuda.synchronize()
        out[name] = (time.perf_counter() - t0) / steps * 1e6
        del sync, masters
    out["note"] = "WeightSync.step wall time per step (widths start at 8 bits; interval 50)"
    return out


def run_reduce_compare(dev_masters, rs, dev, nc=8, reps=10):
    """SURVEY §8f #4, gradient return path: `nc` worker gradient buckets are
    combined as net.gather_and_update does (sample-count weights, pairwise
    tree, / total), the momentum step applied, the new masters packed + normed
    — one adt_reduce_sgd_pack pass (reads (4·nc + 8)·n, writes (8 + r)·n) — vs
    the unfused sequence: torch weighted pairwise sum + divide, the update as
    in-place torch kernels, then adt_pack with the norm. On one GPU the
    buckets are local; at N > 1 the same kernel reads peers' buckets over
    NVLink (ShardedWeightSync.update, transport p2p)."""
    import torch
    from paper_2004_02297_b200 import engine
    from paper_2004_02297_b200.grads import GradBucket
    from paper_2004_02297_b200.layout import PackedLayout
    counts = [m.numel() for m in dev_masters]
    lay = PackedLayout.plan(counts, rs)
    w = [m.clone() for m in dev_masters]
    v = [torch.zeros_like(m) for m in dev_masters]
    buckets = []
    for c in range(nc):
        b = GradBucket(counts, dev, sample_count=32 + c)
        b.flat.normal_(0.0, 0.01)
        buckets.append(b)
    packed = torch.empty(lay.nbytes, dtype=torch.uint8, device=dev)
    ss = torch.empty(len(w), dtype=torch.float64, device=dev)
    table = engine.ReduceSgdTable(w, v, [buckets[0].byte_offset(l) for l in range(len(w))], lay)
    pack_t = engine.SegmentTable(w, lay)
    ptrs = [b.flat.data_ptr() for b in buckets]
    sc = [b.sample_count for b in buckets]
    lr, mu, wd = 1e-4, 0.9, 5e-4
    total = float(sum(sc))

    def fused():
        engine.reduce_sgd_pack(table, ptrs, sc, lr, mu, wd, packed, ss)

    def unfused():
        level = [b.flat * float(b.sample_count) for b in buckets]
        while len(level) > 1:                     # the reference's pairwise association
            carry = level[-1:] if len(level) % 2 else []
            level = [a + b for a, b in zip(level[0::2], level[1::2])] + carry
        g = level[0].div_(total)
        for l, (wi, vi) in enumerate(zip(w, v)):
            gi = g[buckets[0].offsets[l]:buckets[0].offsets[l] + counts[l]]
            gi.add_(wi, alpha=wd)
            vi.mul_(mu).add_(gi)
            wi.sub_(vi, alpha=lr)
        engine.pack(pack_t, packed, ss)

    tf, tu = _time_ms(fused, reps), _time_ms(unfused, reps)
    n = sum(counts)
    pb = lay.total_payload_bytes
    alg = (4 * nc + 16) * n + pb
    return {"contributions": nc, "fused_ms": tf, "unfused_ms": tu, "speedup": tu / tf,
            "fused_GBps": alg / (tf * 1e-3) / 1e9, "algorithmic_bytes": alg,
            "note": "fused: adt_reduce_sgd_pack ((4*nc+16)*n + sum(n*r) B); unfused: torch weighted pairwise "
                    "sum + div + in-place update kernels + adt_pack"}


def run_dp_update(sync, counts, world, dev, backend, reps=10):
    """N > 1, the whole data-parallel step through ShardedWeightSync.update:
    every rank's FP32 gradient bucket -> fused [gather this rank's shard of
    all buckets (p2p: peer loads over NVLink; nccl: all_to_all) + weighted
    pairwise combine + momentum step + pack + norm] -> packed all-gather ->
    unpack -> AWP observe (one 8·L-byte norm read per step). Baseline: the
    uncompressed DDP step — all_reduce of the FP32 bucket, the momentum update
    of the full masters as torch kernels (every rank), no weight exchange.
    Device ms per step, max over ranks (nccl only: gloo timings are not
    meaningful)."""
    import torch
    import torch.distributed as dist
    from paper_2004_02297_b200.grads import GradBucket
    bucket = GradBucket(counts, dev)
    bucket.flat.normal_(0.0, 0.01)
    sc = [64] * world
    lr, mu, wd = 1e-5, 0.9, 5e-4

    def ours():
        sync.update(bucket, sc, lr, mu, wd)

    w = [torch.zeros(n, device=dev) for n in counts]
    v = [torch.zeros(n, device=dev) for n in counts]

    def ddp():
        dist.all_reduce(bucket.flat)
        for l, (wi, vi) in enumerate(zip(w, v)):
            g = bucket.views[l].reshape(-1).div(float(sum(sc)))
            g.add_(wi, alpha=wd)
            vi.mul_(mu).add_(g)
            wi.sub_(vi, alpha=lr)

    t_ours = _time_ms(ours, reps)
    t_ddp = _time_ms(ddp, reps) if backend == "nccl" else None
    if backend != "nccl":
        return {"ms": None, "note": "gloo test hook: exercised, not timed"}
    t = torch.tensor([t_ours, t_ddp], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    a, b = (float(x) for x in t.tolist())
    return {"ms": a, "fp32_ddp_ms": b, "speedup": b / a, "transport": sync.transport,
            "note": "ShardedWeightSync.update (fused reduce+SGD+pack, packed gather, unpack, AWP observe) vs "
                    "FP32 all_reduce + torch momentum step; device ms per step, max over ranks"}


def run_fp32_sync(sync, masters, replicas, K, dev, backend, args):
    """The N > 1 baseline on the SAME transport: ShardedWeightSync at 32 bits
    (r = 4: the packed stream is the FP32 words, byte-swapped) — the raw
    FP32 weight exchange through the same pack / barrier / gather-unpack
    kernels. Device ms per step (K steps between two events), max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2004_02297_b200.precision import FixedPrecision
    from paper_2004_02297_b200.sharded import ShardedWeightSync
    full = ShardedWeightSync(masters, FixedPrecision(len(masters), 32), replicas, transport=sync.transport)
    for _ in range(args.warmup):
        full.launch_graphed(True)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        full.launch_graphed(True)
    b.record()
    b.synchronize()
    if hasattr(full, "check_barrier"):
        full.check_barrier()
    t = torch.tensor([a.elapsed_time(b) / K], device=dev if backend == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del full
    return float(t.item())


def run_fp32_allgather(counts, world, dev, reps=20):
    """Baseline at N > 1: ncclAllGather of the raw FP32 weights (4n bytes)."""
    import torch
    import torch.distributed as dist
    per = -(-4 * sum(counts) // world)
    per = (per + 15) // 16 * 16
    send = torch.empty(per, dtype=torch.uint8, device=dev)
    recv = torch.empty(per * world, dtype=torch.uint8, device=dev)
    ms = _time_ms(lambda: dist.all_gather_into_tensor(recv, send), reps)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"ms": ms, "bytes_per_rank": per, "busbw_GBps": per * (world - 1) / (ms * 1e-3) / 1e9}


def run_e2e(args, dev_masters, rs, dev):
    """Same metric through the reference-facing drop-in API with HOST buffers —
    the calls the reference arm times (weightpack codec.pack_vectorized /
    unpack, precision.l2_norm), layer by layer on NumPy arrays: every step
    copies each layer host->device for pack, the payload bytes back
    (PackedBlock.payload is `bytes`), the payload host->device for unpack, the
    FP32 words back (a NumPy array), and the layer again for l2_norm."""
    import torch
    import paper_2004_02297_b200 as adt
    host = [m.cpu().numpy() for m in dev_masters]

    def one():
        for w, r in zip(host, rs):
            blk = adt.pack_vectorized(w, r)
            adt.unpack(blk)
            adt.l2_norm(w)

    one()
    steps = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    n = [w.size for w in host]
    byts = 2 * sum((4 + r) * k for k, r in zip(n, rs))
    h2d = sum(4 * k + r * k + 4 * k for k, r in zip(n, rs))
    d2h = sum(r * k + 4 * k for k, r in zip(n, rs))
    return {"value": byts / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": steps,
            "note": "drop-in per-layer pack_vectorized + unpack + l2_norm on host NumPy arrays; wall clock"}


def run_e2e_sharded(args, sync, counts, rs, dev, backend, flat_masters):
    """N > 1 end to end through ShardedWeightSync: every step each rank copies
    the FP32 master range it owns from pinned host memory (the paper's CPU
    masters, sharded; one contiguous copy of its slice of the flat master
    store), runs the step (pack with the norm, exchange, gather-unpack of
    every replica) and reads the per-layer norms back (the AWP input). Wall
    time per step, max over ranks; value = the whole job's algorithmic bytes
    per step / time, as the device-timed value."""
    import torch
    import torch.distributed as dist
    b0, b1 = sync.grad_ranges[sync.rank]       # this rank's pieces, contiguous in the flat store
    dev_slice = flat_masters[b0:b1]
    host = dev_slice.cpu().pin_memory()
    h2d = host.numel() * 4
    world = sync.world

    def one():
        dev_slice.copy_(host, non_blocking=True)
        sync.launch_graphed(True)
        sync._norms()                      # D2H of the gathered norm tails + host sync

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    t = torch.tensor([dt, float(h2d)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dt = float(tmax[0].item())
    byts = sum((4 + r) * n for n, r in zip(counts, rs)) * (1 + world)
    return {"value": byts / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(t[1].item()),
            "d2h_bytes_per_step": 8 * world * sync.plan.max_pieces * world, "ms_per_step": dt * 1e3,
            "note": "ShardedWeightSync from pinned host FP32 master shards; wall clock, max over ranks"}


def run_e2e_host_master(args, host, rs, dev, steps=20):
    """The paper's CPU-master setting end to end through the public API
    (hostsync.HostWeightSync): per step the FP32 masters in
    host memory are packed on the host cores with their norms fused
    (adt_pack_host, AVX-512), the packed stream crosses PCIe in copies that
    start while later units are still being packed, and the GPU unpacks it
    into the replicas; the step ends when the replicas are complete (stream
    sync). The norms (the AWP input) come out of the host pass: nothing is
    read back from the device. Wall clock per step."""
    import torch
    import paper_2004_02297_b200 as adt
    from paper_2004_02297_b200.hostsync import host_threads
    from paper_2004_02297_b200.precision import FixedPrecision

    class Fixed(FixedPrecision):
        def round_tos(self):
            return list(rs)

    import numpy as np
    # The masters live in page-locked host memory, as a CPU-master trainer
    # allocates them (torch pin_memory): full-width layers then go to the GPU by
    # DMA straight from the masters (HostWeightSync direct_full, the default).
    pinned = []
    for h in host:
        t = torch.empty(h.size, dtype=torch.float32, pin_memory=True)
        t.numpy()[:] = h
        pinned.append(t.numpy())
    stream = torch.cuda.current_stream(dev)

    tuned = {}

    def measure(direct_full):
        sync = adt.HostWeightSync(pinned, Fixed(len(host), 32), device=dev, direct_full=direct_full)
        if direct_full:                              # setup (untimed): packer threads + copy batch for this set/host
            tuned["timings_ms"] = {k: v * 1e3 for k, v in sync.tune().items()}
            tuned["threads"], tuned["batch"] = sync.threads, sync.min_copy_bytes
        else:
            sync.threads, sync.min_copy_bytes = tuned.get("threads", 0), tuned.get("batch", 0)
        # the step's result lives on the GPU (the replicas): each step reads back the
        # last 4 words of the last replica (16 B D2H, which also completes the step)
        # and checks them against the host masters truncated to their width
        tail_dev = sync.replicas[-1][-4:]
        tail_host = torch.empty(4, dtype=torch.float32, pin_memory=True)
        want = (host[-1][-4:].view(np.uint32) & np.uint32((0xFFFFFFFF << (8 * (4 - rs[-1]))) & 0xFFFFFFFF))

        def one():
            sync.launch(fused_norm=True)
            tail_host.copy_(tail_dev, non_blocking=True)
            stream.synchronize()
            if not np.array_equal(tail_host.numpy().view(np.uint32), want):
                raise AssertionError("host-master e2e: the replica read back differs from the packed masters")

        for _ in range(3):
            one()
        n_steps = max(args.e2e_steps, steps)
        t0 = time.perf_counter()
        for _ in range(n_steps):
            one()
        dt = (time.perf_counter() - t0) / n_steps
        ndirect = int(sync.direct[:len(host)].sum())
        h2d = sync.h2d_bytes
        if direct_full:
            # the pipeline's two legs alone (best of 5, wall clock): the host pass (adt_pack_host
            # of the layers the packer handles, the tuned thread count) and the DMA of the link
            # bytes (the staging stream, direct layers' spans included); the step cannot beat
            # the slower one, and both share host DRAM
            from paper_2004_02297_b200 import _lib
            lib = _lib.load()
            L = len(host)
            segs = _lib.segment_array([(sync._host_segs[i].weights, 0 if sync.direct[i] else sync._host_segs[i].count,
                                        sync._host_segs[i].offset, sync._host_segs[i].round_to) for i in range(L)])
            nb = sync.layout.nbytes
            base = sync._stage_ptr - sync.staging.data_ptr()

            def best(fn, k=5):
                fn()
                b = float("inf")
                for _ in range(k):
                    t1 = time.perf_counter()
                    fn()
                    b = min(b, time.perf_counter() - t1)
                return b

            def pack_leg():
                _lib.check(lib.adt_pack_host(segs, L, sync._stage_ptr, sync._sumsq_ptr, sync.threads))

            def dma_leg():
                sync.packed[:nb].copy_(sync.staging[base:base + nb], non_blocking=True)
                stream.synchronize()

            tuned["legs_ms"] = {"host_pack": best(pack_leg) * 1e3, "dma": best(dma_leg) * 1e3}
            # host DRAM bytes a step moves (both legs share it): masters read by the packer,
            # staging written (non-temporal) and read again by the DMA, direct layers read by the DMA
            tuned["host_dram_bytes"] = sum(
                4 * sync._host_segs[i].count if sync.direct[i]
                else (4 + 2 * sync._host_segs[i].round_to) * sync._host_segs[i].count for i in range(L))
        del sync
        return dt, n_steps, ndirect, h2d

    dt, n_steps, ndirect, h2d = measure(True)
    dt_packed, _, _, _ = measure(False) if ndirect else (dt, 0, 0, 0)
    # the uncompressed alternative timed the same way (wall clock, same read-back
    # and sync): the same masters as ONE contiguous pinned FP32 buffer, one copy
    flat = torch.empty(sum(h.size for h in host), dtype=torch.float32, pin_memory=True)
    dflat = torch.empty(flat.numel(), dtype=torch.float32, device=dev)
    tail_raw = torch.empty(4, dtype=torch.float32, pin_memory=True)

    flat.numpy()[-4:] = host[-1][-4:]
    want_raw = host[-1][-4:].view(np.uint32)

    def raw_one():                                   # same read-back and check as one()
        dflat.copy_(flat, non_blocking=True)
        tail_raw.copy_(dflat[-4:], non_blocking=True)
        stream.synchronize()
        if not np.array_equal(tail_raw.numpy().view(np.uint32), want_raw):
            raise AssertionError("raw FP32 e2e: read-back differs")

    for _ in range(3):
        raw_one()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        raw_one()
    dt_raw = (time.perf_counter() - t0) / n_steps
    del flat, dflat
    # the same host arrays as one raw FP32 pinned copy would move: the baseline
    n = sum(h.size for h in host)
    byts = 2 * sum((4 + r) * h.size for h, r in zip(host, rs))
    return {"value": byts / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 16,
            "ms_per_step": dt * 1e3, "steps": n_steps, "host_threads": tuned.get("threads") or host_threads(),
            "host_threads_available": host_threads(), "copy_batch_bytes": tuned.get("batch"),
            "legs_ms": tuned.get("legs_ms"), "host_dram_bytes_per_step": tuned.get("host_dram_bytes"),
            "host_dram_GBps": (tuned["host_dram_bytes"] / dt / 1e9) if tuned.get("host_dram_bytes") else None,
            "frac_of_legs_floor": (max(tuned["legs_ms"].values()) / (dt * 1e3)) if tuned.get("legs_ms") else None,
            "tuning_ms": tuned.get("timings_ms"),
            "raw_fp32_bytes": 4 * n, "raw_fp32_wall_ms_per_step": dt_raw * 1e3, "vs_raw_fp32": dt_raw / dt,
            "direct_full_layers": ndirect, "all_packed_ms_per_step": dt_packed * 1e3,
            "note": "HostWeightSync: pinned host FP32 masters -> adt_pack_host (host_threads cores and the copy batch "
                    "picked at setup by HostWeightSync.tune; norms fused) -> "
                    "packed H2D overlapped with the packing -> adt_unpack; full-width layers DMA'd straight from "
                    "the masters (direct_full); 16 B read-back check; wall clock; the norms come from the host pass"}


def run_e2e_weightsync(args, dev_masters, rs, dev):
    """WeightSync from pinned host FP32 masters: per step H2D of the masters,
    pack (norm fused) + unpack on device, D2H of the L float64 sums. The
    masters live in one flat buffer (layers at 16-B aligned offsets, as a
    flat parameter store keeps them), so the step's H2D is one copy rather
    than one per layer (161 for ResNet-50)."""
    import torch
    import paper_2004_02297_b200 as adt
    from paper_2004_02297_b200.grads import bucket_offsets
    from paper_2004_02297_b200.precision import FixedPrecision
    counts = [m.numel() for m in dev_masters]
    offs, total = bucket_offsets(counts)
    flat_host = torch.zeros(max(total, 4), dtype=torch.float32).pin_memory()
    flat_dev = torch.empty_like(flat_host, device=dev)
    for o, n, m in zip(offs, counts, dev_masters):
        flat_host[o:o + n].copy_(m.reshape(-1).cpu())
    masters = [flat_dev[o:o + n] for o, n in zip(offs, counts)]

    class Fixed(FixedPrecision):
        def round_tos(self):
            return list(rs)

    sync = adt.WeightSync(masters, Fixed(len(masters), 32))
    h2d = flat_host.numel() * 4
    d2h = 8 * len(masters)

    def one():
        flat_dev.copy_(flat_host, non_blocking=True)
        sync.launch_graphed(fused_norm=True)   # the step's CUDA graph (as WeightSync.step)
        sync.read_norms()                      # D2H of the L float64 sums + host sync

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    steps = max(args.e2e_steps, 20)            # the host link is noisy: >= 20 steps
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    byts = sync.layout.roundtrip_bytes()
    return {"value": byts / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": steps,
            "note": "WeightSync from pinned host FP32 masters (one flat buffer, one H2D per step); wall clock"}


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        main_reference(a)
    else:
        main_ours(a)
