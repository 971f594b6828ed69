#!/usr/bin/env python
"""Render BASELINE.md §4's table from a directory of bench JSON lines.

    python scripts/results_table.py gpurun_out/r01c
"""
import json
import os
import sys

ORDER = [("bench_lenet.json", "LeNet r=1 (430,500 w)"), ("bench.json", "**AlexNet 8/16/24/32/8/16/24/32 bits**"),
         ("bench_vgg16.json", "VGG-16 r=1"), ("bench_resnet50.json", "ResNet-50, 161 tensors, r=1"),
         ("bench_1b_8.json", "1B synthetic r=1"), ("bench_1b_16.json", "1B synthetic r=2"),
         ("bench_1b_24.json", "1B synthetic r=3"), ("bench_1b_32.json", "1B synthetic r=4")]


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        try:
            return json.loads(line)
        except Exception:
            continue
    return None


def main(d):
    print("| Config | Round trip GB/s (% of measured copy peak) | step µs | pack GB/s | unpack GB/s | e2e GB/s (pinned host masters) "
          "| pinned H2D: ADT vs raw FP32 | clocks |")
    print("|---|---|---|---|---|---|---|---|")
    for f, name in ORDER:
        p = os.path.join(d, f)
        if not os.path.exists(p):
            continue
        j = last_json(p)
        r = j.get("roofline") or {}
        h = j.get("host_to_device") or {}
        e = j.get("e2e") or {}
        c = j.get("clocks") or {}
        pct = 100 * j["value"] / ((j.get("roofline") or {}).get("peak") or 6533.2)
        print(f"| {name} | {j['value']:.0f} ({pct:.1f} %) | {j['ms_per_step'] * 1e3:.1f} | {r.get('pack_GBps', 0):.0f} | "
              f"{r.get('unpack_GBps', 0):.0f} | {e.get('value', 0):.1f} | {h.get('speedup_vs_fp32', 0):.2f}× | "
              f"{c.get('sm_mhz')} MHz {','.join(c.get('reasons') or []) or 'no throttle'} |")


if __name__ == "__main__":
    main(sys.argv[1])
