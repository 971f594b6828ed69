#!/usr/bin/env python
"""Render BASELINE.md §4's table from a directory of bench JSON lines.

    python scripts/results_table.py gpurun_out/r02i
"""
import json
import os
import sys

ORDER = [("bench_lenet.json", "LeNet r=1 (430,500 w)"), ("bench.json", "**AlexNet 8/16/24/32/8/16/24/32 bits**"),
         ("bench_vgg16.json", "VGG-16 r=1"), ("bench_vgg16_8.json", "VGG-16 r=1"),
         ("bench_vgg16_16.json", "VGG-16 r=2"), ("bench_vgg16_24.json", "VGG-16 r=3"),
         ("bench_vgg16_32.json", "VGG-16 r=4"), ("bench_resnet50.json", "ResNet-50, 161 tensors, r=1"),
         ("bench_1b_8.json", "1B synthetic r=1"), ("bench_1b_16.json", "1B synthetic r=2"),
         ("bench_1b_24.json", "1B synthetic r=3"), ("bench_1b_32.json", "1B synthetic r=4")]


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        try:
            return json.loads(line)
        except Exception:
            continue
    return None


def f3(x):
    return f"{x:.2f}" if isinstance(x, (int, float)) else "—"


def main(d):
    print("| Config | Round trip GB/s (% of measured copy peak) | step µs | cold pack / unpack (frac of copy peak) "
          "| cold vs size-matched copy | e2e GB/s (host masters) · ms | e2e vs raw FP32 H2D (wall clock) | clocks |")
    print("|---|---|---|---|---|---|---|---|")
    for f, name in ORDER:
        p = os.path.join(d, f)
        if not os.path.exists(p):
            continue
        j = last_json(p)
        if j is None:
            continue
        r = j.get("roofline") or {}
        cold = r.get("cold") or {}
        h = j.get("host_to_device") or {}
        e = j.get("e2e") or {}
        c = j.get("clocks") or {}
        pct = 100 * j["value"] / (r.get("peak") or 6538.3)
        raw = e.get("raw_fp32_wall_ms_per_step") or h.get("raw_fp32_ms")   # wall clock like e2e when present
        e_ms = e.get("ms_per_step")
        vs_raw = f"{raw / e_ms:.2f}×" if raw and e_ms else "—"
        cold_s = (f"{f3(cold.get('pack_frac'))} / {f3(cold.get('unpack_frac'))}" if "pack_frac" in cold
                  else "— (fits in L2)")
        print(f"| {name} | {j['value']:.0f} ({pct:.1f} %) | {j['ms_per_step'] * 1e3:.1f} | {cold_s} | "
              f"{f3(cold.get('frac_of_size_matched_copy'))} | {e.get('value', 0):.1f} · {f3(e_ms)} | {vs_raw} | "
              f"{c.get('sm_mhz')} MHz {','.join(c.get('reasons') or []) or 'no throttle'} |")


if __name__ == "__main__":
    main(sys.argv[1])
