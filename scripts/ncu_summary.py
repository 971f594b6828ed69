#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV for profiles/.

    python scripts/ncu_summary.py report gpurun_out/x/prof.ncu-rep > profiles/...md
    python scripts/ncu_summary.py launches gpurun_out/x/launches.csv
    python scripts/ncu_summary.py traffic gpurun_out/x/prof.ncu-rep alexnet   # -> profiles/ncu_traffic.json
"""

import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occ limit (smem)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio", "stall long scoreboard"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def report(rep):
    hdr, units, rows = raw_rows(rep)
    print(f"# ncu --set full summary: `{os.path.basename(rep)}`\n")
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        print(f"## {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")
        try:
            rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
            wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
            t = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            tu = units[hdr.index("gpu__time_duration.sum")]
            t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-6)
            print(f"\nDRAM traffic {(rd + wr) / 1e6:.1f} MB per launch; DRAM GB/s under ncu (cold, serialised) "
                  f"{(rd + wr) / t_s / 1e9:.0f}\n")
        except Exception:
            pass


def traffic(rep, config):
    hdr, units, rows = raw_rows(rep)
    res = {}
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        short = ("adt_unpack_kernel" if "unpack" in name else
                 "adt_norm_finalize_kernel" if "finalize" in name else "adt_pack_kernel")
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        res[short] = rd + wr
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    d = {}
    if os.path.exists(path):
        d = json.load(open(path))
    d[config] = res
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d))


def launches(path):
    """Launch list: per kernel, launches, mean duration and share of the total;
    when the capture also holds dram__bytes_read/write.sum, the mean DRAM bytes
    per launch. Then each adt_ kernel's share of one step."""
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    ii = hdr.index("ID") if "ID" in hdr else None
    dur, rd, wr = {}, {}, {}
    dur_unit = "ns"
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0]
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        v = float(r[vi].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            dur.setdefault(k, []).append(v)
            dur_unit = r[ui]
        elif metric == "dram__bytes_read.sum":
            rd.setdefault(k, []).append(v * _SCALE.get(r[ui], 1.0))
        elif metric == "dram__bytes_write.sum":
            wr.setdefault(k, []).append(v * _SCALE.get(r[ui], 1.0))
    all_t = sum(sum(v) for v in dur.values())
    has_dram = bool(rd)
    extra_h = " DRAM read MB / launch | DRAM write MB / launch |" if has_dram else ""
    print(f"| kernel | launches | mean duration | total share |{extra_h}\n|---|---|---|---|" + ("---|---|" if has_dram else ""))
    for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        extra = ""
        if has_dram:
            r_ = rd.get(k, [0.0])
            w_ = wr.get(k, [0.0])
            extra = f" {sum(r_) / len(r_) / 1e6:.1f} | {sum(w_) / len(w_) / 1e6:.1f} |"
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} {dur_unit} | {sum(v) / all_t:.1%} |{extra}")
    # the ADT step alone (the process also launches setup kernels: input
    # generation, the L2-flush read): each adt_ kernel's share of the step
    adt = {k: v for k, v in dur.items() if "adt_" in k}
    step = sum(sum(v) / len(v) for v in adt.values())
    if adt:
        print("\nShare of one step (mean launch time of each adt_ kernel / their sum; ncu serialises launches, "
              "so the side-stream finalize is counted as if it ran alone):\n")
        print("| kernel | mean duration | share of step |\n|---|---|---|")
        for k, v in sorted(adt.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
            m = sum(v) / len(v)
            print(f"| `{k}` | {m:.2f} {dur_unit} | {m / step:.1%} |")


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2])
