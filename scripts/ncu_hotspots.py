#!/usr/bin/env python
"""Warp-stall hotspots of one kernel from an ncu --set full report captured
with --import-source on: stall reasons summed over the kernel, and the SASS
instructions holding the most samples.

    python scripts/ncu_hotspots.py gpurun_out/r01i/prof_alexnet.ncu-rep adt_pack [top]
"""

import csv
import io
import subprocess
import sys


def hotspots(rep, kernel, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kernel}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    # the page may repeat per launch; keep the first kernel block
    name = lines[0].split(",", 1)[1].strip('",') if lines else kernel
    body = []
    for ln in lines[1:]:
        if ln.startswith('"Kernel Name"'):
            break
        body.append(ln)
    rows = list(csv.DictReader(io.StringIO("\n".join(body))))
    if not rows:
        return f"no source rows for {kernel} in {rep}\n"
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(int(r[c] or 0) for r in rows) for c in stall_cols}
    samples = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    md = [f"## `{name}`\n", f"{len(rows)} SASS instructions, {samples} warp-stall samples.\n",
          "| stall reason | samples | share |", "|---|---|---|"]
    for c, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if v:
            md.append(f"| {c[6:]} | {v} | {v / max(1, samples):.1%} |")
    md += ["", "| SASS | samples | share | top reason |", "|---|---|---|---|"]
    for r in sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        reason = max(stall_cols, key=lambda c: int(r[c] or 0))
        md.append(f"| `{r['Source'].strip()}` | {s} | {s / max(1, samples):.1%} | {reason[6:]} |")
    return "\n".join(md) + "\n"


if __name__ == "__main__":
    print(hotspots(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 12))
