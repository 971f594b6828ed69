#!/bin/bash
# Fused gradient combine + SGD + pack over contribution counts (AlexNet set):
# fused vs unfused device time. usage: bash scripts/reduce_sweep.sh <outdir>
OUT=${1:-gpurun_out/reduce_sweep}; mkdir -p $OUT
echo "| contributions | fused µs | unfused µs | fused GB/s | % of copy peak | speedup |"
echo "|---|---|---|---|---|---|"
for k in ${KS:-1 2 3 4 5 6 7 8 9 10 11 12 13 14 15 16}; do
  timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-awp-step --quiet-extra --reduce-contribs $k > $OUT/red_$k.json 2>/dev/null
  python - $OUT/red_$k.json <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
r, peak = d["fused_reduce_sgd_pack"], json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
print(f"| {r['contributions']} | {r['fused_ms'] * 1e3:.1f} | {r['unfused_ms'] * 1e3:.1f} | {r['fused_GBps']:.0f} | "
      f"{100 * r['fused_GBps'] / peak:.1f} % | {r['speedup']:.2f}x |")
PY
done
