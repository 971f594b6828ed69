#!/bin/bash
# Copy one evidence pass (gpurun_out/<tag>, from scripts/gpu_full.sh or gpu_r02.sh) into the
# tracked profiles/: bench lines, ncu summaries, launch lists, traffic table, Table-2, step
# overhead, host probes. Files a pass did not produce are skipped.
# usage: bash scripts/refresh_profiles.sh <tag> [round-prefix, default r02]
set -e
O=gpurun_out/$1
P=${2:-r02}
have() { [ -s "$1" ]; }
for j in $O/bench*.json; do
  f=$(basename $j .json)
  python - "$j" "profiles/${P}_$f.json" <<'PY'
import json, sys
line = None
for l in open(sys.argv[1]):
    try:
        line = json.loads(l)
    except Exception:
        pass
if line is not None:
    json.dump(line, open(sys.argv[2], "w")); open(sys.argv[2], "a").write("\n")
PY
done
have $O/launches.csv && python scripts/ncu_summary.py launches $O/launches.csv > profiles/${P}_alexnet_launches.md
have $O/launches_resnet50.csv && python scripts/ncu_summary.py launches $O/launches_resnet50.csv > profiles/${P}_resnet50_launches.md
have $O/launches_awp_device.csv && python scripts/ncu_summary.py launches $O/launches_awp_device.csv > profiles/${P}_awp_device_launches.md
for k in alexnet resnet50 sgd reduce vgg16_r1 vgg16_r2 vgg16_r3; do
  have $O/prof_$k.ncu-rep && python scripts/ncu_summary.py report $O/prof_$k.ncu-rep > profiles/${P}_${k}_ncu_full.md
done
have $O/prof_alexnet.ncu-rep && python scripts/ncu_summary.py traffic $O/prof_alexnet.ncu-rep alexnet > /dev/null
have $O/prof_resnet50.ncu-rep && python scripts/ncu_summary.py traffic $O/prof_resnet50.ncu-rep resnet50 > /dev/null
have $O/table2.md && cp $O/table2.md profiles/${P}_table2.md
have $O/nvsmi.txt && cp $O/nvsmi.txt profiles/${P}_nvsmi.txt
have $O/step_overhead.txt && cp $O/step_overhead.txt profiles/${P}_step_overhead.txt
have $O/host_probe.txt && cp $O/host_probe.txt profiles/${P}_host_probe.txt
have $O/small_step.txt && cp $O/small_step.txt profiles/${P}_small_step.txt
have $O/pytest_gpu.log && tail -n 30 $O/pytest_gpu.log > profiles/${P}_pytest_gpu_tail.txt
for t in memcheck racecheck synccheck; do
  have $O/sanitize_$t.log && tail -n 3 $O/sanitize_$t.log > profiles/${P}_sanitize_$t.txt
done
python scripts/results_table.py $O > profiles/${P}_results_table.md || true
have $O/refsuite_plug.txt && { echo "# the reference's whole test suite on the unmodified reference package with codec + precision replaced by this repo (tests/refsuite/run.py --plug)"; cat $O/refsuite_plug.txt; } > profiles/${P}_reference_suite_plugged.txt
have $O/small_host_breakdown.txt && cp $O/small_host_breakdown.txt profiles/${P}_small_host_breakdown.txt
true
