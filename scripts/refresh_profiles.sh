#!/bin/bash
# Copy one gpu_full.sh run (gpurun_out/<tag>) into the tracked profiles/: bench lines,
# ncu summaries, launch lists, traffic table, Table-2, bench-codec, step overhead, training runs.
# usage: bash scripts/refresh_profiles.sh r01g
set -e
O=gpurun_out/$1
for f in bench bench_1b_16 bench_1b_24 bench_1b_32 bench_1b_8 bench_lenet bench_resnet50 bench_vgg16 bench_reference; do
  python - "$O/$f.json" "profiles/r01_$f.json" <<'PY'
import json, sys
line = None
for l in open(sys.argv[1]):
    try:
        line = json.loads(l)
    except Exception:
        pass
json.dump(line, open(sys.argv[2], "w")); open(sys.argv[2], "a").write("\n")
PY
done
python scripts/ncu_summary.py launches $O/launches.csv > profiles/r01_alexnet_launches.md
python scripts/ncu_summary.py launches $O/launches_resnet50.csv > profiles/r01_resnet50_launches.md
python scripts/ncu_summary.py launches $O/launches_awp_device.csv > profiles/r01_awp_device_launches.md
python scripts/ncu_summary.py report $O/prof_alexnet.ncu-rep > profiles/r01_alexnet_ncu_full.md
python scripts/ncu_summary.py report $O/prof_resnet50.ncu-rep > profiles/r01_resnet50_ncu_full.md
python scripts/ncu_summary.py report $O/prof_sgd.ncu-rep > profiles/r01_sgd_ncu_full.md
python scripts/ncu_summary.py report $O/prof_reduce.ncu-rep > profiles/r01_reduce_ncu_full.md
python scripts/ncu_summary.py traffic $O/prof_alexnet.ncu-rep alexnet > /dev/null
python scripts/ncu_summary.py traffic $O/prof_resnet50.ncu-rep resnet50 > /dev/null
cp $O/table2.md profiles/r01_table2.md
cp $O/nvsmi.txt profiles/r01_nvsmi.txt
tail -n 1 $O/bench_n2_gloo_p2p.log > profiles/r01_bench_n2_gloo_p2p.json
python scripts/results_table.py $O > profiles/r01_results_table.md
cp $O/step_overhead.txt profiles/r01_step_overhead.txt
cat $O/train_fp32.json $O/train_awp.json $O/train_awp_device.json > profiles/r01_train_example.jsonl
cp $O/reduce_sweep.md profiles/r01_reduce_sweep.md
