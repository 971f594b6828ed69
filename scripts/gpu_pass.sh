#!/bin/bash
# One GPU pass: parity tests (both kernel families), smoke, benches, ncu launch list + full capture.
# usage: bash scripts/gpu_pass.sh <tag> [bench configs...]
TAG=${1:-run}; shift
CONFIGS=${@:-alexnet}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/nvsmi.txt
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
ADT_KERNEL=tma timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_tma.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  ADT_KERNEL=tma timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_${c}_tma.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --quiet-extra > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 4 -c 2 -o $OUT/prof_alexnet python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --quiet-extra > $OUT/ncu_full.log 2>&1
tail -3 $OUT/pytest_gpu.log $OUT/pytest_gpu_tma.log $OUT/smoke.log
for f in $OUT/bench_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
  try: d=json.loads(l)
  except Exception: continue
  r=d.get('roofline') or {}
  print(round(d['value'],1), d['ms_per_step'], {k:round(v,3) if isinstance(v,float) else v for k,v in r.items() if k in ('pack_GBps','unpack_GBps','frac','kernel')}, (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))
"; done
