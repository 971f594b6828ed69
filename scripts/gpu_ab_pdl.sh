#!/bin/bash
# A/B: unpack as a programmatic dependent of the pack (ADT_PDL=1, default) vs ordinary launch.
OUT=gpurun_out/${1:-r02e}; mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
for pdl in 1 0; do
  for c in alexnet resnet50 lenet; do
    ADT_PDL=$pdl timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step > $OUT/bench_${c}_pdl$pdl.json 2>&1
  done
done
ADT_PDL=1 python scripts/small_step_probe.py > $OUT/small_pdl1.txt 2>&1
ADT_PDL=0 python scripts/small_step_probe.py > $OUT/small_pdl0.txt 2>&1
