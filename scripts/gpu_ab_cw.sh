#!/bin/bash
# A/B: CTA size of the pack/unpack grids (8 warps = one tile per CTA, 4 / 2 = split tiles).
OUT=gpurun_out/${1:-r02g}; mkdir -p $OUT
for v in default cw4 cw2; do
  lib=""; [ $v != default ] && lib=paper_2004_02297_b200/variants/libadt_$v.so
  for c in resnet50 alexnet lenet vgg16; do
    ADT_LIB=$lib timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step > $OUT/bench_${c}_${v}.json 2>&1
  done
done
ADT_LIB=paper_2004_02297_b200/variants/libadt_cw4.so timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py > $OUT/pytest_cw4.log 2>&1; tail -1 $OUT/pytest_cw4.log
