#!/bin/bash
# A/B: finalize CTA size x unpack PDL (step time of the bench graph).
OUT=gpurun_out/${1:-r02f}; mkdir -p $OUT
for v in default fin128 fin256; do
  lib=""; [ $v != default ] && lib=paper_2004_02297_b200/variants/libadt_$v.so
  for pdl in 1 0; do
    for c in alexnet resnet50 lenet vgg16; do
      ADT_LIB=$lib ADT_PDL=$pdl timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step > $OUT/bench_${c}_${v}_pdl$pdl.json 2>&1
    done
  done
done
