#!/bin/bash
# A/B the fused gradient-combine kernel's load hoisting / occupancy variants
# (scripts/build_variants.sh) over contribution counts. usage: bash scripts/ab_reduce_hoist.sh "h4 h4b2" "1 2 3 4"
mkdir -p gpurun_out/r01h
for rep in 1 2; do
for v in $1; do for k in $2; do
  ADT_LIB=$PWD/paper_2004_02297_b200/variants/libadt_$v.so timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-awp-step --quiet-extra --reduce-contribs $k > gpurun_out/r01h/abred_${v}_$k.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r01h/abred_${v}_$k.json'))['fused_reduce_sgd_pack']; print('$v', $k, round(d['fused_ms']*1e3,1), 'us', round(d['fused_GBps'],1))"
done; done; done
