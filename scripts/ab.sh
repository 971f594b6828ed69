#!/bin/bash
# A/B the kernel variants on one workload: bash scripts/ab.sh <tag> <config> [variants...]
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
summ() { python -c "
import json,sys
for l in open('$1'):
  try: d=json.loads(l)
  except Exception: continue
  r=d.get('roofline') or {}
  print('$2', round(d['value'],1), round(r.get('pack_GBps',0)), round(r.get('unpack_GBps',0)), d['clocks']['sm_mhz'])
"; }
for v in default tma "$@"; do
  for nn in "" "--no-norm"; do
    case $v in
      tma) env="ADT_KERNEL=tma";;
      default) env="";;
      *) env="ADT_LIB=$PWD/paper_2004_02297_b200/variants/libadt_$v.so";;
    esac
    f=$OUT/ab_${CFG}_${v}${nn// /}.json
    env $env timeout 300 python bench.py --config $CFG --steps 500 --no-cpu-baseline --no-e2e $nn > $f 2>&1
    summ $f "$v$nn"
  done
done
