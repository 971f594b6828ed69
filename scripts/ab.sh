#!/bin/bash
# A/B kernel variants: bash scripts/ab.sh <tag> "<bench args>" [variant ...]
# variants: default (in-tree libadt.so), tma (ADT_KERNEL=tma), or a name from
# scripts/build_variants.sh (paper_2004_02297_b200/variants/libadt_<name>.so).
TAG=$1; ARGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  case $v in
    default) env="";;
    tma) env="ADT_KERNEL=tma";;
    *) env="ADT_LIB=$PWD/paper_2004_02297_b200/variants/libadt_$v.so";;
  esac
  f=$OUT/ab_$(echo "$v $ARGS" | tr ' -' '_').json
  env $env timeout 300 python bench.py $ARGS --no-cpu-baseline --no-e2e --no-h2d > $f 2>&1
  python - "$f" "$v $ARGS" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        continue
    r = d.get("roofline") or {}
    print(f"{sys.argv[2]:<40} value {d['value']:8.1f}  pack {r.get('pack_GBps', 0):8.1f}  unpack {r.get('unpack_GBps', 0):8.1f}  step_us {d['ms_per_step'] * 1e3:8.1f}")
PY
done
