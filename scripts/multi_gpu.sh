#!/bin/bash
# Multi-GPU evidence on one node (needs N GPUs): bench.py at N = 2/4/8 for both
# transports (value = whole-job bytes/s, sync_ms_per_iter, fp32_allgather,
# dp_update, e2e), the data-parallel example, and an nsys-free NVLink check via
# ncu's nvlink counters on rank 0 of a 2-GPU p2p step.
# usage: bash scripts/multi_gpu.sh <tag> [config]
TAG=${1:-multi}; CFG=${2:-alexnet}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NGPU=$(nvidia-smi -L | wc -l)
echo "GPUs visible: $NGPU" | tee $OUT/gpus.txt
nvidia-smi topo -m >> $OUT/gpus.txt 2>&1
port=29600
for n in 2 4 8; do
  [ "$n" -le "$NGPU" ] || continue
  for t in p2p nccl; do
    port=$((port + 1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n --config $CFG --transport $t > $OUT/bench_n${n}_$t.json 2> $OUT/bench_n${n}_$t.err
    python - "$OUT/bench_n${n}_$t.json" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        continue
    fp, ex = d.get("fp32_allgather") or {}, d.get("exchange") or {}
    print(f"N={d['n_gpus']} {d['setup']['transport']:<4} value {d['value']:9.1f} GB/s  sync {d['ms_per_step'] * 1e3:8.1f} us"
          f"  busbw {ex.get('busbw_GBps', float('nan')):7.1f} GB/s  fp32 all-gather {fp.get('ms', float('nan')) * 1e3:8.1f} us"
          f" ({fp.get('busbw_GBps', float('nan')):7.1f} GB/s)  e2e {(d.get('e2e') or {}).get('value', 0):8.1f}")
PY
  done
  port=$((port + 1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port examples/train_mlp_dp.py --steps 200 > $OUT/train_dp_n$n.json 2>&1
done
port=$((port + 1))
timeout 900 ncu --target-processes all --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum --clock-control none \
  -k regex:adt_unpack -c 4 --csv --log-file $OUT/nvlink_n2.csv \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port \
  bench.py --gpus 2 --config $CFG --transport p2p --steps 3 --warmup 1 --eager --quiet-extra \
  --no-e2e --no-reduce > $OUT/nvlink_n2.log 2>&1
