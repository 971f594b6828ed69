#!/bin/bash
# Full evidence pass: tests, smoke, default bench line, extra configs, reference arm,
# ncu launch list + --set full capture of pack/unpack. usage: bash scripts/gpu_full.sh <tag>
TAG=${1:-full}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw,driver_version --format=csv > $OUT/nvsmi.txt
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2>&1
for c in resnet50 vgg16 lenet; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-reduce > $OUT/bench_$c.json 2>&1; done
for b in 8 16 24 32; do timeout 600 python bench.py --config 1b --bits $b --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 3 > $OUT/bench_1b_$b.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_alexnet python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > $OUT/ncu_full.log 2>&1
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_sgd -c 1 -o $OUT/prof_sgd python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-h2d --no-reduce --quiet-extra --eager > $OUT/ncu_sgd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_sgd -c 1 -o $OUT/prof_reduce python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --quiet-extra --eager > $OUT/ncu_reduce.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_resnet50 python bench.py --config resnet50 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > $OUT/ncu_resnet.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_resnet50.csv python bench.py --config resnet50 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 python scripts/table2.py > $OUT/table2.md 2>&1
ADT_KERNEL=tma timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_tma.log 2>&1
for t in memcheck racecheck synccheck initcheck; do timeout 600 compute-sanitizer --tool $t python scripts/sanitize_smoke.py > $OUT/sanitize_$t.log 2>&1; done
ADT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --transport p2p --config lenet > $OUT/bench_n2_gloo_p2p.log 2>&1
tail -n 2 $OUT/pytest_gpu_tma.log $OUT/sanitize_*.log
python scripts/step_overhead.py > $OUT/step_overhead.txt 2>&1
timeout 600 python -m paper_2004_02297_b200 bench-codec --sizes 1000000,67108864 --workers 1,2,8 > $OUT/bench_codec.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_awp_device.csv python scripts/awp_device_profile.py resnet50 > /dev/null 2>&1
timeout 300 python examples/train_mlp_adt.py > $OUT/train_awp.json 2>&1; timeout 300 python examples/train_mlp_adt.py --awp-on-device > $OUT/train_awp_device.json 2>&1; timeout 300 python examples/train_mlp_adt.py --fp32 > $OUT/train_fp32.json 2>&1
bash scripts/reduce_sweep.sh $OUT/sweep > $OUT/reduce_sweep.md 2>&1
