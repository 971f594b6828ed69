#!/bin/bash
# Round-2 evidence pass on one GPU box: tests, smoke, the driver's bench commands (both arms),
# every config, ncu launch lists + --set full captures, sanitizers, host-path probes.
#   bash scripts/gpu_r02.sh <tag>      -> gpurun_out/<tag>/
TAG=${1:-r02}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw,driver_version --format=csv > $OUT/nvsmi.txt
timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > $OUT/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
for c in resnet50 lenet; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_$c.json 2>&1; done
for b in 8 16 24 32; do timeout 600 python bench.py --config vgg16 --bits $b --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_vgg16_$b.json 2>&1; done
for b in 8 16 24 32; do timeout 900 python bench.py --config 1b --bits $b --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-sgd --no-reduce --no-awp-step > $OUT/bench_1b_$b.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_resnet50.csv python bench.py --config resnet50 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_alexnet python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_resnet50 python bench.py --config resnet50 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
for v in 1 2 3; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 2 -o $OUT/prof_vgg16_r$v python bench.py --config vgg16 --bits $((8*v)) --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1; done
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t python scripts/sanitize_smoke.py > $OUT/sanitize_$t.log 2>&1; done
ADT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --transport p2p > $OUT/bench_n2_gloo_p2p.json 2> $OUT/bench_n2_gloo_p2p.err
ADT_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 3 --warmup 3 --transport p2p --no-reduce > $OUT/bench_n8_gloo_p2p.json 2> $OUT/bench_n8_gloo_p2p.err
PROBE_QUICK=1 timeout 900 python scripts/host_pack_probe.py > $OUT/host_probe.txt 2>&1
timeout 900 python scripts/direct_probe.py > $OUT/direct_probe.txt 2>&1
timeout 300 python scripts/small_step_probe.py > $OUT/small_step.txt 2>&1
timeout 600 python scripts/step_overhead.py > $OUT/step_overhead.txt 2>&1
timeout 600 python scripts/table2.py > $OUT/table2.md 2>&1
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log $OUT/sanitize_*.log
