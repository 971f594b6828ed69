#!/bin/bash
# Round-2 final evidence pass on one GPU box (after the host-path and K7 changes): tests, smoke,
# the reference's own suite on the plugged hot path, both bench arms, every config, ncu launch
# lists + --set full captures, sanitizers, the gloo N>1 hook, small-set and step probes.
#   bash scripts/gpu_r02_final.sh <tag>      -> gpurun_out/<tag>/   (then scripts/refresh_profiles.sh <tag>)
TAG=${1:-r02z}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw,driver_version --format=csv > $OUT/nvsmi.txt
timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > $OUT/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
(cd /tmp && timeout 900 python $GRAFT_REPO_ROOT/tests/refsuite/run.py --plug $GRAFT_REPO_ROOT/baseline/_ref/tests test_codec.py test_precision.py test_transfer.py test_training.py test_acceptance.py test_cli.py test_net.py test_dataset_config.py -rf) > $OUT/refsuite_plug.txt 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
for c in resnet50 lenet; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_$c.json 2>&1; done
for b in 8 16 24 32; do timeout 600 python bench.py --config vgg16 --bits $b --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_vgg16_$b.json 2>&1; done
for b in 8 16 24 32; do timeout 900 python bench.py --config 1b --bits $b --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-sgd --no-reduce --no-awp-step > $OUT/bench_1b_$b.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_resnet50.csv python bench.py --config resnet50 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_alexnet python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_ -s 6 -c 3 -o $OUT/prof_resnet50 python bench.py --config resnet50 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-reduce --no-awp-step --quiet-extra --eager > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adt_sgd_pack_kernel -c 1 -o $OUT/prof_reduce python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-h2d --no-sgd --no-awp-step --quiet-extra --eager --reduce-contribs 16 > /dev/null 2>&1
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t python scripts/sanitize_smoke.py > $OUT/sanitize_$t.log 2>&1; done
ADT_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --transport p2p > $OUT/bench_n2_gloo_p2p.json 2> $OUT/bench_n2_gloo_p2p.err
ADT_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 3 --warmup 3 --transport p2p --no-reduce > $OUT/bench_n8_gloo_p2p.json 2> $OUT/bench_n8_gloo_p2p.err
timeout 600 python scripts/small_host_probe.py breakdown > $OUT/small_host_breakdown.txt 2>&1
timeout 300 python scripts/small_step_probe.py > $OUT/small_step.txt 2>&1
timeout 600 python scripts/step_overhead.py > $OUT/step_overhead.txt 2>&1
timeout 600 python scripts/table2.py > $OUT/table2.md 2>&1
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log $OUT/refsuite_plug.txt $OUT/sanitize_*.log
