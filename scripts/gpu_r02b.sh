OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_hostsync.py -x -q > $OUT/pytest_hostsync.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
lscpu > $OUT/lscpu.txt; cat /sys/devices/system/cpu/cpu0/cache/index3/size >> $OUT/lscpu.txt 2>&1
PROBE_QUICK=1 timeout 900 python scripts/host_pack_probe.py > $OUT/host_probe.txt 2>&1
tail -3 $OUT/pytest_hostsync.log
