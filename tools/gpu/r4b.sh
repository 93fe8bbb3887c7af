# weight-only receive staging: Brunel+ parity + timing + launch list; one-rank shard exchange costs
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_big.py tests/test_gpu_rates.py tests/test_gpu_schedules.py -q -x -p no:cacheprovider > gpurun_out/r4b_tests.log 2>&1; echo "pytest rc=$?"
tail -n 4 gpurun_out/r4b_tests.log
for i in 1 2; do timeout 300 python tools/plus_run.py 1e8 2000; done > gpurun_out/r4b_plus.txt 2>&1
timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/r4b_plus.txt 2>&1
cat gpurun_out/r4b_plus.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv --log-file gpurun_out/r4b_plus_launches.csv python tools/plus_run.py 1e8 300 > /dev/null 2>&1; echo "ncu rc=$?"
SYNQ_WATCHDOG=60 timeout 900 python tools/shard1_probe.py > gpurun_out/r4b_shard1.txt 2>&1; echo "shard1 rc=$?"
grep -v Warn gpurun_out/r4b_shard1.txt | tail
