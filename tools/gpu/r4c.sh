# fused catch-up in the windowed receive (trace-STDP): parity + timing A/B; NCCL one-rank shard without the watchdog
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_big.py tests/test_gpu_rates.py tests/test_gpu_schedules.py tests/test_gpu_cpp.py -q -x -p no:cacheprovider > gpurun_out/r4c_tests.log 2>&1; echo "pytest rc=$?"
tail -n 4 gpurun_out/r4c_tests.log
for i in 1 2; do timeout 300 python tools/plus_run.py 1e8 2000; SYNQ_FUSED_CATCHUP=0 timeout 300 python tools/plus_run.py 1e8 2000; done > gpurun_out/r4c_plus.txt 2>&1
timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/r4c_plus.txt 2>&1
SYNQ_FUSED_CATCHUP=0 timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/r4c_plus.txt 2>&1
cat gpurun_out/r4c_plus.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node --csv --log-file gpurun_out/r4c_plus_launches.csv python tools/plus_run.py 1e8 300 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python tools/shard1_probe.py unsharded nccl > gpurun_out/r4c_shard1.txt 2>&1; echo "shard1 rc=$?"
grep -v Warn gpurun_out/r4c_shard1.txt | tail
