for a in "0.001 100" "0.001 10" "0.01 100" "0.001 100"; do timeout 300 build/sweep point 1e9 $a 1000; done > gpurun_out/r4g_sweep.txt 2>&1
cat gpurun_out/r4g_sweep.txt
timeout 300 python tools/profile_run.py vogels 3.2e5 10000 1000
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_schedules.py -q -x -p no:cacheprovider 2>&1 | tail -3
