timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -p no:cacheprovider 2>&1 | grep -v "^$" | tail -15 > gpurun_out/r2w_test.txt
timeout 600 build/sweep 1e9 2000 > gpurun_out/r2w_sweep.txt 2>&1
timeout 300 python tools/profile_run.py vogels 320000 10000 1000 > gpurun_out/r2w_vogels.txt 2>&1
