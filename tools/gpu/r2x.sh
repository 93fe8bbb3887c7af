for i in 1 2; do timeout 120 python tools/profile_run.py brunel 1e9 10000 1000 >> gpurun_out/r2x.txt 2>&1; done
SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 >> gpurun_out/r2x.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_parity_big.py tests/test_gpu_shard.py -q -x -p no:cacheprovider -k "not brunel_plus" 2>&1 | grep -v "^$" | tail -5 >> gpurun_out/r2x.txt
