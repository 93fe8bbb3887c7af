for i in 1 2; do timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
timeout 300 python tools/profile_run.py vogels 3.2e5 10000 1000
SYNQ_PROFILE=1 timeout 300 python tools/profile_run.py brunel 1e9 5000 1000 2>&1 | tail -4
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_sweep.py -q -x -p no:cacheprovider 2>&1 | tail -3
