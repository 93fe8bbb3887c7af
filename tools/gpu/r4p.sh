for i in 1 2; do timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
SYNQ_PROFILE=1 timeout 300 python tools/profile_run.py brunel 1e9 5000 1000 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_schedules.py -q -x -p no:cacheprovider 2>&1 | tail -2
