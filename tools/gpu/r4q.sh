for v in "" "SYNQ_MAXPASS=8" ""; do env $v timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
timeout 900 python -m pytest tests/test_gpu_schedules.py -q -x -p no:cacheprovider 2>&1 | tail -2
