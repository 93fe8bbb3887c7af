for i in 1 2; do timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
timeout 900 python tools/shard1_probe.py unsharded peer 2>&1 | grep -v Warn
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_parity_big.py tests/test_gpu_shard.py -q -x -p no:cacheprovider 2>&1 | tail -2
