timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -q -k "peer" > gpurun_out/r3u.log 2>&1
tail -n 30 gpurun_out/r3u.log
