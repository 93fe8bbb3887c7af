set -x
python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r2b_test.txt
