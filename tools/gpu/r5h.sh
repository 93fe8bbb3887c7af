for i in 1 2; do timeout 300 python tools/plus_run.py 1e8 2000; done
timeout 300 python tools/plus_run.py 1e9 300
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_big.py tests/test_gpu_rates.py tests/test_gpu_cpp.py -q -x -p no:cacheprovider 2>&1 | tail -2
