timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_rates.py tests/test_gpu_schedules.py -q -x -p no:cacheprovider -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/r2i_test.txt
timeout 600 python tools/plus_probe.py 1e8 2000 50 > gpurun_out/r2i_plus.txt 2>&1
timeout 300 python tools/profile_run.py brunel 1e9 10000 1000 >> gpurun_out/r2i_plus.txt 2>&1
