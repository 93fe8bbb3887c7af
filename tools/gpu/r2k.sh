timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_rates.py tests/test_gpu_schedules.py tests/test_gpu_shard.py -q -x -p no:cacheprovider -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/r2k_test.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_plus_launches.csv python tools/plus_run.py 1e8 300 > gpurun_out/r2k_plus.txt 2>&1
timeout 300 python tools/plus_run.py 1e8 2000 >> gpurun_out/r2k_plus.txt 2>&1
