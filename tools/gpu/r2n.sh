timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_rates.py tests/test_gpu_schedules.py tests/test_gpu_shard.py tests/test_abi.py tests/test_cli.py -q -p no:cacheprovider 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2n_test.txt
timeout 300 python tools/plus_run.py 1e8 2000 > gpurun_out/r2n_plus.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_plus_launches.csv python tools/plus_run.py 1e8 300 >> gpurun_out/r2n_plus.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_catchup1|k_recv_win" -s 900 -c 2 -o gpurun_out/r2n_plus python tools/plus_run.py 1e8 400 > gpurun_out/r2n_ncu.log 2>&1
