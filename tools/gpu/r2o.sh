timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_rates.py tests/test_gpu_parity_big.py -q -p no:cacheprovider -k "not brunel_1e9" 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2o_test.txt
timeout 300 python tools/plus_run.py 1e8 2000 > gpurun_out/r2o_plus.txt 2>&1
timeout 900 ncu --graph-profiling node --set full --import-source on --clock-control none -k regex:"k_catchup1|k_recv_win|k_update" -s 1500 -c 3 -o gpurun_out/r2o_plus python tools/plus_run.py 1e8 600 > gpurun_out/r2o_ncu.log 2>&1
