timeout 600 python -m pytest tests/test_gpu_cpp.py -q -x -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2l_test.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_update|k_catchup1|k_recv_win" -s 900 -c 3 -o gpurun_out/r2l_plus python tools/plus_run.py 1e8 400 > gpurun_out/r2l_ncu.log 2>&1
