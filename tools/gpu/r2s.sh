timeout 300 python tools/profile_run.py vogels 320000 10000 1000 > gpurun_out/r2s_vogels.txt 2>&1
SYNQ_SOLO=0 timeout 300 python tools/profile_run.py vogels 320000 10000 1000 >> gpurun_out/r2s_vogels.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_schedules.py tests/test_abi.py tests/test_cli.py -q -x -p no:cacheprovider 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2s_test.txt
