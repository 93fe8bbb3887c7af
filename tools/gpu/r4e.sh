timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -p no:cacheprovider > gpurun_out/r4e_tests.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/r4e_tests.log
for i in 1 2; do timeout 300 python tools/plus_run.py 1e8 2000; done
