set -x
python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_parity_big.py -q -x -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2d_test.txt
for v in 1 0 1 0; do SYNQ_FOLD_TABLE=$v python tools/profile_run.py brunel 1e9 10000 1000 >> gpurun_out/r2d_ab.txt 2>&1; done
