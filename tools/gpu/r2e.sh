set -x
timeout 600 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2e_test.txt
for v in "SYNQ_FLIST=1" "SYNQ_FLIST=0" "SYNQ_FLIST=1 SYNQ_DEFER=0" "SYNQ_FLIST=1"; do echo "$v" >> gpurun_out/r2e_ab.txt; env $v timeout 120 python tools/profile_run.py brunel 1e9 10000 1000 >> gpurun_out/r2e_ab.txt 2>&1; done
SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 > gpurun_out/r2e_phase.txt 2>&1
