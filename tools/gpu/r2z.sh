for sz in 16 8; do SYNQ_CLUSTER=1 SYNQ_CLUSTER_SIZE=$sz timeout 120 python tools/profile_run.py vogels 320000 10000 1000 >> gpurun_out/r2z.txt 2>&1; done
timeout 120 python tools/profile_run.py vogels 320000 10000 1000 >> gpurun_out/r2z.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_schedules.py -q -p no:cacheprovider -k cluster 2>&1 | grep -v "^$" | tail -15 >> gpurun_out/r2z.txt
