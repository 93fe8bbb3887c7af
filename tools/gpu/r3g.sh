for v in 0 2 0 2; do SYNQ_DBG=$v SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 >> gpurun_out/r3g.txt 2>&1; done
