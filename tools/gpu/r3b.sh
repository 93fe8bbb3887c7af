for u in 4 2 4 2; do SYNQ_CATCHUP_U=$u timeout 300 python tools/plus_run.py 1e8 2000 >> gpurun_out/r3b.txt 2>&1; done
SYNQ_CATCHUP_U=2 timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/r3b.txt 2>&1
