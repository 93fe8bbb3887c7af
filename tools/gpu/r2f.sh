set -x
SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 > gpurun_out/r2f_phase1.txt 2>&1
SYNQ_FLIST=0 SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 > gpurun_out/r2f_phase0.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/r2f_pipe python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/r2f_ncu.log 2>&1
