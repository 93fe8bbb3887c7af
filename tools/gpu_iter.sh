set -x
for t in 1 3; do timeout 60 python tools/hang_probe.py $t 2>&1 | tail -2; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
SYNQ_LEAD=8 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/pipe_bm python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/ncu_bm.log 2>&1; tail -2 gpurun_out/ncu_bm.log
