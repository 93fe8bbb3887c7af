set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1b.log 2>&1; tail -1 gpurun_out/bench_r1b.log | cut -c1-600
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/pipe_final python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/ncu_final.log 2>&1; tail -1 gpurun_out/ncu_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches_r1b.csv
