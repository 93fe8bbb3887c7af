# round-2 measurement pass (1 GPU): tests, bench, launch lists, ncu captures, secondary configs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/f_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/f_gputest.txt
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/f_bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/f_pipe python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/f_ncu.log 2>&1
SYNQ_PROFILE=1 timeout 120 python tools/profile_run.py brunel 1e9 5000 1000 > gpurun_out/f_phase.txt 2>&1
timeout 600 build/sweep 1e9 2000 > gpurun_out/f_sweep.txt 2>&1
timeout 900 python tools/plus_probe.py 1e8 2000 50 > gpurun_out/f_plus.txt 2>&1
timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/f_plus.txt 2>&1
timeout 600 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_plus_launches.csv python tools/plus_run.py 1e8 300 > /dev/null 2>&1
timeout 300 python tools/shard1_probe.py > gpurun_out/f_shard1.txt 2>&1
timeout 300 python tools/profile_run.py vogels 320000 10000 1000 > gpurun_out/f_vogels.txt 2>&1
