set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r2a_gputest.txt
ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/r2a_pipe python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/r2a_ncu.log 2>&1
SYNQ_PROFILE=1 python tools/profile_run.py brunel 1e9 5000 1000 > gpurun_out/r2a_phase.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench.txt 2>&1
