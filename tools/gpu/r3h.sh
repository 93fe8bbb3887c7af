timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err
