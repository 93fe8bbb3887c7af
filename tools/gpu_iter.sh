timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1e.log 2>&1; tail -1 gpurun_out/bench_r1e.log | cut -c1-200
timeout 300 python tools/e2e_probe.py 2>&1 | tail -2
