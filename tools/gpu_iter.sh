timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 build/sweep 1e9 2000 2>&1 | tee gpurun_out/sweep_r1b.txt | tail -10
