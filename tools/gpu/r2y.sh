timeout 300 python tools/e2e_probe.py > gpurun_out/r2y.txt 2>&1
