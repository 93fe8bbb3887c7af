timeout 900 python -m pytest tests/test_gpu_sweep.py -q -p no:cacheprovider 2>&1 | grep -v "^$" | tail -8 > gpurun_out/r3i.txt
