timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "bursts" 2>&1 | grep -v "^$" | tail -25 > gpurun_out/r3c.txt
