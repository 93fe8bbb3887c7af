set -x
timeout 1500 python tools/b8_probe.py > gpurun_out/r2c_b8.txt 2>&1
nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/r2c_b8.txt
