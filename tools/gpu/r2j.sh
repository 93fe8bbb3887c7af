timeout 300 python tools/repro_win.py > gpurun_out/r2j.txt 2>&1
