timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solo -s 2 -c 1 -o gpurun_out/r2t_solo python tools/profile_run.py vogels 320000 3000 1000 > gpurun_out/r2t_ncu.log 2>&1
