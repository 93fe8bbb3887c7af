timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 1 -c 1 -o gpurun_out/r3j_ell build/sweep point 1e9 0.001 100 600 > gpurun_out/r3j.log 2>&1
