mkdir -p /tmp/r5g
timeout 600 ncu --set full --clock-control none --graph-profiling node -k regex:k_catchup1 -s 60 -c 1 -o /tmp/r5g/catchup python tools/plus_run.py 1e8 120 > /tmp/r5g/log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --graph-profiling node -k regex:k_recv_win -s 60 -c 1 -o /tmp/r5g/recv python tools/plus_run.py 1e8 120 >> /tmp/r5g/log 2>&1; echo "ncu rc=$?"
for k in catchup recv; do ncu -i /tmp/r5g/$k.ncu-rep --page raw --csv > gpurun_out/r5g_${k}_raw.csv 2>/dev/null; done
ls -la gpurun_out/r5g_*; rm -rf /tmp/r5g
