timeout 900 python tools/shard1_probe.py unsharded peer nccl+peer > gpurun_out/r4f_shard1.txt 2>&1; echo "shard1 rc=$?"
grep -v Warn gpurun_out/r4f_shard1.txt | tail -4
SYNQ_PROFILE=1 timeout 300 python tools/profile_run.py vogels 3.2e5 10000 1000 > gpurun_out/r4f_vogels_prof.txt 2>&1
timeout 300 python tools/profile_run.py vogels 3.2e5 10000 1000 >> gpurun_out/r4f_vogels_prof.txt 2>&1
cat gpurun_out/r4f_vogels_prof.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pipeline -s 1 -c 1 -o gpurun_out/r4f_vogels python tools/profile_run.py vogels 3.2e5 3000 1000 > gpurun_out/r4f_ncu.log 2>&1; echo "ncu rc=$?"
