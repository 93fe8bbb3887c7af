# A/B: Brunel+ 1e8 fused catch-up x catch-up U; Brunel 1e9 pipeline 16+16 vs 8+24 warps
for i in 1 2 3; do
  for v in "" "SYNQ_FUSED_CATCHUP=0" "SYNQ_CATCHUP_U=8" "SYNQ_CATCHUP_U=8 SYNQ_FUSED_CATCHUP=0"; do
    echo -n "[$v] "; env $v timeout 300 python tools/plus_run.py 1e8 2000
  done
done > gpurun_out/r4d_plus.txt 2>&1
cat gpurun_out/r4d_plus.txt
for v in "" "SYNQ_UW1024=8" "" "SYNQ_UW1024=8"; do env $v timeout 300 python tools/brunel_time.py 1e9 30000 10000; done > gpurun_out/r4d_brunel.txt 2>&1
cat gpurun_out/r4d_brunel.txt
