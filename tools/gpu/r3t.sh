export SYNQ_WATCHDOG=60
for cfg in "0 1e9 3 49 1000" "0 1e9 4 37 1000"; do
  echo "== $cfg"; timeout 150 python tools/peer_w4.py $cfg 2>&1 | grep -v "cta .*r_next 0 next" | head -30; echo "rc=$?"
done > gpurun_out/r3t.log 2>&1
timeout 900 python tools/peer_probe.py 1e9 3000 2 3 4 >> gpurun_out/r3t.log 2>&1
grep -v Warn gpurun_out/r3t.log | head -70
