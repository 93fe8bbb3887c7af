export CUDA_DEVICE_MAX_CONNECTIONS=32
for cfg in "0 1e9 4 30 1000" "0 1e9 3 49 1000" "0 1e9 4 37 1000"; do
  echo "== $cfg"; timeout 150 python tools/peer_w4.py $cfg; echo "rc=$?"
done > gpurun_out/r3p.log 2>&1
timeout 900 python tools/peer_probe.py 1e9 3000 2 3 4 >> gpurun_out/r3p.log 2>&1
cat gpurun_out/r3p.log | grep -v Warn
