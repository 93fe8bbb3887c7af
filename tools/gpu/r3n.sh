set -x
timeout 900 python tools/peer_probe.py 1e9 3000 2 4 > gpurun_out/r3n_probe.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/r3n_bench.log 2>&1
tail -n 12 gpurun_out/r3n_probe.log
tail -n 1 gpurun_out/r3n_bench.log | cut -c1-400
