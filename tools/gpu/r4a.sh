# round 2 (session 3): full GPU suite, bench, peer-exchange probe
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r4a_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4a_gputest.log
tail -n 15 gpurun_out/r4a_gputest.log
timeout 600 python bench.py > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r4a_bench.json
SYNQ_WATCHDOG=60 timeout 900 python tools/peer_probe.py 1e9 3000 1 2 > gpurun_out/r4a_peer.log 2>&1; echo "peer rc=$?"
grep -v Warn gpurun_out/r4a_peer.log | tail -20
