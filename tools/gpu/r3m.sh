set -x
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -x -q -k peer > gpurun_out/r3m_peer.log 2>&1
tail -n 30 gpurun_out/r3m_peer.log
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r3m_shard.log 2>&1
tail -n 3 gpurun_out/r3m_shard.log
timeout 600 python tools/peer_probe.py 1e9 2000 2 > gpurun_out/r3m_probe.log 2>&1
cat gpurun_out/r3m_probe.log | tail -n 8
