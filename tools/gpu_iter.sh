# One GPU iteration (run under gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_iter.sh'
# parity tests, smoke, bench, and the schedule A/B on Brunel 1e9.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200
SYNQ_PROFILE=1 AB_ONLY=bitmap AB_NO_SERIAL=1 timeout 300 python tools/ab_pipeline.py brunel 1e9 5000 15 2>&1 | grep us/step
