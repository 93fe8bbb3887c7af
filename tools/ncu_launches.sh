#!/bin/bash
# Launch list + one full capture of the step kernel for the headline config.
# Usage (under gpurun): bash tools/ncu_launches.sh <outdir>
set -e
out=${1:-gpurun_out}
mkdir -p "$out"
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > "$out/launches_bench.log" 2>&1
# one full capture of the persistent step kernel (a 200-step batch)
ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 2 -c 1 \
    -o "$out/prof_brunel1e9" python tools/profile_run.py brunel 1e9 800 200 > "$out/prof_capture.log" 2>&1
