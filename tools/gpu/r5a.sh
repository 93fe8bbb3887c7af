for a in "0.001 100" "0.01 100" "0.001 10" "0.001 100"; do timeout 300 build/sweep point 1e9 $a 2000; done 2>&1 | grep -v Warn
timeout 120 python tools/vogels_tiles.py 0 2>&1 | grep tiles=
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_schedules.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
