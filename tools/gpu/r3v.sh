for a in "4 7" "4 1000" "3 7" "2 7" "4 7 16 1 1 1 1 1 1 1 1 1 1 100" "4 7 16 20 200"; do echo "== $a"; timeout 120 python tools/peer_diff.py $a 2>&1 | grep -v Warn; done > gpurun_out/r3v.log 2>&1
cat gpurun_out/r3v.log
