for v in "" "SYNQ_MAXPASS=8" "SYNQ_MAXPASS=6" ""; do env $v timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
