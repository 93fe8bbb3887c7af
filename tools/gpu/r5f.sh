for v in "" "SYNQ_LEAD=14" "SYNQ_LEAD=12" "SYNQ_LEAD=10" "SYNQ_MAXPASS=7 SYNQ_LEAD=13"; do env $v timeout 300 python tools/brunel_time.py 1e9 30000 10000; done
