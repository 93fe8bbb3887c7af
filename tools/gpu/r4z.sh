for v in "" "SYNQ_BITMAP=2" "SYNQ_BITMAP=2 SYNQ_UW=8" "SYNQ_UW=8" "SYNQ_BITMAP=2 SYNQ_MAXPASS=2"; do echo "[$v]"; env $v timeout 120 python tools/vogels_tiles.py 0 32 64 2>&1 | grep tiles=; done
