SYNQ_PROFILE=1 timeout 300 python tools/profile_run.py brunel 1e9 5000 1000 2>&1 | tail -5
