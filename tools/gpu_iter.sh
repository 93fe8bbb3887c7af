timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SYNQ_PROFILE=1 AB_ONLY=bitmap AB_NO_SERIAL=1 timeout 300 python tools/ab_pipeline.py brunel 1e9 5000 15 2>&1 | grep us/step | cut -c1-120
