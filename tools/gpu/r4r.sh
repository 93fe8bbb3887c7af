for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'])"; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cli.py tests/test_gpu_shard.py tests/test_gpu_cpp.py -q -x -p no:cacheprovider 2>&1 | tail -2
