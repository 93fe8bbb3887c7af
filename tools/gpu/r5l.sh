timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "raster or runs_bit_exact" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r5l_bench.json 2> gpurun_out/r5l_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r5l_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])"
