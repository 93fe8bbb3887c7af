# full suite + smoke + bench on the final tree (streamed-update prefetch)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4y_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4y_gputest.log
tail -n 4 gpurun_out/r4y_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4y_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r4y_smoke.log
timeout 600 python bench.py > gpurun_out/r4y_bench.json 2> gpurun_out/r4y_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r4y_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['secondary'], d['clocks'])"
