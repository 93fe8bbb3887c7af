# round-2 final measurement pass on the final tree
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4o_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4o_gputest.log
tail -n 4 gpurun_out/r4o_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4o_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r4o_smoke.log
timeout 600 python bench.py > gpurun_out/r4o_bench.json 2> gpurun_out/r4o_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r4o_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4o_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-secondary > gpurun_out/r4o_launches_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/r4o_pipe python tools/profile_run.py brunel 1e9 1200 200 > gpurun_out/r4o_capture.log 2>&1; echo "ncu full rc=$?"
