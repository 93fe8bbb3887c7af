timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpp.py tests/test_gpu_rates.py tests/test_gpu_parity_big.py -q -p no:cacheprovider -k "not brunel_1e9" 2>&1 | grep -v "^$" | tail -6 > gpurun_out/r3f_test.txt
for v in 1 0 1; do SYNQ_PDL=$v timeout 300 python tools/plus_run.py 1e8 2000 >> gpurun_out/r3f_plus.txt 2>&1; done
timeout 300 python tools/plus_run.py 1e9 300 >> gpurun_out/r3f_plus.txt 2>&1
