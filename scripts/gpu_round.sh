set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for TR in "8 48" "12 48" "16 64" "8 32" "4 32"; do set -- $TR; MW_HYST_T=$1 MW_HYST_ROWS=$2 timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hyst_T$1_R$2.log 2>&1; done
timeout 300 python bench.py --workload saxpy --no-cpu > gpurun_out/bench_saxpy.log 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/bench_filter.log 2>&1
MW_HYST_T=16 MW_HYST_ROWS=64 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "hysteresis or graph" > gpurun_out/gpu_tests_T16.log 2>&1
tail -2 gpurun_out/gpu_tests_T16.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" -x -k hysteresis > gpurun_out/gpu_tests_slow.log 2>&1
tail -2 gpurun_out/gpu_tests_slow.log
