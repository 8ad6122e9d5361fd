set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for u in 2 4 8; do MW_RGBA_UNROLL=$u timeout 300 python bench.py --workload filter --no-cpu > gpurun_out/bench_filter_u$u.log 2>&1; done
timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hysteresis.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" -x > gpurun_out/gpu_tests_slow.log 2>&1
tail -3 gpurun_out/gpu_tests_slow.log
