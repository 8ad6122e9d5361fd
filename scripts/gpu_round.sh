set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
MW_NBODY_SPLIT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu" -x -k "nbody or rebalance" > gpurun_out/gpu_tests_nosplit.log 2>&1
tail -1 gpurun_out/gpu_tests_nosplit.log
for c in 5 6 1; do MW_RGBA_TMA=$c timeout 300 python bench.py --no-cpu --steps 3000 > gpurun_out/bench_filter_tma$c.log 2>&1; done
for sp in 1 0; do MW_NBODY_SPLIT=$sp timeout 300 python bench.py --workload nbody --no-cpu > gpurun_out/bench_nbody_split$sp.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" -x -k "nbody or filter" > gpurun_out/gpu_tests_slow.log 2>&1
tail -1 gpurun_out/gpu_tests_slow.log
