python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py --workload rebalance > gpurun_out/bench_rebalance.log 2>&1
