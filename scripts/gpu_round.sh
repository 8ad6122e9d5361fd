set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hysteresis.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" -x -k hysteresis > gpurun_out/gpu_tests_slow.log 2>&1
tail -3 gpurun_out/gpu_tests_slow.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_hyst.csv python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch_hyst.log 2>&1
