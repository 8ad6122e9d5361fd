set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x -k "nbody or rebalance" > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --workload nbody --no-cpu > gpurun_out/bench_nbody.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_filter.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_filter.csv python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rgba -s 5 -c 1 -o gpurun_out/prof_filter python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nbody -s 0 -c 1 -o gpurun_out/prof_nbody python bench.py --workload nbody --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_nbody.log 2>&1
