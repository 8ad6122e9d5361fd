set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
for c in 1 2 3 4; do MW_RGBA_TMA=$c timeout 300 python bench.py --no-cpu --steps 3000 > gpurun_out/bench_filter_tma$c.log 2>&1; done
for c in 2 3 4; do MW_RGBA_TMA=$c timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu" -x -k "filter" > gpurun_out/gpu_tests_tma$c.log 2>&1; tail -1 gpurun_out/gpu_tests_tma$c.log; done
timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hysteresis.log 2>&1
timeout 300 python bench.py --workload segmentation --no-cpu > gpurun_out/bench_segmentation.log 2>&1
timeout 300 python bench.py --workload mapreduce_dot --no-cpu > gpurun_out/bench_mapreduce_dot.log 2>&1
