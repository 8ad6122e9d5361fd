# Hysteresis iteration on one B200: build, the hysteresis GPU tests, the bench
# line at P = 1 and 8, and the per-pass device timestamps (MW_HYST_PROF).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -k "hyst or plane or loop" > gpurun_out/gpu_hyst_tests.log 2>&1
tail -3 gpurun_out/gpu_hyst_tests.log
timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hyst.json 2> gpurun_out/bench_hyst.err
cut -c1-300 gpurun_out/bench_hyst.json
timeout 300 python bench.py --workload hysteresis --parts 8 --no-cpu > gpurun_out/bench_hyst_p8.json 2>> gpurun_out/bench_hyst.err
cut -c1-300 gpurun_out/bench_hyst_p8.json
MW_HYST_PROF=1 timeout 300 python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu 2>&1 >/dev/null | grep MW_HYST_PROF | tail -2
