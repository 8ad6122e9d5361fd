# Round check on one B200: build, smoke, the whole GPU suite, default bench and
# the bench lines of the hysteresis / FFT workloads.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
cut -c1-400 gpurun_out/bench_default.json
timeout 300 python bench.py --workload hysteresis --no-cpu > gpurun_out/bench_hyst.json 2>&1
cut -c1-300 gpurun_out/bench_hyst.json
MW_HYST_PROF=1 timeout 300 python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu 2>&1 >/dev/null | grep MW_HYST_PROF | tail -1
