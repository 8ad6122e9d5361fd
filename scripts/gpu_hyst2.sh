# Hysteresis (all partition modes) on one B200: build, the whole GPU suite, bench at P = 1, 2, 8.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for P in 1 2 8; do
timeout 300 python bench.py --workload hysteresis --parts $P --no-cpu > gpurun_out/bench_hyst_p$P.json 2>> gpurun_out/bench_hyst.err
python -c "import json;d=json.loads(open('gpurun_out/bench_hyst_p$P.json').read().strip().splitlines()[-1]);print('P=$P', d['ms_per_step'])"
done
