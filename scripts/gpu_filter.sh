# Filter iteration on one B200: build, the filter / RGBA GPU tests, the default bench line (3 runs).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -k "filter or rgba or noise or solar or mirror" > gpurun_out/gpu_filter_tests.log 2>&1
tail -2 gpurun_out/gpu_filter_tests.log
for i in 1 2 3; do
timeout 300 python bench.py --no-cpu > gpurun_out/bench_filter_$i.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_filter_$i.json').read().strip().splitlines()[-1]);print(d['ms_per_step']*1e3, d['roofline']['frac'], d['clocks'], d['aux']['trials_ms_per_step'])"
done
