# FFT iteration on one B200: build, the FFT GPU tests, the FFT bench line.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -k "fft" > gpurun_out/gpu_fft_tests.log 2>&1
tail -2 gpurun_out/gpu_fft_tests.log
timeout 300 python bench.py --workload fft --no-cpu > gpurun_out/bench_fft.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_fft.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline'])"
