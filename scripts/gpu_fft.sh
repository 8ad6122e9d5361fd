# FFT iteration on one B200: build, the FFT GPU tests, the FFT bench line for both paths.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -k "fft" > gpurun_out/gpu_fft_tests.log 2>&1
tail -2 gpurun_out/gpu_fft_tests.log
grep -m5 -B3 'Error\|assert' gpurun_out/gpu_fft_tests.log | head -30
for v in 1 0; do
MW_FFT_4STEP=$v timeout 300 python bench.py --workload fft --no-cpu > gpurun_out/bench_fft$v.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_fft$v.json').read().strip().splitlines()[-1]);print('4step=$v', d['ms_per_step'], d['roofline']['frac'])"
done
