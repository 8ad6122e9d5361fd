# 4-step FFT: tests, bench at several chunk sizes, launch list of the default.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -k "fft" > gpurun_out/gpu_fft_tests.log 2>&1
tail -1 gpurun_out/gpu_fft_tests.log
for ch in 64 128 256 512; do
MW_FFT4_CHUNK=$ch timeout 300 python bench.py --workload fft --no-cpu > gpurun_out/bench_fft_c$ch.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_fft_c$ch.json').read().strip().splitlines()[-1]);print('chunk=$ch', d['ms_per_step'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fft4.csv \
  python bench.py --workload fft --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python scripts/launch_list.py gpurun_out/launches_fft4.csv | head -6
