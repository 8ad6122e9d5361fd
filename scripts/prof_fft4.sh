# ncu --set full of the 4-step FFT kernels (full-batch launches of the warm-up).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/f4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft4 -s 3 -c 3 \
  -o gpurun_out/f4/fft4 -f python bench.py --workload fft --steps 2 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/f4/fft4.ncu-rep --page raw --csv > gpurun_out/f4/fft4_raw.csv 2>&1
ls gpurun_out/f4
