# ncu --set full of the 16 x 4096 FFT kernels (full-batch launches of the warm-up).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/f16
MW_FFT_4STEP=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft16 -s 3 -c 3 \
  -o gpurun_out/f16/fft16 -f python bench.py --workload fft --steps 2 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/f16/fft16.ncu-rep --page raw --csv > gpurun_out/f16/fft16_raw.csv 2>&1
ncu -i gpurun_out/f16/fft16.ncu-rep --page details --csv > gpurun_out/f16/fft16_details.csv 2>&1
ls gpurun_out/f16
