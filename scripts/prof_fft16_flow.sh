# Default FFT bench (16 x 4096 dataflow launch): launch list and ncu --set full of one k_fft16_flow launch.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/f16f
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/f16f/fft_launches.csv python bench.py --workload fft --steps 2 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft16_flow -s 3 -c 1 \
  -o gpurun_out/f16f/fft16_flow -f python bench.py --workload fft --steps 2 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/f16f/fft16_flow.ncu-rep --page raw --csv > gpurun_out/f16f/fft16_flow_raw.csv 2>&1
ncu -i gpurun_out/f16f/fft16_flow.ncu-rep --page details --csv > gpurun_out/f16f/fft16_flow_details.csv 2>&1
