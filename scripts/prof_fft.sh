# ncu --set full capture of the fused FFT -> IFFT kernel (source-level stalls).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fft -s 2 -c 1 \
  -o gpurun_out/fft -f python bench.py --workload fft --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_fft.log 2>&1
tail -2 gpurun_out/ncu_fft.log
