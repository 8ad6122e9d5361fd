python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fft -s 2 -c 1 \
  -o gpurun_out/fft -f python bench.py --workload fft --steps 3 --warmup 3 --no-cpu > gpurun_out/prof_fft.log 2>&1
tail -2 gpurun_out/prof_fft.log
