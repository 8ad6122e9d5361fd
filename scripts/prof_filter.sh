# Filter (bench default): launch list of the default bench command and one
# ncu --set full capture of the fused TMA kernel.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/filter_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rgba_ns_tma -s 3 -c 1 \
  -o gpurun_out/filter -f python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/filter*
