# ncu --set full capture of the one-partition plane loop (source-level stalls).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_planes_loop -s 2 -c 1 \
  -o gpurun_out/hyst_loop -f python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_hyst.log 2>&1
tail -3 gpurun_out/ncu_hyst.log
ls -la gpurun_out/hyst_loop.ncu-rep
