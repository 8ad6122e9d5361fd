# ncu --set full capture of the fused multi-partition plane loop (P = 8).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_planes_multi -s 2 -c 1 \
  -o gpurun_out/hyst_multi -f python bench.py --workload hysteresis --parts 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_hyst_multi.log 2>&1
tail -2 gpurun_out/ncu_hyst_multi.log
