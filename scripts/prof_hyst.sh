# ncu --set full of the one-partition hysteresis loop kernel (one launch per step)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_planes_loop -s 2 -c 1 \
  -o gpurun_out/hyst_loop -f python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > gpurun_out/prof_hyst.log 2>&1
tail -3 gpurun_out/prof_hyst.log
