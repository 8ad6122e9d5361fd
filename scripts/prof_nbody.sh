python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_nbody$" -c 1 \
  -o gpurun_out/nbody -f python bench.py --workload nbody --steps 1 --warmup 3 --no-cpu > gpurun_out/prof_nbody.log 2>&1
tail -2 gpurun_out/prof_nbody.log
