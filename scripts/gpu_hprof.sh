python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
MW_HYST_PROF=1 timeout 300 python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu 2>&1 >/dev/null | grep MW_HYST_PROF | tail -1
