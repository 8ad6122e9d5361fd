# Per-pass device timestamps of the plane loop (MW_HYST_PROF) at P = 1 and P = $1.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
MW_HYST_PROF=1 timeout 300 python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu 2>&1 >/dev/null | grep MW_HYST_PROF | tail -1
MW_HYST_PROF=1 timeout 300 python bench.py --workload hysteresis --parts ${1:-8} --steps 3 --warmup 3 --no-cpu 2>&1 >/dev/null | grep MW_HYST_PROF | tail -1
