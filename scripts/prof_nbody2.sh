# ncu --set full capture of the N-body kernel (one launch) + raw export.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/nb
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_nbody$" -c 1 \
  -o gpurun_out/nb/nbody -f python bench.py --workload nbody --steps 1 --warmup 3 --trials 1 --no-cpu > gpurun_out/nb/ncu.log 2>&1
ncu -i gpurun_out/nb/nbody.ncu-rep --page raw --csv > gpurun_out/nb/nbody_raw.csv 2>&1
tail -2 gpurun_out/nb/ncu.log
