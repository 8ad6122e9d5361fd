# Round-2 evidence pass (one GPU): ALU peak microbenchmarks, the bench
# default's launch list and one ncu --set full capture of its kernel, the
# hysteresis loop kernels (P = 1 cooperative loop, P = 8 fused multi-partition
# loop) with L2 traffic, and compute-sanitizer memcheck / racecheck /
# synccheck over scripts/sanitize_small.py.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mb scripts/microbench_peaks.cu && \
  ./gpurun_out/mb > gpurun_out/alu_peaks.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/filter_launches_r02.csv python bench.py --steps 2 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rgba_ns_tma -s 3 -c 1 \
  -o gpurun_out/filter_r02 -f python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/filter_r02.ncu-rep --page raw --csv > gpurun_out/filter_r02_raw.csv 2>&1
ncu -i gpurun_out/filter_r02.ncu-rep --page details --csv > gpurun_out/filter_r02_details.csv 2>&1
for P in 1 8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_planes_(loop|multi)" -c 1 \
    -o gpurun_out/hyst_p${P}_r02 -f python bench.py --workload hysteresis --parts $P --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
  ncu -i gpurun_out/hyst_p${P}_r02.ncu-rep --page raw --csv > gpurun_out/hyst_p${P}_r02_raw.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/hyst_p8_launches_r02.csv python bench.py --workload hysteresis --parts 8 --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
ls -la gpurun_out/
