# Round measurement pass on one B200: build, smoke, GPU suite, bench lines of
# every workload, launch lists and one ncu --set full capture of the
# hysteresis loop kernel (gpurun_out/ is scratch; summaries go to profiles/).
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 1200 python bench.py --workload all --no-cpu > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
timeout 300 python bench.py --workload mapreduce_max --no-cpu >> gpurun_out/bench_all.json 2>> gpurun_out/bench_all.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hyst_launches.csv \
  python bench.py --workload hysteresis --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_planes_loop -s 2 -c 1 \
  -o gpurun_out/hyst_loop -f python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_planes_pack -s 2 -c 1 \
  -o gpurun_out/hyst_pack -f python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_planes_unpack -s 2 -c 1 \
  -o gpurun_out/hyst_unpack -f python bench.py --workload hysteresis --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out
