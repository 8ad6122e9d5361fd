# Final round-2 bench lines of every workload + hysteresis at 1/2/4/8 partitions.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/fin
timeout 1500 python bench.py --workload all --no-cpu > gpurun_out/fin/bench_all.jsonl 2> gpurun_out/fin/bench_all.err
for P in 1 2 4 8; do
  timeout 300 python bench.py --workload hysteresis --parts $P --no-cpu >> gpurun_out/fin/bench_parts.jsonl 2>> gpurun_out/fin/bench_all.err
done
timeout 300 python bench.py > gpurun_out/fin/bench_default.json 2>> gpurun_out/fin/bench_all.err
wc -l gpurun_out/fin/*.jsonl
