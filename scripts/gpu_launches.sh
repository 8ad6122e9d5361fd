# ncu launch list (gpu__time_duration per kernel) of a workload's bench command: $1 = workload
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv \
  python bench.py --workload $1 --steps 2 --warmup 3 --no-cpu ${2:-} > /dev/null 2>&1
python scripts/launch_list.py gpurun_out/launches_$1.csv
