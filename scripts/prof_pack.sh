# pack kernel duration at unlocked clocks (ncu launch list of 3 launches)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_planes_pack -s 2 -c 3 \
  python bench.py --workload hysteresis --steps 2 --warmup 3 --no-cpu 2>/dev/null | grep -E "duration"
