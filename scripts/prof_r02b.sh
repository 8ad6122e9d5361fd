# Round-2 (second session) evidence pass on one B200 after the plane-loop and
# FFT changes: compute-sanitizer memcheck / racecheck / synccheck over
# scripts/sanitize_small.py, ncu --set full captures (raw CSV) of the
# one-partition plane loop, the fused multi-partition loop (P = 8) and the
# FFT kernel, launch lists, and the bench lines of every workload.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py \
    > $O/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_summary.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_planes_loop -s 2 -c 1 \
  -o $O/hyst_p1 -f python bench.py --workload hysteresis --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_planes_multi -s 2 -c 1 \
  -o $O/hyst_p8 -f python bench.py --workload hysteresis --parts 8 --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fft -s 2 -c 1 \
  -o $O/fft -f python bench.py --workload fft --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
for r in hyst_p1 hyst_p8 fft; do ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/hyst_p1_launches.csv python bench.py --workload hysteresis --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/hyst_p8_launches.csv python bench.py --workload hysteresis --parts 8 --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/fft_launches.csv python bench.py --workload fft --steps 3 --warmup 3 --trials 1 --no-cpu > /dev/null 2>&1
timeout 1500 python bench.py --workload all --no-cpu > $O/bench_all.jsonl 2> $O/bench_all.err
for P in 1 2 4 8; do
  timeout 300 python bench.py --workload hysteresis --parts $P --no-cpu >> $O/bench_parts.jsonl 2>> $O/bench_all.err
done
ls -la $O
