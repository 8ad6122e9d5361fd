# DRAM bytes of the dominant kernel of every bench workload (one launch each,
# ncu, not a bench run): profiles/dram_traffic.json is built from these.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {  # workload kernel-regex
  timeout 900 ncu --metrics $M --clock-control none -k regex:$2 -s 3 -c 1 --csv \
    python bench.py --workload $1 --steps 2 --warmup 3 --no-cpu 2>/dev/null | grep -E '"dram__|"gpu__time' > gpurun_out/traffic_$1.csv
}
run saxpy k_saxpy_vec
run segmentation k_u8
run mapreduce_sum k_reduce_chunks
run mapreduce_dot k_reduce_chunks
run mapreduce_max k_reduce_chunks
run hysteresis k_planes_loop
run nbody "k_nbody<"
ls -la gpurun_out/traffic_*
