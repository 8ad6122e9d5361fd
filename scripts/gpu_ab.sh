# A/B of two kernels.cu variants on the same box: $1 = bench args; alternates
mkdir -p gpurun_out/ab
# builds of gpurun_out/ab/kernels_{base,new}.cu and prints ms_per_step of each run.
for round in 1 2; do
for v in base new; do
  cp abtmp/kernels_$v.cu paper_1510_06585_b200/csrc/kernels.cu
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build_$v.log 2>&1 || { tail -5 gpurun_out/ab/build_$v.log; continue; }
  timeout 300 python bench.py --no-cpu $1 > gpurun_out/ab/b_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab/b_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step']*1e3,2), d['aux']['trials_ms_per_step'], d['clocks']['reasons'])"
done
done
