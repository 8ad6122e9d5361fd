# A/B of two variants of one csrc file on the same box: $1 = bench args,
# $2 = file name under paper_1510_06585_b200/csrc (variants abtmp/<file>.base
# and abtmp/<file>.new, git-ignored); alternates builds, prints ms_per_step.
mkdir -p gpurun_out/ab
F=${2:-chains.cu}
for round in 1 2; do
for v in base new; do
  cp abtmp/$F.$v paper_1510_06585_b200/csrc/$F
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build_$v.log 2>&1 || { tail -5 gpurun_out/ab/build_$v.log; continue; }
  timeout 300 python bench.py --no-cpu $1 > gpurun_out/ab/b_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab/b_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step']*1e3,2), d['aux']['trials_ms_per_step'], d['clocks']['reasons'])"
done
done
