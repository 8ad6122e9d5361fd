# N-body: the NBODY_SPLIT knob's two variants, bench lines.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in 0 1; do
  MW_NBODY_SPLIT=$s timeout 600 python bench.py --workload nbody --steps 2 --warmup 3 --trials 1 --no-cpu > gpurun_out/nb_split$s.json 2> gpurun_out/nb_split$s.err
  python -c "import json; d=json.loads(open('gpurun_out/nb_split$s.json').read().strip().splitlines()[-1]); print('split=$s', d['ms_per_step'], d['roofline']['frac'])"
done
