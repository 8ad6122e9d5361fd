"""One-GPU proxy of strong scaling for every sharded workload:
the time of ONE rank's share of an N-rank job, run alone on one B200, against
the whole job on one GPU.  T(1) / T(share) bounds the N-GPU speed-up from
above: it leaves out the cross-rank work (MapReduce: one all-reduce of the
chunk partials; hysteresis: a peer-memory barrier per pass; N-body: the
allgather of 32 MiB of state per step) and the max over ranks.

* filter / segmentation / MapReduce / FFT: bench.py's own workload classes
  set up on the share's size (8192/N rows, 512/N slabs, 2^30/N elements,
  512/N transforms) as an independent problem, with the same rotating
  buffer sets (>= 2x L2 per step) and run pipelining as the bench; the
  step time is the median of 3 trials of K runs (CUDA events on the
  stream, after warm-up).
* hysteresis: scripts/probe_hyst_share.py (the share must run the global
  E = 48 executions).
* N-body: the 2^20-body step on N virtual partitions of one ctx (each
  partition its own launch over its 2^20/N targets against all 2^20
  sources); the share = the slowest partition's kernel time from the
  monitoring events (mw_last_timings).

Prints one JSON line per (workload, N)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1510_06585_b200 import marrow as M, trees  # noqa: E402

DEV = torch.device("cuda:0")
NS = (1, 2, 4, 8)
ONLY = set(sys.argv[1:])   # workload names to run (default: all)


def share_setup(name, n):
    c = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_monitoring(c, False)
    w = bench.WORKLOADS[name](M, trees, synth, torch, c, DEV, 0)
    if name == "filter":
        w.setup(H=8192 // n)
    elif name == "segmentation":
        w.setup(shape=(512 // n, 1024, 1024))
    elif name.startswith("mapreduce"):
        w.setup(n=(1 << 30) // n)
    elif name == "fft":
        w.setup(B=512 // n)
    return c, w


def time_steps(w, K, trials=3, warm=5):
    s = torch.cuda.current_stream()
    for i in range(warm):
        w.step(i)
    torch.cuda.synchronize()
    out = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(K):
            f = w.step(i)
        e1.record(s)
        f.wait()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / K * 1e3)
    return statistics.median(out), min(out), max(out)


def emit(d):
    print(json.dumps(d), flush=True)


for name, K in (("filter", 200), ("segmentation", 100), ("mapreduce_sum", 40), ("mapreduce_dot", 20),
                ("fft", 40)):
    if ONLY and name not in ONLY:
        continue
    base = None
    for n in NS:
        c, w = share_setup(name, n)
        med, lo, hi = time_steps(w, K)
        base = base or med
        emit({"workload": name, "ranks": n, "share_units": w.n, "buffer_sets": w.B,
              "us_per_step": round(med, 2), "min_us": round(lo, 2), "max_us": round(hi, 2),
              "speedup_bound": round(base / med, 2)})
        del w, c
        torch.cuda.empty_cache()

# N-body: virtual partitions of one ctx, the slowest partition's kernel time
if ONLY and "nbody" not in ONLY:
    sys.exit(0)
pos = torch.empty((1 << 20, 4), dtype=torch.float32, device=DEV)
vel = torch.empty_like(pos)
synth.dev_fill_nbody(pos, vel, synth.SEED_NBODY, 0, 2.0 ** -20)
base = None
for n in NS:
    c = M.mw_ctx_create(0, 0, 1, n)
    M.mw_ctx_set_monitoring(c, True)
    al = M.ArgList([M.arg(pos, M.MW_COPY), M.arg(vel, M.MW_COPY)])
    tree = trees.nbody(1)
    M.mw_run(c, tree, al).wait()
    shares = []
    for _ in range(3):
        M.mw_run(c, tree, al).wait()
        ms, _wall = M.mw_last_timings(c)
        shares.append(max(ms) * 1e3)
    med = statistics.median(shares)
    base = base or med
    emit({"workload": "nbody", "ranks": n, "share_units": (1 << 20) // n, "us_per_step": round(med, 1),
          "min_us": round(min(shares), 1), "max_us": round(max(shares), 1),
          "speedup_bound": round(base / med, 2), "timing": "slowest virtual partition (monitoring events)"})
    del c
