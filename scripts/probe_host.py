"""Probe: host time per mw_run and GPU time per run with/without monitoring
events, against CUDA-graph replay (context for the bench; not a bench number)."""
import time, torch, json, sys
sys.path.insert(0, '.')
import synth
from paper_1510_06585_b200 import marrow as M, trees
ctx = M.mw_ctx_create(0, 0, 1, 1)
H = W = 8192
src = torch.empty((H, W, 4), dtype=torch.uint8, device="cuda"); synth.dev_fill_rgba(src, 3, 0)
dst = torch.empty_like(src)
tree = trees.filter_pipeline()
args = [M.arg(src), M.arg(dst)]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for _ in range(5): M.mw_run(ctx, tree, args).wait()
torch.cuda.synchronize()
out = {}
for stats, mon in ((False, True), (True, True), (False, False)):
    M.mw_ctx_set_monitoring(ctx, mon)
    M.mw_stats_enable(ctx, stats)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(s)
    fs = [M.mw_run(ctx, tree, args) for _ in range(200)]
    t1 = time.perf_counter(); e1.record(s); torch.cuda.synchronize()
    out[f"stats={stats},monitor={mon}"] = {"host_us_per_run": (t1 - t0) / 200 * 1e6, "gpu_us_per_run": e0.elapsed_time(e1) / 200 * 1e3}
    del fs
g = M.mw_graph_capture(ctx, tree, args, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(200): g.launch(s)
e1.record(s); torch.cuda.synchronize()
out["graph_gpu_us_per_run"] = e0.elapsed_time(e1) / 200 * 1e3
print(json.dumps(out))
