"""Per-rank cost of the filter pipeline at strong-scaling shares of the
8192^2 image (N = 1, 2, 4, 8 ranks -> 8192/N rows on one GPU): device time
per run (CUDA events over K back-to-back runs) and host time per mw_run
call (wall clock of the enqueue loop)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1510_06585_b200 import marrow as M, trees
W = 8192
for rows in [int(r) for r in os.environ.get("ROWS", "8192,4096,2048,1024").split(",")]:
    c = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_monitoring(c, False)
    nsets = max(2, (512 << 20) // (rows * W * 8))   # rotate buffers >= 2x L2
    sets = []
    for i in range(nsets):
        a = torch.empty((rows, W, 4), dtype=torch.uint8, device="cuda")
        synth.dev_fill_rgba(a, 3, 0) if hasattr(synth, "dev_fill_rgba") else a.random_(0, 255)
        sets.append([M.arg(a), M.arg(torch.empty_like(a))])
    t = trees.filter_pipeline()
    for i in range(20):
        M.mw_run(c, t, sets[i % nsets])
    torch.cuda.synchronize()
    K = 400
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for i in range(K):
        f = M.mw_run(c, t, sets[i % nsets])
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / K * 1e3
    print(f"rows={rows} device_us/run={dev_us:.2f} host_us/call={(h1 - h0) / K * 1e6:.2f} "
          f"GB/s={rows * W * 8 / dev_us / 1e3:.0f}", flush=True)
