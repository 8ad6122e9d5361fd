import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1510_06585_b200 import marrow as M, trees
W = 8192
for rows in (8192, 1024):
  for cfg, pipe in ((1, 0), (1, 1), (9, 1), (3, 1)):
    c = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_monitoring(c, False)
    M.mw_ctx_set_run_pipelining(c, pipe)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_RGBA_TMA, cfg)
    nsets = max(2, (512 << 20) // (rows * W * 8))
    sets = []
    for i in range(nsets):
        a = torch.empty((rows, W, 4), dtype=torch.uint8, device="cuda")
        synth.dev_fill_rgba(a, 3, 0)
        sets.append(M.ArgList([M.arg(a), M.arg(torch.empty_like(a))]))
    t = trees.filter_pipeline()
    for i in range(20):
        M.mw_run(c, t, sets[i % nsets])
    torch.cuda.synchronize()
    K = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        f = M.mw_run(c, t, sets[i % nsets])
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) / K * 1e3
    print(f"rows={rows} cfg={cfg} pipe={pipe} device_us/run={dev_us:.2f} GB/s={rows * W * 8 / dev_us / 1e3:.0f}", flush=True)
    del sets, c
