"""Per-rank share of the 8192^2 filter (8192/N rows) on one GPU: back-to-back
mw_run calls (pipelined) vs one CUDA graph of the B rotating-buffer runs
(mw_graph_capture_many: independent runs on up to 4 lanes, or 1 lane)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1510_06585_b200 import marrow as M, trees  # noqa: E402

W = 8192
for rows in (8192, 4096, 2048, 1024):
    nsets = max(1, -(-(512 << 20) // (rows * W * 8)))
    sets = []
    for i in range(nsets):
        a = torch.empty((rows, W, 4), dtype=torch.uint8, device="cuda")
        synth.dev_fill_rgba(a, 3, 0)
        sets.append([M.arg(a), M.arg(torch.empty_like(a))])
    t = trees.filter_pipeline()
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for mode in ("runs", "graph1", "graph4"):
        c = M.mw_ctx_create(0, 0, 1, 1)
        M.mw_ctx_set_monitoring(c, False)
        M.mw_ctx_set_run_pipelining(c, True)
        K = max(nsets, 400 // nsets * nsets)
        if mode == "runs":
            al = [M.ArgList(x) for x in sets]
            fn = lambda i: M.mw_run(c, t, al[i % nsets], stream=s)  # noqa: E731
            step = 1
        else:
            M.mw_ctx_set_tuning(c, M.MW_TUNE_GRAPH_LANES, 1 if mode == "graph1" else 4)
            g = M.mw_graph_capture_many(c, t, sets, stream=s)
            fn = lambda i: g.launch(s)  # noqa: E731
            step = nsets
        for i in range(0, 40, step):
            fn(i)
        torch.cuda.synchronize()
        e0.record(s)
        for i in range(0, K, step):
            fn(i)
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / K * 1e3
        print(f"rows={rows} sets={nsets} {mode}: {us:.2f} us/run  {rows * W * 8 / us / 1e3:.0f} GB/s", flush=True)
