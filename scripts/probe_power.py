"""Sustained-load probe: per-trial time of a torch device copy (the copy peak's
method) and of the fused filter step, 8 trials of 0.2 s each, with NVML SM
clock samples — shows how much of the power-cap slowdown is the kernel's."""
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def clocks(stop, out):
    while not stop.is_set():
        out.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.005)


def trial(fn, k):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    cl, stop = [], threading.Event()
    t = threading.Thread(target=clocks, args=(stop, cl))
    t.start()
    s.record()
    for i in range(k):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    return s.elapsed_time(e) / k, statistics.median(cl) if cl else None


a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
c = [torch.empty(256 << 20, dtype=torch.uint8, device="cuda") for _ in range(2)]
d = [torch.empty_like(x) for x in c]
for which in ("copy", "filter", "copy"):
    if which == "copy":
        fn = lambda i: d[i % 2].copy_(c[i % 2])   # noqa: E731
    else:
        ctx = M.mw_ctx_create(0, 0, 1, 1)
        M.mw_ctx_set_monitoring(ctx, False)
        src = torch.empty((8192, 8192, 4), dtype=torch.uint8, device="cuda")
        synth.dev_fill_rgba(src, 3, 0)
        dst = torch.empty_like(src)
        al = M.ArgList([M.arg(src), M.arg(dst)])
        node = trees.filter_pipeline()
        fn = lambda i: M.mw_run(ctx, node, al)   # noqa: E731
    time.sleep(2.0)   # idle: power recovers
    res = [trial(fn, 2000) for _ in range(8)]
    print(which, " ".join(f"{1e3 * ms:.1f}us@{mhz}" for ms, mhz in res), flush=True)
