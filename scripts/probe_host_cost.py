"""Host cost of one mw_run (filter, 1024 x 8192 rows): the Python binding vs
the C call alone (prebuilt ctypes arguments), device idle between calls."""
import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import torch
from paper_1510_06585_b200 import marrow as M, trees
rows, W = 1024, 8192
c = M.mw_ctx_create(0, 0, 1, 1)
M.mw_ctx_set_monitoring(c, False)
a = torch.zeros((rows, W, 4), dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
t = trees.filter_pipeline()
args = [M.arg(a), M.arg(b)]
for _ in range(50):
    M.mw_run(c, t, args).wait()
torch.cuda.synchronize()
K = 2000
# (1) python wrapper, future kept alive in a list (no release in the loop)
keep = []
h0 = time.perf_counter()
for i in range(K):
    keep.append(M.mw_run(c, t, args))
h1 = time.perf_counter()
torch.cuda.synchronize(); keep.clear()
print(f"python mw_run: {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
al = M.ArgList(args)
keep = []
h0 = time.perf_counter()
for i in range(K):
    keep.append(M.mw_run(c, t, al))
h1 = time.perf_counter()
torch.cuda.synchronize(); keep.clear()
print(f"python mw_run (ArgList): {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
h0 = time.perf_counter()
for i in range(K):
    f = M.mw_run(c, t, al)
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"python mw_run (ArgList, futures dropped): {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
# (2) the C entry point alone
lib = M.lib()
arr = (M.mw_arg * 2)(*args)
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
outs = [ctypes.c_void_p() for _ in range(K)]
h0 = time.perf_counter()
for i in range(K):
    lib.mw_run(c.ptr, t.ptr, arr, 2, sp, ctypes.byref(outs[i]))
h1 = time.perf_counter()
torch.cuda.synchronize()
for o in outs:
    lib.mw_future_release(o)
print(f"C mw_run: {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
# (3) raw launch cost reference: torch elementwise op
h0 = time.perf_counter()
for i in range(K):
    b.add_(0)
h1 = time.perf_counter()
torch.cuda.synchronize()
print(f"torch add_: {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
# (4) graph replay of one run
s = torch.cuda.Stream()
g = M.mw_graph_capture(c, t, args, s)
if g is not None:
    for _ in range(10):
        M.mw_graph_launch(g, s) if hasattr(M, "mw_graph_launch") else None
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for i in range(K):
        M.mw_graph_launch(g, s)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"graph launch: {(h1 - h0) / K * 1e6:.2f} us/call (host)", flush=True)
