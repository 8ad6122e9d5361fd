"""Time the one-partition bit-plane hysteresis on the 16384^2 config image for
every built (T, ROWS) pair of the plane loop (MW_TUNE_HYST_T / _ROWS)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1510_06585_b200 import marrow as M, trees
N = 16384
g = torch.from_numpy(synth.np_u8_stream(8, 0, N * N).reshape(N, N)).cuda()
out = torch.empty_like(g)
for T, R in [(4, 32), (6, 32), (8, 32), (8, 40), (12, 40), (6, 48), (8, 48)]:
    c = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_monitoring(c, False)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, 8)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_ROWS, R)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, T)
    t = trees.hysteresis()
    for _ in range(3):
        M.mw_run(c, t, [M.arg(g), M.arg(out)]).wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20):
        f = M.mw_run(c, t, [M.arg(g), M.arg(out)])
    e1.record(); f.wait(); torch.cuda.synchronize()
    print(f"T={T} ROWS={R} ms/run={e0.elapsed_time(e1)/20:.4f} E={f.result()['executions']}", flush=True)
