import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_1510_06585_b200 import marrow as M, trees
from oracle import kernels as K
def run(c, n, a):
    f = M.mw_run(c, n, a); f.wait(); return f.result()
for H, W in ((1, 1), (1, 4096), (4096, 1)):
    for ppr, d in ((1, None), (2, [0.5, 0.5])):
        c = M.mw_ctx_create(0, 0, 1, ppr)
        if d: M.mw_set_distribution(c, d)
        gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
        out = torch.empty((H, W), dtype=torch.uint8, device="cuda")
        try:
            r = run(c, trees.hysteresis(), [M.arg(torch.from_numpy(gray).cuda()), M.arg(out)])
            print(H, W, ppr, "ok", r)
        except Exception as e:
            print(H, W, ppr, "ERR", e)
        torch.cuda.synchronize()
