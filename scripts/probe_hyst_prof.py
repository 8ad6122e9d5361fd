import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1510_06585_b200 import marrow as M, trees
N = 16384
c = M.mw_ctx_create(0, 0, 1, 1)
M.mw_ctx_set_monitoring(c, False)
g = torch.from_numpy(synth.np_u8_stream(8, 0, N * N).reshape(N, N)).cuda()
out = torch.empty_like(g)
t = trees.hysteresis()
for _ in range(4):
    f = M.mw_run(c, t, [M.arg(g), M.arg(out)]); f.wait()
print(f.result())
