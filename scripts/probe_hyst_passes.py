"""Time the one-partition bit-plane hysteresis loop for a fixed number of
executions n (loop_for) on the 16384^2 config image: the per-pass cost of the
dense temporally blocked loop (differences between successive n)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_1510_06585_b200 import marrow as M, trees

N = 16384
c = M.mw_ctx_create(0, 0, 1, 1)
M.mw_ctx_set_monitoring(c, False)
g = torch.empty((N, N), dtype=torch.uint8, device="cuda")
g.copy_(torch.from_numpy(synth.np_u8_stream(8, 0, N * N).reshape(N, N)))
out = torch.empty_like(g)
def tree(n):
    if n is None:
        return trees.hysteresis()
    return M.mw_pipeline([M.mw_kernel_segment(173, 250),
                          M.mw_loop_for(M.mw_kernel_hysteresis_step(), n),
                          M.mw_kernel_hysteresis_finalize()])
for n in [0, 1, 8, 16, 24, 32, 40, 48, None]:
    t = tree(n if n else 1) if n != 0 else None
    if t is None:
        t = M.mw_pipeline([M.mw_kernel_segment(173, 250), M.mw_kernel_hysteresis_finalize()])
    args = [M.arg(g), M.arg(out)]
    for _ in range(3):
        M.mw_run(c, t, args).wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    K = 20
    for _ in range(K):
        f = M.mw_run(c, t, args)
    e1.record()
    f.wait()
    torch.cuda.synchronize()
    print(f"n={n} ms/run={e0.elapsed_time(e1)/K:.4f} result={f.result()}", flush=True)
