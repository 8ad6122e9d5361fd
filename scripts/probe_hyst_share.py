"""Per-rank share of the 16384^2 hysteresis at N ranks (16384/N rows) on one
GPU: the share alone as one partition running exactly the global execution
count (loop_for(step, 48): the ranks of a strong-scaled run all execute the
global E = 48), against the whole image (loop_while_changed).  Missing from
the proxy: the per-pass cross-rank barrier over NVLink and the boundary strips
forced active every pass."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1510_06585_b200 import marrow as M, trees  # noqa: E402

N = 16384
g = torch.empty((N, N), dtype=torch.uint8, device="cuda")
synth.dev_fill_u8_stream(g, 8, 0)
c = M.mw_ctx_create(0, 0, 1, 1)
M.mw_ctx_set_monitoring(c, False)


def timed(tree, src, dst, K=20):
    args = M.ArgList([M.arg(src), M.arg(dst)])
    for _ in range(3):
        M.mw_run(c, tree, args).wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        f = M.mw_run(c, tree, args)
    e1.record()
    f.wait()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, f.result()


full, r = timed(trees.hysteresis(), g, torch.empty_like(g))
print(f"whole image: {full * 1e3:.1f} us per step, executions {r.get('executions')}")
for n in (2, 4, 8):
    rows = N // n
    src = g[:rows].contiguous()
    fixed = M.mw_pipeline([M.mw_kernel_segment(173, 250),
                           M.mw_loop_for(M.mw_kernel_hysteresis_step(), r.get("executions", 48)),
                           M.mw_kernel_hysteresis_finalize()])
    t, _ = timed(fixed, src, torch.empty_like(src))
    print(f"N={n}: share {rows} rows, {t * 1e3:.1f} us per step -> {full / t:.2f}x the whole image")
