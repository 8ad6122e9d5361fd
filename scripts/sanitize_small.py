"""Small runs of every kernel family for compute-sanitizer:
memcheck / racecheck / synccheck over the TMA rings (filter, u8 chains), the
bit-plane hysteresis kernels (one-partition cooperative loop, per-partition
pass, fused multi-partition loop, pack/unpack), the cluster FFT, the
four-step FFTs at 2^16 (16 x 4096; 256 x 256 three launches and dataflow), N-body and
the MapReduce reduction — each checked against the oracle, so a sanitizer
pass is also a parity pass.  Sizes are small (sanitizers are ~100x slower)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import fft as FF  # noqa: E402
from oracle import kernels as K  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def run(c, node, args):
    return M.mw_run(c, node, args).wait().result()


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


# filter: TMA ring (W*4 a multiple of the 16 KiB chunk) and the LSU variant
for W, H in ((4096, 24), (1000, 7)):
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    for parts in (1, 3):
        c = M.mw_ctx_create(0, 0, 1, parts)
        dst = torch.empty((H, W, 4), dtype=torch.uint8, device=DEV)
        run(c, trees.filter_pipeline(), [M.arg(dev(img)), M.arg(dst)])
        check(f"filter {H}x{W} parts={parts}", np.array_equal(dst.cpu().numpy(), want))
# segmentation: TMA ring for u8 chains
vol = synth.np_u8_stream(7, 0, 6 * 64 * 256).reshape(6, 64, 256)
c = M.mw_ctx_create(0, 0, 1, 2)
dst = torch.empty_like(dev(vol))
run(c, trees.segmentation(), [M.arg(dev(vol)), M.arg(dst)])
check("segmentation", np.array_equal(dst.cpu().numpy(), K.segment(vol, 85, 170)))
# hysteresis: one partition (cooperative loop), 4 partitions fused, 4 per-pass
H, W = 200, 300
gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
L = K.segment(gray, 173, 250)
fixed, D = K.hyst_bfs(L)
want = K.hyst_finalize(fixed)
for parts, fused in ((1, 1), (4, 1), (4, 0)):
    c = M.mw_ctx_create(0, 0, 1, parts)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_FUSED, fused)
    dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
    r = run(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)])
    check(f"hysteresis parts={parts} fused={fused}",
          np.array_equal(dst.cpu().numpy(), want) and r["executions"] == D + 1)
# FFT: one cluster per transform, fused fft -> ifft
B, log2n = 2, 13
N = 1 << log2n
x = synth.np_f32_um11(11, 0, B * N * 2).reshape(B, N, 2)
c = M.mw_ctx_create(0, 0, 1, 1)
dst = torch.empty_like(dev(x))
run(c, trees.fft_pipeline(log2n), [M.arg(dev(x)), M.arg(dst)])
err = FF.rel_l2(FF.as_complex(dst.cpu().numpy()), FF.fft_chain(FF.as_complex(x), "FI"))
check("fft", bool(np.all(err <= FF.tolerance(N, 2))))
# FFT at N = 65536: the 16 x 4096 four-step path as its dataflow launch
# (default) and as three launches, the 256 x 256 one as three launches and
# as the dataflow launch (ticket + readiness counters; each dataflow launch
# bit-identical to the three launches of its decomposition)
B, N = 3, 1 << 16
x = synth.np_f32_um11(12, 0, B * N * 2).reshape(B, N, 2)
want = FF.fft_chain(FF.as_complex(x), "FI")
outs = {}
for four in (1, 4, 3, 2):
    c = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_FFT_4STEP, four)
    dst = torch.empty_like(dev(x))
    run(c, trees.fft_pipeline(16), [M.arg(dev(x)), M.arg(dst)])
    outs[four] = dst.cpu().numpy()
    err = FF.rel_l2(FF.as_complex(outs[four]), want)
    check(f"fft 2^16 form {four}", bool(np.all(err <= FF.tolerance(N, 2))))
check("fft 2^16 dataflow == three launches", np.array_equal(outs[2], outs[3]) and np.array_equal(outs[1], outs[4]))
# N-body
pos, vel = synth.np_nbody(9, 0, 700, 2.0 ** -9)
po, vo, _ = K.nbody_step(pos, vel, 1e-4, 1e-3)
c = M.mw_ctx_create(0, 0, 1, 2)
p, v = dev(pos), dev(vel)
run(c, trees.nbody(1), [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)])
check("nbody", np.allclose(p.cpu().numpy()[:, :3], po[:, :3], rtol=0, atol=1e-6))
# MapReduce
n = 3 * (1 << 16) + 5
xs = synth.np_f32_um11(5, 0, n)
ys = synth.np_f32_um11(6, 0, n)
c = M.mw_ctx_create(0, 0, 1, 2)
r = run(c, trees.mapreduce(True), [M.arg(dev(xs)), M.arg(dev(ys))])["reduced"]
check("mapreduce", abs(r - K.dot(xs, ys)) <= 1e-12 * K.abs_sum(xs, ys))
print("sanitize_small: all ok", flush=True)
