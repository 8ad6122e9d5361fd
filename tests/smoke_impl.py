"""__graft_entry__.smoke(): one small invocation of the hot path on cuda:0,
checked against the oracle (test infrastructure)."""
import numpy as np


def run():
    import torch

    import synth
    from oracle import kernels as K
    from paper_1510_06585_b200 import marrow as M
    from paper_1510_06585_b200 import trees

    assert torch.cuda.is_available(), "smoke() needs a CUDA device"
    dev = "cuda:0"
    ctx = M.mw_ctx_create(0, 0, 1, 2)
    M.mw_set_distribution(ctx, [0.6, 0.4])
    # fused filter pipeline (the headline workload), 2 partitions
    H, W = 96, 128
    img = synth.np_rgba(synth.SEED_IMAGE, 0, H * W).reshape(H, W, 4)
    src = torch.from_numpy(img).to(dev)
    dst = torch.empty_like(src)
    M.mw_run(ctx, trees.filter_pipeline(), [M.arg(src), M.arg(dst)]).wait()
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    assert np.array_equal(dst.cpu().numpy(), want), "filter pipeline mismatch"
    # hysteresis loop (halo exchange + device loop condition)
    gray = synth.np_u8_stream(synth.SEED_HYST, 0, 64 * 80).reshape(64, 80)
    out = torch.empty((64, 80), dtype=torch.uint8, device=dev)
    f = M.mw_run(ctx, trees.hysteresis(), [M.arg(torch.from_numpy(gray).to(dev)), M.arg(out)])
    r = f.wait().result()
    fixed, D = K.hyst_bfs(K.segment(gray, 173, 250))
    assert np.array_equal(out.cpu().numpy(), K.hyst_finalize(fixed)) and r["executions"] == D + 1
    # MapReduce dot (fp64 chunk partials + canonical combine)
    n = 3 * (1 << 16) + 7
    x, y = synth.np_f32_um11(5, 0, n), synth.np_f32_um11(6, 0, n)
    got = M.mw_run(ctx, trees.mapreduce(True), [M.arg(torch.from_numpy(x).to(dev)),
                                               M.arg(torch.from_numpy(y).to(dev))]).wait().result()
    assert abs(got["reduced"] - K.dot(x, y)) <= 1e-12 * K.abs_sum(x, y)
    # FFT -> IFFT pipeline (NEXT-3): 3 transforms of 8192 points over 2 partitions
    from oracle import fft as FF
    xf = synth.np_f32_um11(11, 0, 2 * 3 * 8192).reshape(3, 8192, 2)
    yf = torch.empty((3, 8192, 2), dtype=torch.float32, device=dev)
    M.mw_run(ctx, trees.fft_pipeline(13), [M.arg(torch.from_numpy(xf).to(dev)), M.arg(yf)]).wait()
    got = FF.as_complex(yf.cpu().numpy())
    assert FF.rel_l2(got, FF.fft_chain(FF.as_complex(xf), "FI")).max() <= FF.tolerance(8192, 2)
    assert M.mw_ctx_launch_count(ctx) > 0
    ctx.destroy()
    print("smoke OK")
