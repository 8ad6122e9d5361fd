"""Runtime ordering and lifetime rules of libmarrow (marrow.h): host-staged
uploads wait for earlier work on the run's stream, runs of one ctx are FIFO
across streams, and scratch baked into a live CUDA graph survives growth."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import kernels as K  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402

DEV = "cuda:0"


def test_staged_upload_waits_for_prior_d2h_on_the_stream():
    """A pinned host input filled by an async D2H on the run's stream (behind
    a long kernel) is uploaded only after that copy landed."""
    H, W = 2048, 1024
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    s = torch.cuda.Stream()
    c = M.mw_ctx_create(0, 0, 1, 1)
    src_d = torch.from_numpy(img).to(DEV)
    torch.cuda.synchronize()
    for trial in range(3):
        h_in = torch.zeros((H, W, 4), dtype=torch.uint8).pin_memory()
        h_out = torch.zeros((H, W, 4), dtype=torch.uint8).pin_memory()
        with torch.cuda.stream(s):
            torch.cuda._sleep(50_000_000)            # ~25 ms of device time first
            h_in.copy_(src_d, non_blocking=True)    # then the input arrives
            f = M.mw_run(c, trees.filter_pipeline(), [M.arg(h_in), M.arg(h_out)], stream=s)
        f.wait()
        s.synchronize()
        assert np.array_equal(h_out.numpy(), want), trial


def test_runs_are_fifo_across_streams():
    """Two MapReduce runs of one ctx on two streams share the ctx's partials
    scratch: the second waits for the first (which sits behind a long kernel)."""
    n = 9 * (1 << 16)
    x = torch.from_numpy(synth.np_f32_um11(5, 0, n)).to(DEV)
    y = torch.ones(n, device=DEV)
    want_x = K.sum_(x.cpu().numpy())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c = M.mw_ctx_create(0, 0, 1, 2)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            torch.cuda._sleep(20_000_000)
            fa = M.mw_run(c, trees.mapreduce(False), [M.arg(x)], stream=s1)
        fb = M.mw_run(c, trees.mapreduce(False), [M.arg(y)], stream=s2)
        assert fb.wait().result()["reduced"] == float(n)
        assert fa.wait().result()["reduced"] == want_x


def test_graph_scratch_survives_growth():
    """Capture a hysteresis run (plane scratch baked into the graph), run the
    same ctx on a larger image (the scratch grows), then replay the graph:
    its output is still right and a tensor allocated after the growth is
    untouched."""
    H, W = 300, 400
    gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
    L = K.segment(gray, 173, 250)
    fixed, D = K.hyst_bfs(L)
    want = K.hyst_finalize(fixed)
    c = M.mw_ctx_create(0, 0, 1, 1)
    s = torch.cuda.Stream()
    src = torch.from_numpy(gray).to(DEV)
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    g = M.mw_graph_capture(c, trees.hysteresis(), [M.arg(src), M.arg(dst)], stream=s)
    g.launch(s)
    s.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)
    big = torch.from_numpy(synth.np_u8_stream(8, 1, 4 * H * 4 * W).reshape(4 * H, 4 * W)).to(DEV)
    bdst = torch.empty_like(big)
    with torch.cuda.stream(s):
        M.mw_run(c, trees.hysteresis(), [M.arg(big), M.arg(bdst)], stream=s).wait()
    s.synchronize()
    # fresh allocations now may take the memory the old scratch had
    probes = [torch.full((H + 2, 4 * ((W + 127) // 128)), 7, dtype=torch.int32, device=DEV)
              for _ in range(8)]
    torch.cuda.synchronize()
    dst.zero_()
    g.launch(s)
    s.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)
    assert all(bool((p == 7).all()) for p in probes)
    del g
