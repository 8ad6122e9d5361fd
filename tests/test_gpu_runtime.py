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


@pytest.mark.parametrize("lanes", [1, 2, 4])
def test_graph_lanes_keep_data_dependencies(lanes):
    """mw_graph_capture_many puts runs on parallel lanes only when no set
    writes what another set touches: disjoint sets give each set's own result;
    sets sharing y (a chain of dependent runs) still replay in order."""
    n = (1 << 16) + 3
    c = M.mw_ctx_create(0, 0, 1, 2)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_GRAPH_LANES, lanes)
    s = torch.cuda.Stream()
    x = [torch.from_numpy(synth.np_f32_um11(1, k * n, n)).to(DEV) for k in range(6)]
    y0 = [synth.np_f32_um11(2, k * n, n) for k in range(6)]
    y = [torch.from_numpy(v).to(DEV) for v in y0]
    torch.cuda.synchronize()
    g = M.mw_graph_capture_many(c, trees.saxpy(0.75), [[M.arg(x[k]), M.arg(y[k])] for k in range(6)], stream=s)
    g.launch(s)
    s.synchronize()
    for k in range(6):
        assert np.array_equal(y[k].cpu().numpy(), K.saxpy(0.75, x[k].cpu().numpy(), y0[k]))
    # dependent: every set updates the same y
    yd = torch.from_numpy(y0[0]).to(DEV)
    torch.cuda.synchronize()
    g2 = M.mw_graph_capture_many(c, trees.saxpy(0.75), [[M.arg(x[k]), M.arg(yd)] for k in range(6)], stream=s)
    g2.launch(s)
    s.synchronize()
    want = y0[0]
    for k in range(6):
        want = K.saxpy(0.75, x[k].cpu().numpy(), want)
    assert np.array_equal(yd.cpu().numpy(), want)
    # filter sets reading one source into distinct outputs are independent
    img = synth.np_rgba(3, 0, 64 * 128).reshape(64, 128, 4)
    src = torch.from_numpy(img).to(DEV)
    outs = [torch.empty_like(src) for _ in range(4)]
    torch.cuda.synchronize()
    g3 = M.mw_graph_capture_many(c, trees.filter_pipeline(), [[M.arg(src), M.arg(o)] for o in outs], stream=s)
    g3.launch(s)
    s.synchronize()
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    assert all(np.array_equal(o.cpu().numpy(), want) for o in outs)


@pytest.mark.parametrize("parts", [1, 3])
def test_run_pipelining_keeps_dependencies(parts):
    """mw_ctx_set_run_pipelining: runs over rotating buffer sets read ahead of
    the dependent-launch wait; a run reading what the previous run wrote
    (filter applied twice through an intermediate) still waits for it."""
    H, W = 1024, 4096   # W*4 a multiple of the TMA chunk: the TMA kernel runs
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    want2 = K.mirror(K.solarize(K.gauss_noise(want, 4, 8), 128))
    c = M.mw_ctx_create(0, 0, 1, parts)
    M.mw_ctx_set_monitoring(c, False)
    M.mw_ctx_set_run_pipelining(c, True)
    s = torch.cuda.Stream()
    srcs = [torch.from_numpy(img).to(DEV) for _ in range(3)]
    dsts = [torch.empty_like(srcs[0]) for _ in range(3)]
    mid, out = torch.empty_like(srcs[0]), torch.empty_like(srcs[0])
    node = trees.filter_pipeline()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for i in range(30):
            M.mw_run(c, node, [M.arg(srcs[i % 3]), M.arg(dsts[i % 3])], stream=s)
            if i % 7 == 3:   # a dependent pair
                M.mw_run(c, node, [M.arg(srcs[0]), M.arg(mid)], stream=s)
                M.mw_run(c, node, [M.arg(mid), M.arg(out)], stream=s)
    s.synchronize()
    assert all(np.array_equal(d.cpu().numpy(), want) for d in dsts)
    assert np.array_equal(out.cpu().numpy(), want2)
    # u8 chains (segmentation TMA ring) the same way
    vol = synth.np_u8_stream(7, 0, 64 * 256 * 256).reshape(64, 256, 256)
    vs = [torch.from_numpy(vol).to(DEV) for _ in range(2)]
    vd = [torch.empty_like(vs[0]) for _ in range(2)]
    v2 = torch.empty_like(vs[0])
    seg = trees.segmentation()
    seg2 = trees.segmentation(100, 200)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        for i in range(10):
            M.mw_run(c, seg, [M.arg(vs[i % 2]), M.arg(vd[i % 2])], stream=s)
        M.mw_run(c, seg2, [M.arg(vd[1]), M.arg(v2)], stream=s)   # reads the last run's output
    s.synchronize()
    ref = K.segment(vol, 85, 170)
    assert all(np.array_equal(d.cpu().numpy(), ref) for d in vd)
    assert np.array_equal(v2.cpu().numpy(), K.segment(ref, 100, 200))
