"""NEXT-2 on the GPU: Alg. 1 profile building and the Fig. 5
managed-run decision process, with two device classes (NEXT-4,
P:386-391) realised by the slowdown injector.  Every run's output is checked
against the oracle: the profile search only changes speed."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import kernels as K  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402

DEV = "cuda:0"


def filt(H, W):
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    return img, K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))


def two_class_ctx(slow=3.0):
    """4 partitions: 0, 1 on class 0; 2, 3 on class 1, which computes `slow`
    times slower (the builder is not told: rel_perf stays 1)."""
    c = M.mw_ctx_create(0, 0, 1, 4)
    for p in (2, 3):
        M.mw_ctx_set_device_class(c, p, 1, 1.0)
        M.mw_ctx_set_slowdown(c, p, slow)
    return c


def test_profile_build_finds_the_class_split():
    H, W = 8192, 4096
    img, want = filt(H, W)
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty_like(src)
    node = trees.filter_pipeline()
    c = two_class_ctx(3.0)
    args = [M.arg(src), M.arg(dst)]
    # time with the uniform (relative-performance) distribution
    M.mw_run(c, node, args).wait()
    M.mw_run(c, node, args).wait()
    uniform = max(M.mw_last_timings(c)[0])   # makespan of the virtual devices
    kb = M.mw_kb_open(None)
    p = M.mw_profile_defaults()
    p.executions = 2
    r = M.mw_profile_build(c, node, args, p, kb)
    shareA = r["fractions"][0] + r["fractions"][1]
    # class 1 is 3x slower: the balanced split gives class 0 three quarters
    assert 0.62 <= shareA <= 0.88, r
    assert r["runs"] > 0 and r["best_ms"] < uniform
    assert M.mw_get_distribution(c) == r["fractions"]
    found, prov, ms = M.mw_kb_find(kb, node, [H, W, 4])
    assert found and prov == M.MW_PROV_BUILT and ms == r["best_ms"]
    dst.zero_()
    M.mw_run(c, node, args).wait()
    assert np.array_equal(dst.cpu().numpy(), want)


def test_profile_build_knobs_one_class():
    H, W = 300, 500
    gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
    L = K.segment(gray, 173, 250)
    fixed, D = K.hyst_bfs(L)
    c = M.mw_ctx_create(0, 0, 1, 2)
    src = torch.from_numpy(gray).to(DEV)
    dst = torch.empty_like(src)
    node = trees.hysteresis()
    kb = M.mw_kb_open(None)
    r = M.mw_profile_build(c, node, [M.arg(src), M.arg(dst)], None, kb)
    assert r["runs"] >= 4 and r["fractions"] == [0.5, 0.5]
    for k in range(M.MW_TUNE_COUNT):
        assert M.mw_ctx_get_tuning(c, k) == r["tune"][k]
    res = M.mw_run(c, node, [M.arg(src), M.arg(dst)]).wait().result()
    assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(fixed)) and res["executions"] == D + 1
    assert M.mw_kb_find(kb, node, [H, W])[0]


def test_profile_build_restores_in_place_arguments():
    n = 5 * (1 << 16) + 9
    x = torch.from_numpy(synth.np_f32_um11(1, 0, n)).to(DEV)
    y0 = synth.np_f32_um11(2, 0, n)
    y = torch.from_numpy(y0).to(DEV)
    c = two_class_ctx(2.0)
    M.mw_profile_build(c, trees.saxpy(), [M.arg(x), M.arg(y)])
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y0)


def test_managed_runs_fig5():
    """New pair -> derived from the KB; recurrent + unbalanced -> adjusted
    (or built once when asked); results persisted with their provenance."""
    node = trees.filter_pipeline()
    kb = M.mw_kb_open(None)
    c = two_class_ctx(3.0)
    # KB knowledge: a built profile of another image size of the same SCT
    img0, _ = filt(8192, 4096)
    s0 = torch.from_numpy(img0).to(DEV)
    M.mw_profile_build(c, node, [M.arg(s0), M.arg(torch.empty_like(s0))], None, kb)
    d_built = M.mw_get_distribution(c)
    # forget: back to the relative-performance distribution
    for p in range(4):
        M.mw_ctx_set_device_class(c, p, 0 if p < 2 else 1, 1.0)
    img, want = filt(6144, 4096)
    src = torch.from_numpy(img).to(DEV)
    dst = torch.empty_like(src)
    args = [M.arg(src), M.arg(dst)]
    acts = []
    for i in range(8):
        f, act = M.mw_run_managed(c, kb, node, args)
        f.wait()
        acts.append(act)
        assert np.array_equal(dst.cpu().numpy(), want), i
    assert acts[0] == "derived" and M.mw_get_distribution(c) != [0.25] * 4
    assert all(a in ("recurrent", "adjusted") for a in acts[1:])
    M.mw_managed_flush(c)
    found, prov, ms = M.mw_kb_find(kb, node, [6144, 4096, 4])
    assert found and prov in (M.MW_PROV_DERIVED, M.MW_PROV_BALANCED) and ms > 0
    # the derived distribution came from the built profile of the other size
    assert acts[0] == "derived" and abs(d_built[0] + d_built[1] - 0.75) < 0.15
    # profile building on demand: a new pair far from balance builds once
    c2 = two_class_ctx(6.0)
    kb2 = M.mw_kb_open(None)
    prm = M.mw_managed_defaults()
    prm.build_profiles = 1
    acts = []
    for i in range(7):
        f, act = M.mw_run_managed(c2, kb2, node, args, prm)
        f.wait()
        acts.append(act)
        assert np.array_equal(dst.cpu().numpy(), want), i
    assert acts[0] == "no_knowledge" and acts.count("built") == 1, acts
    assert M.mw_kb_find(kb2, node, [6144, 4096, 4])[1] == M.MW_PROV_BUILT
