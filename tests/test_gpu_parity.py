"""CUDA path (through the C-ABI) vs the oracle, element by element.

Bit-exact for integer work (filter, segmentation, hysteresis, traits) and
for saxpy (single-rounding fma on both sides); MapReduce within 1e-5
relative (north_star) — in practice ~1e-15; N-body accelerations within the
SURVEY §8(c) c.5 bounds (1e-5 relative, conditioning-aware).
"""
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import kernels as K  # noqa: E402
from oracle import partition as OP  # noqa: E402
from oracle import sct  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402

DEV = "cuda:0"


def ctx(ppr=1, dist=None):
    c = M.mw_ctx_create(0, 0, 1, ppr)
    if dist is not None:
        M.mw_set_distribution(c, dist)
    return c


def run(c, node, args):
    f = M.mw_run(c, node, args)
    f.wait()
    return f.result()


def dists(k, rng, n=3):
    out = [[1.0 / k] * k]
    for _ in range(n):
        w = rng.integers(0, 4, size=k).astype(float)
        if w.sum() == 0:
            w[0] = 1
        out.append(list(w / w.sum()))
    return out


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


# ----------------------------------------------------------------- saxpy
@pytest.mark.parametrize("n", [1, 3, 4, 67, 1000, (1 << 20) + 3])
def test_saxpy_bitwise(n):
    rng = np.random.default_rng(n)
    x = synth.np_f32_um11(1, 0, n)
    y = synth.np_f32_um11(2, 0, n)
    want = K.saxpy(2.5, x, y)
    for d in dists(4, rng):
        c = ctx(4, d)
        xd, yd = dev(x), dev(y)
        run(c, trees.saxpy(2.5), [M.arg(xd), M.arg(yd)])
        assert np.array_equal(yd.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_saxpy_rounding_pin_and_chain():
    a = np.float32(1 + 2.0 ** -12)
    x = np.full(9, a, np.float32)
    y = np.full(9, -(1 + 2.0 ** -11), np.float32)
    xd, yd = dev(x), dev(y)
    run(ctx(), trees.saxpy(float(a)), [M.arg(xd), M.arg(yd)])
    assert np.all(yd.cpu().numpy() == 2.0 ** -24)
    # Loop equals its unrolled body, and both equal the oracle's sequential evaluation
    x = synth.np_f32_um11(1, 0, 1001)
    y = synth.np_f32_um11(2, 0, 1001)
    want = sct.evaluate(sct.LoopFor(sct.Leaf("saxpy", {"a": 0.75}), 20), (x, y)).value[1]
    yd = dev(y)
    run(ctx(), M.mw_loop_for(M.mw_kernel_saxpy(0.75), 20), [M.arg(dev(x)), M.arg(yd)])
    assert np.array_equal(yd.cpu().numpy(), want)


# ----------------------------------------------------------------- filter pipeline
def oracle_filter(img, seed=4, S=8, T=128):
    return sct.evaluate(sct.Pipeline([sct.Leaf("gauss_noise", {"seed": seed, "scale": S}),
                                      sct.Leaf("solarize", {"threshold": T}),
                                      sct.Leaf("mirror")]), img).value


@pytest.mark.parametrize("H,W", [(2, 4), (37, 64), (33, 61), (5, 1), (256, 512), (900, 1440), (1125, 1800),
                                 (33, 4096), (7, 8192)])
def test_filter_pipeline_bitwise(H, W):
    rng = np.random.default_rng(H * 7 + W)
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = oracle_filter(img)
    for d in dists(3, rng):
        c = ctx(3, d)
        src, dst = dev(img), torch.empty((H, W, 4), dtype=torch.uint8, device=DEV)
        run(c, trees.filter_pipeline(), [M.arg(src), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want), d


def test_filter_golden_vector_and_fused_equals_unfused():
    W, H = 4, 2
    img = np.array([[(16 * i) % 256, (255 - 16 * i) % 256, (37 * i) % 256, 200]
                    for i in range(W * H)], dtype=np.uint8).reshape(H, W, 4)
    c = ctx()
    src, dst = dev(img), torch.empty_like(dev(img))
    run(c, trees.filter_pipeline(), [M.arg(src), M.arg(dst)])
    from tests.golden_io import filter_w4h2
    _, _, rows = filter_w4h2()
    assert [[tuple(int(v) for v in px) for px in row] for row in dst.cpu().numpy()] == rows
    # three separate Map runs (unfused) give the same bytes as the fused pipeline
    img = synth.np_rgba(3, 0, 123 * 77).reshape(123, 77, 4)
    a, b, o = dev(img), torch.empty((123, 77, 4), dtype=torch.uint8, device=DEV), None
    run(c, M.mw_map(M.mw_kernel_gauss_noise(4, 8)), [M.arg(a), M.arg(b)])
    o1 = torch.empty_like(b)
    run(c, M.mw_map(M.mw_kernel_solarize(128)), [M.arg(b), M.arg(o1)])
    o = torch.empty_like(b)
    run(c, M.mw_map(M.mw_kernel_mirror()), [M.arg(o1), M.arg(o)])
    fused = torch.empty_like(b)
    run(c, trees.filter_pipeline(), [M.arg(dev(img)), M.arg(fused)])
    assert torch.equal(o, fused)
    assert np.array_equal(o.cpu().numpy(), oracle_filter(img))


def test_rgba_long_chains_and_loops():
    img = synth.np_rgba(5, 0, 41 * 36).reshape(41, 36, 4)
    c = ctx(2, [0.3, 0.7])
    # LoopFor(mirror, 2) is the identity; long chains split into several launches
    dst = torch.empty((41, 36, 4), dtype=torch.uint8, device=DEV)
    run(c, M.mw_loop_for(M.mw_kernel_mirror(), 2), [M.arg(dev(img)), M.arg(dst)])
    assert np.array_equal(dst.cpu().numpy(), img)
    body = sct.Pipeline([sct.Leaf("gauss_noise", {"seed": 11, "scale": 3}), sct.Leaf("mirror"),
                         sct.Leaf("solarize", {"threshold": 90})])
    want = sct.evaluate(sct.LoopFor(body, 9), img).value
    mb = M.mw_pipeline([M.mw_kernel_gauss_noise(11, 3), M.mw_kernel_mirror(), M.mw_kernel_solarize(90)])
    run(c, M.mw_loop_for(mb, 9), [M.arg(dev(img)), M.arg(dst)])
    assert np.array_equal(dst.cpu().numpy(), want)
    run(c, M.mw_loop_for(mb, 0), [M.arg(dev(img)), M.arg(dst)])
    assert np.array_equal(dst.cpu().numpy(), img)


def test_filter_host_staged_equals_device():
    H, W = 700, 1024
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    src = torch.from_numpy(img).pin_memory()
    dst = torch.empty((H, W, 4), dtype=torch.uint8).pin_memory()
    c = ctx(2, [0.6, 0.4])
    run(c, trees.filter_pipeline(), [M.arg(src), M.arg(dst)])
    assert np.array_equal(dst.numpy(), oracle_filter(img))


# ----------------------------------------------------------------- segmentation
@pytest.mark.parametrize("shape", [(37, 16, 48), (5, 3, 7), (64, 64, 64), (1, 1, 1)])
@pytest.mark.parametrize("lohi", [(85, 170), (0, 0), (256, 256), (0, 256), (128, 200), (3, 129)])
def test_segmentation_bitwise(shape, lohi):
    n = int(np.prod(shape))
    vol = synth.np_u8_stream(7, 0, n).reshape(shape)
    want = K.segment(vol, *lohi)
    c = ctx(3, [0.5, 0.0, 0.5])
    dst = torch.empty(shape, dtype=torch.uint8, device=DEV)
    run(c, trees.segmentation(*lohi), [M.arg(dev(vol)), M.arg(dst)])
    assert np.array_equal(dst.cpu().numpy(), want)


# ----------------------------------------------------------------- MapReduce
@pytest.mark.parametrize("n", [1, 1000, 1 << 16, (1 << 16) + 1, 3 * (1 << 16) + 12345, 1 << 22])
@pytest.mark.parametrize("dot", [False, True])
def test_mapreduce_vs_oracle_and_canonical(n, dot):
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    want = K.dot(x, y) if dot else K.sum_(x)
    scale = K.abs_sum(x, y if dot else None)
    args = [M.arg(dev(x))] + ([M.arg(dev(y))] if dot else [])
    rng = np.random.default_rng(n)
    vals = set()
    for d in dists(4, rng):
        r = run(ctx(4, d), trees.mapreduce(dot), args)["reduced"]
        tol = 1e-5 * abs(want) if abs(want) >= 1e-5 * scale else 1e-5 * scale
        assert abs(r - want) <= tol
        assert abs(r - want) <= 1e-12 * scale + 1e-300   # per-element fp64 accuracy
        vals.add(np.float64(r).tobytes())
    assert len(vals) == 1, "canonical mode must be bit-identical across distributions"


@pytest.mark.parametrize("n", [1, 5, (1 << 16) - 1, 1 << 16, 3 * (1 << 16) + 17, (1 << 22) + 5])
@pytest.mark.parametrize("dot", [False, True])
def test_mapreduce_reduction_stage(n, dot):
    """Device reduction stage (NEXT-4, R28): MAX / MIN bit-exact against
    the oracle's serial fold for every distribution; SUM bit-identical to the
    canonical mw_map_reduce(+)."""
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    args = [M.arg(dev(x))] + ([M.arg(dev(y))] if dot else [])
    rng = np.random.default_rng(n + dot)
    for op, is_min in ((M.MW_REDUCE_MAX, False), (M.MW_REDUCE_MIN, True)):
        want = K.fold_extreme(x, y if dot else None, is_min)
        for k, d in [(1, None)] + [(4, dd) for dd in dists(4, rng, 2)]:
            r = run(ctx(k, d), trees.mapreduce_sct(op, dot), args)
            assert r["reduced"] == want and r["reduced32"] == float(np.float32(want))
    canon = run(ctx(), trees.mapreduce(dot), args)["reduced"]
    for k, d in [(1, None), (3, [0.5, 0.0, 0.5])]:
        assert run(ctx(k, d), trees.mapreduce_sct(M.MW_REDUCE_SUM, dot), args)["reduced"] == canon


def test_mapreduce_reduction_stage_edges():
    e = torch.zeros(0, device=DEV)
    assert run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_MAX, False), [M.arg(e)])["reduced"] == -np.inf
    assert run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_MIN, False), [M.arg(e)])["reduced"] == np.inf
    assert run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_SUM, False), [M.arg(e)])["reduced"] == 0.0
    z = torch.tensor([np.nan, -2.0, np.nan, 3.0, np.nan], dtype=torch.float32, device=DEV)
    assert run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_MAX, False), [M.arg(z)])["reduced"] == 3.0
    assert run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_MIN, False), [M.arg(z)])["reduced"] == -2.0
    # the maximum in the ragged tail of the last chunk, and the exact product
    n = 5 * (1 << 16) + 9
    x = torch.full((n,), -1.0, device=DEV)
    x[n - 2] = 1 + 2.0 ** -23
    r = run(ctx(3, [0.2, 0.3, 0.5]), trees.mapreduce_sct(M.MW_REDUCE_MAX, True), [M.arg(x), M.arg(x)])
    assert r["reduced"] == (1 + 2.0 ** -23) ** 2
    # a 2^20-element minimum on one partition
    xs = dev(synth.np_f32_um11(5, 0, 1 << 20))
    want = run(ctx(), trees.mapreduce_sct(M.MW_REDUCE_MIN, False), [M.arg(xs)])["reduced"]
    assert want == K.fold_extreme(xs.cpu().numpy(), None, True)


def test_mapreduce_closed_forms():
    n = (1 << 25) + 3
    r = run(ctx(), trees.mapreduce(False), [M.arg(torch.ones(n, device=DEV))])
    assert r["reduced"] == float(n) and r["reduced32"] == float(np.float32(n))
    x = (torch.arange(1 << 20, device=DEV) % 1024).float() / 1024
    assert run(ctx(), trees.mapreduce(False), [M.arg(x)])["reduced"] == 523776.0
    e = torch.zeros(1000, device=DEV)
    e[17] = 1
    y = dev(synth.np_f32_um11(6, 0, 1000))
    assert run(ctx(), trees.mapreduce(True), [M.arg(y), M.arg(e)])["reduced"] == float(y[17])
    assert run(ctx(), trees.mapreduce(False), [M.arg(torch.zeros(0, device=DEV))])["reduced"] == 0.0


# ----------------------------------------------------------------- hysteresis
def oracle_hyst(gray, lo=173, hi=250):
    L = K.segment(gray, lo, hi)
    fixed, D = K.hyst_bfs(L)
    return K.hyst_finalize(fixed), D


def pctx(ppr, dist, planes):
    c = ctx(ppr, dist)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_PLANES, planes)
    return c


@pytest.mark.parametrize("H,W", [(64, 64), (100, 37), (257, 300), (1, 1), (3, 1000)])
@pytest.mark.parametrize("ce", [1, 4, 16])
@pytest.mark.parametrize("planes", [0, 1])
def test_hysteresis_bitwise_and_E(H, W, ce, planes):
    rng = np.random.default_rng(H * W + ce)
    gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)
    # planes=0: byte stencil with one-row halo exchange; planes=1: bit planes,
    # one partition -> cooperative device-side loop, several -> per-pass
    # kernels with T-row plane halos
    for k, d in [(3, x) for x in dists(3, rng, 2) + [[0.0, 1.0, 0.0]]] + [(1, [1.0])]:
        c = pctx(k, d, planes)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(check_every=ce), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want), d
        assert r["executions"] == D + 1 and r["converged"]


@pytest.mark.parametrize("planes", [0, 1])
def test_hysteresis_long_chains_partitions(planes):
    # a long weak snake crossing every partition boundary (1-row partitions)
    H, W = 12, 40
    L = np.zeros((H, W), np.uint8)
    L[:, :] = 128
    L[::2, 1:] = 0
    L[1::2, :-1] = 0
    L[1::4, -1] = 128
    L[3::4, 0] = 128
    L[0, 0] = 255
    gray = np.where(L == 255, 255, np.where(L == 128, 200, 0)).astype(np.uint8)
    want, D = oracle_hyst(gray)
    for d in ([1 / 12] * 12, [0.5] + [0.5 / 11] * 11, [0.25, 0.0, 0.5, 0.25] + [0.0] * 8):
        c = pctx(12, d, planes)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(check_every=3), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want) and r["executions"] == D + 1


@pytest.mark.parametrize("planes", [0, 1])
def test_hysteresis_loop_for_and_max_iters(planes):
    rng = np.random.default_rng(0)
    gray = rng.integers(0, 256, size=(50, 70), dtype=np.uint8)
    L = K.segment(gray, 173, 250)
    _, D = K.hyst_bfs(L)
    c = pctx(2, None, planes)
    for n in (0, 1, 2, 5):
        dst = torch.empty((50, 70), dtype=torch.uint8, device=DEV)
        run(c, M.mw_loop_for(M.mw_kernel_hysteresis_step(), n), [M.arg(dev(L)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), K.hyst_bfs(L, n)[0])
    for cc in (c, pctx(1, None, planes)):   # 2 partitions and 1 partition
        if D >= 2:
            dst = torch.empty((50, 70), dtype=torch.uint8, device=DEV)
            r = run(cc, trees.hysteresis(max_iters=2), [M.arg(dev(gray)), M.arg(dst)])
            assert r["executions"] == 2 and not r["converged"]
            assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(K.hyst_bfs(L, 2)[0]))
        for n in (0, 1, 3, D + 5):   # pipeline(threshold, loop_for(step, n), finalize)
            tree = M.mw_pipeline([M.mw_kernel_segment(173, 250),
                                  M.mw_loop_for(M.mw_kernel_hysteresis_step(), n),
                                  M.mw_kernel_hysteresis_finalize()])
            dst = torch.empty((50, 70), dtype=torch.uint8, device=DEV)
            run(cc, tree, [M.arg(dev(gray)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(K.hyst_bfs(L, n)[0])), n
        # threshold + loop only (labels out, no finalize)
        tree = M.mw_pipeline([M.mw_kernel_segment(173, 250),
                              M.mw_loop_while_changed(M.mw_kernel_hysteresis_step(), 1000)])
        dst = torch.empty((50, 70), dtype=torch.uint8, device=DEV)
        r = run(cc, tree, [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), K.hyst_bfs(L)[0]) and r["executions"] == D + 1


@pytest.mark.parametrize("W", [4096, 8192 + 4096])
def test_hysteresis_wide_rows(W):
    """Rows of a multiple of 4096 pixels take the warp-wide finalize unpack."""
    H = 45
    gray = synth.np_u8_stream(8, 3, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)
    for k, d in ((1, [1.0]), (3, [0.3, 0.3, 0.4])):
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(pctx(k, d, 1), trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want) and r["executions"] == D + 1


@pytest.mark.parametrize("T", [4, 6, 8, 12])
def test_hysteresis_planes_partitions_depths(T):
    """Several partitions on the bit-plane path: T-row halos, T clamped to the
    smallest active partition, boundary tiles always active."""
    rng = np.random.default_rng(T)
    H, W = 700, 1100
    gray = synth.np_u8_stream(8, 7, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)
    for k, d in [(4, x) for x in dists(4, rng, 2)] + [(5, [0.2, 0.003, 0.0, 0.397, 0.4])]:
        c = pctx(k, d, 1)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, 8)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_ROWS, 40 if T in (8, 12) else 32)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, T)
        for ce in (1, 5):
            dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
            r = run(c, trees.hysteresis(check_every=ce), [M.arg(dev(gray)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), want), (d, ce)
            assert r["executions"] == D + 1 and r["converged"]
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(max_iters=D - 3), [M.arg(dev(gray)), M.arg(dst)])
        L = K.segment(gray, 173, 250)
        assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(K.hyst_bfs(L, D - 3)[0]))
        assert r["executions"] == D - 3 and not r["converged"]


# ----------------------------------------------------------------- N-body
def _nb_check(acc_g, acc_o, cond):
    err = np.linalg.norm(acc_g - acc_o, axis=1)
    nrm = np.linalg.norm(acc_o, axis=1)
    C = cond
    ok_cond = (C / np.maximum(nrm, 1e-300)) <= 1e3
    assert np.all(err[ok_cond] <= 1e-5 * nrm[ok_cond])
    assert np.all(err <= 1e-5 * np.maximum(nrm, 1e-3 * C))
    assert np.linalg.norm(acc_g - acc_o) <= 1e-5 * np.linalg.norm(acc_o)


@pytest.mark.parametrize("N", [1, 2, 300, 1024, 4096 + 256])
def test_nbody_accel_vs_oracle(N):
    pos, _ = synth.np_nbody(9, 0, N, 2.0 ** -10)
    acc_o, cond = K.nbody_accel(pos, 1e-4)
    c = ctx(3, [0.2, 0.5, 0.3])
    acc = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    run(c, M.mw_kernel_nbody_accel(1e-4), [M.arg(dev(pos), M.MW_COPY), M.arg(acc)])
    _nb_check(acc.cpu().numpy()[:, :3].astype(np.float64), acc_o, cond)


def test_nbody_step_vs_oracle_and_partition_invariance():
    N = 2048 + 512
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -11)
    po, vo, acc_o = K.nbody_step(pos, vel, 1e-4, 1e-3)
    _, cond = K.nbody_accel(pos, 1e-4)
    results = []
    for d in ([1.0, 0.0, 0.0, 0.0], [0.25] * 4, [0.1, 0.4, 0.0, 0.5]):
        c = ctx(4, d)
        p, v = dev(pos), dev(vel)
        run(c, trees.nbody(1), [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)])
        dv = (v.cpu().numpy()[:, :3].astype(np.float64) - vel[:, :3]) / np.float64(np.float32(1e-3))
        _nb_check(dv, acc_o, cond)
        results.append((p.cpu().numpy().tobytes(), v.cpu().numpy().tobytes()))
    assert all(r == results[0] for r in results), "trajectories must not depend on the distribution"


def test_nbody_loop_equals_repeated_runs():
    N = 1024
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -10)
    c = ctx(2)
    p1, v1 = dev(pos), dev(vel)
    run(c, trees.nbody(3), [M.arg(p1, M.MW_COPY), M.arg(v1, M.MW_COPY)])
    p2, v2 = dev(pos), dev(vel)
    for _ in range(3):
        run(c, trees.nbody(1), [M.arg(p2, M.MW_COPY), M.arg(v2, M.MW_COPY)])
    assert torch.equal(p1, p2) and torch.equal(v1, v2)


# ----------------------------------------------------------------- traits / partition
def test_debug_traits_reproduce_partitions():
    rng = np.random.default_rng(1)
    for trial in range(30):
        k = int(rng.integers(1, 6))
        L = int(rng.integers(0, 500))
        epu = int(rng.choice([1, 2, 4, 6]))
        d = dists(k, rng, 1)[-1]
        c = ctx(k, d)
        out = torch.full((L, 2), -1, dtype=torch.int64, device=DEV)
        node = M.mw_kernel_debug_traits(epu, 1)
        run(c, node, [M.arg(out)])
        off, ln = OP.partition(L, OP.granule([(epu, 1)]), d)
        want = np.concatenate([np.tile([n, o], (n, 1)) for o, n in zip(off, ln)] + [np.zeros((0, 2))]).astype(np.int64)
        assert np.array_equal(out.cpu().numpy(), want.reshape(L, 2))
        assert M.mw_partition(c, node, L) == (off, ln)


# ----------------------------------------------------------------- rebalancing
def test_rebalance_slowdown_nbody_bitwise():
    N = 8192
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -13)
    c = ctx(4)
    M.mw_ctx_set_slowdown(c, 3, 8.0)
    p, v = dev(pos), dev(vel)
    node = trees.nbody(1)
    trig_at = None
    for step in range(6):
        run(c, node, [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)])
        if M.mw_rebalance(c) and trig_at is None:
            trig_at = step
    assert trig_at == 2, "three consecutive unbalanced runs trigger (lbt 0.963)"
    d = M.mw_get_distribution(c)
    assert d[3] < 0.5 * d[0]
    # identical trajectory to a run that never rebalanced
    c2 = ctx(1)
    p2, v2 = dev(pos), dev(vel)
    run(c2, trees.nbody(6), [M.arg(p2, M.MW_COPY), M.arg(v2, M.MW_COPY)])
    assert torch.equal(p, p2) and torch.equal(v, v2)


# ----------------------------------------------------------------- full config sizes
@pytest.mark.slow
def test_config_filter_8192_bitwise():
    H = W = 8192
    src = torch.empty((H, W, 4), dtype=torch.uint8, device=DEV)
    synth.dev_fill_rgba(src, synth.SEED_IMAGE, 0)
    dst = torch.empty_like(src)
    run(ctx(), trees.filter_pipeline(), [M.arg(src), M.arg(dst)])
    img = synth.host_rgba(synth.SEED_IMAGE, 0, H * W).reshape(H, W, 4)
    assert np.array_equal(src.cpu().numpy(), img)
    got = dst.cpu().numpy()
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    assert np.array_equal(got, want)
    assert zlib.crc32(got.tobytes()) == 0x60CC7642


@pytest.mark.slow
def test_config_hysteresis_16384():
    n = 16384
    src = torch.empty((n, n), dtype=torch.uint8, device=DEV)
    synth.dev_fill_u8_stream(src, synth.SEED_HYST, 0)
    gray = synth.host_u8_stream(synth.SEED_HYST, 0, n * n).reshape(n, n)
    want, D = oracle_hyst(gray)
    # one partition (the cooperative plane loop, bench default) and the
    # per-partition pass protocol of bench --parts / N > 1 (T-row plane halos,
    # lagged loop condition), uneven and with a zero share
    for k, d in [(1, None), (8, [0.05, 0.2, 0.1, 0.15, 0.1, 0.1, 0.2, 0.1]), (3, [0.5, 0.0, 0.5])]:
        dst = torch.zeros_like(src)
        r = run(ctx(k, d), trees.hysteresis(), [M.arg(src), M.arg(dst)])
        assert r["executions"] == D + 1 == 48, (k, d)
        assert np.array_equal(dst.cpu().numpy(), want), (k, d)


@pytest.mark.slow
def test_config_segmentation_bitwise():
    shape = (512, 1024, 1024)
    src = torch.empty(shape, dtype=torch.uint8, device=DEV)
    synth.dev_fill_u8_stream(src, synth.SEED_SEGMENT, 0)
    dst = torch.empty_like(src)
    run(ctx(), trees.segmentation(), [M.arg(src), M.arg(dst)])
    got = dst.cpu().numpy()
    assert zlib.crc32(got.data) == 0x9417CCB7
    vol = synth.host_u8_stream(synth.SEED_SEGMENT, 0, got.size)
    assert np.array_equal(got.ravel(), K.segment(vol, 85, 170))


@pytest.mark.slow
def test_config_mapreduce_2p30():
    n = 1 << 30
    x = torch.empty(n, dtype=torch.float32, device=DEV)
    y = torch.empty(n, dtype=torch.float32, device=DEV)
    synth.dev_fill_f32_um11(x, synth.SEED_MR_X, 0)
    synth.dev_fill_f32_um11(y, synth.SEED_MR_Y, 0)
    s = run(ctx(), trees.mapreduce(False), [M.arg(x)])["reduced"]
    d = run(ctx(), trees.mapreduce(True), [M.arg(x), M.arg(y)])["reduced"]
    exact_s = -383760319397 / 2.0 ** 23
    exact_d = 643773335475643653 / 2.0 ** 46
    assert abs(s - exact_s) <= 1e-12 * abs(exact_s)
    assert abs(d - exact_d) <= 1e-12 * abs(exact_d)


@pytest.mark.slow
def test_config_nbody_2p20_sampled():
    N = 1 << 20
    pos = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    synth.dev_fill_nbody(pos, None, synth.SEED_NBODY, 0, 2.0 ** -20)
    acc = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    run(ctx(), M.mw_kernel_nbody_accel(1e-4), [M.arg(pos, M.MW_COPY), M.arg(acc)])
    hp = pos.cpu().numpy()
    samples = np.concatenate([synth.nbody_sample_indices(N, 256), [0, N - 1, 284297]])
    acc_o, cond = K.nbody_accel(hp, 1e-4, targets=samples)
    _nb_check(acc.cpu().numpy()[samples, :3].astype(np.float64), acc_o, cond)


@pytest.mark.slow
def test_config_fft_512x65536_sampled():
    """The bench's FFT workload (512 x 65536 points, fused fft -> ifft, one
    launch): sampled transforms against the fp64 oracle, plus the forward
    leaf alone on the same batch."""
    B, N = 512, 1 << 16
    src = torch.empty((B, N, 2), dtype=torch.float32, device=DEV)
    synth.dev_fill_f32_um11(src, 11, 0)
    dst = torch.empty_like(src)
    run(ctx(), trees.fft_pipeline(16), [M.arg(src), M.arg(dst)])
    rows = [0, 1, 255, 256, 300, 511]
    x = np.stack([synth.np_f32_um11(11, r * 2 * N, 2 * N).reshape(N, 2) for r in rows])
    assert np.array_equal(src.cpu().numpy()[rows], x)
    _fft_check(dst.cpu().numpy()[rows], x, "FI")
    run(ctx(), M.mw_kernel_fft(16, False), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy()[rows], x, "F")


# ----------------------------------------------------------------- NCCL call sites (1-rank communicator)
def test_nccl_communicator_paths():
    """force_nccl routes the MapReduce merge and the loop-condition reduction
    through a real (1-rank) NCCL communicator: the same call sites a
    multi-GPU run uses; results must be identical to the device-copy path."""
    nid = M.mw_nccl_unique_id()
    c = M.mw_ctx_create(0, 0, 1, 3, nid, force_nccl=True)
    M.mw_set_distribution(c, [0.5, 0.25, 0.25])
    n = 5 * (1 << 16) + 77
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    xd, yd = dev(x), dev(y)
    r = run(c, trees.mapreduce(True), [M.arg(xd), M.arg(yd)])["reduced"]
    r0 = run(ctx(3, [0.5, 0.25, 0.25]), trees.mapreduce(True), [M.arg(xd), M.arg(yd)])["reduced"]
    assert r == r0 and abs(r - K.dot(x, y)) <= 1e-12 * K.abs_sum(x, y)
    gray = synth.np_u8_stream(8, 0, 90 * 70).reshape(90, 70)
    want, D = oracle_hyst(gray)
    for planes in (1, 0):   # T-row plane halos / one-row byte halos
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_PLANES, planes)
        dst = torch.empty((90, 70), dtype=torch.uint8, device=DEV)
        res = run(c, trees.hysteresis(check_every=2), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want) and res["executions"] == D + 1
    ms, wall = M.mw_last_timings(c)
    assert len(ms) == 3 and all(t > 0 for t in ms) and wall > 0
    c.destroy()


# ----------------------------------------------------------------- CUDA graph replay
def test_graph_capture_replay():
    s = torch.cuda.Stream()
    c = ctx(2, [0.25, 0.75])
    x = dev(synth.np_f32_um11(1, 0, 4099))
    y0 = synth.np_f32_um11(2, 0, 4099)
    y = dev(y0)
    with torch.cuda.stream(s):
        g = M.mw_graph_capture(c, trees.saxpy(0.5), [M.arg(x), M.arg(y)], s)
        for _ in range(7):
            g.launch(s)
    s.synchronize()
    want = y0
    for _ in range(7):
        want = K.saxpy(0.5, synth.np_f32_um11(1, 0, 4099), want)
    assert np.array_equal(y.cpu().numpy(), want) and g.kernels >= 2
    # MapReduce result through the graph's pinned slot
    xs = synth.np_f32_um11(5, 0, 3 * (1 << 16) + 5)
    xd = dev(xs)
    with torch.cuda.stream(s):
        g2 = M.mw_graph_capture(c, trees.mapreduce(False), [M.arg(xd)], s)
        g2.launch(s)
    s.synchronize()
    assert abs(g2.result()["reduced"] - K.sum_(xs)) <= 1e-12 * K.abs_sum(xs)
    # one-partition hysteresis: the whole while-loop runs on the device -> capturable
    gray = synth.np_u8_stream(8, 0, 77 * 130).reshape(77, 130)
    want_h, D = oracle_hyst(gray)
    c1 = ctx(1)
    dst = torch.empty((77, 130), dtype=torch.uint8, device=DEV)
    with torch.cuda.stream(s):
        g3 = M.mw_graph_capture(c1, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)], s)
        g3.launch(s)
    s.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want_h) and g3.result()["executions"] == D + 1
    # multi-partition per-pass protocol (HYST_FUSED = 0) needs the host for its
    # loop condition (the fused multi-partition loop is capturable: see
    # test_hysteresis_fused_partitions_graph_capture)
    M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_FUSED, 0)
    with pytest.raises(M.MwError) as e:
        with torch.cuda.stream(s):
            M.mw_graph_capture(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)], s)
    assert e.value.status == M.MW_E_UNSUPPORTED


# ----------------------------------------------------------------- degenerate inputs
def test_empty_inputs():
    c = ctx(3, [0.2, 0.3, 0.5])
    e = torch.empty((0, 16, 4), dtype=torch.uint8, device=DEV)
    run(c, trees.filter_pipeline(), [M.arg(e), M.arg(torch.empty_like(e))])
    v = torch.empty((0, 8, 8), dtype=torch.uint8, device=DEV)
    run(c, trees.segmentation(), [M.arg(v), M.arg(torch.empty_like(v))])
    x = torch.empty(0, dtype=torch.float32, device=DEV)
    run(c, trees.saxpy(), [M.arg(x), M.arg(torch.empty_like(x))])
    g = torch.empty((0, 33), dtype=torch.uint8, device=DEV)
    for cc in (c, ctx(1)):
        r = run(cc, trees.hysteresis(), [M.arg(g), M.arg(torch.empty_like(g))])
        assert r["executions"] == 1 and r["converged"]   # one execution that changes nothing
    p = torch.empty((0, 4), dtype=torch.float32, device=DEV)
    run(c, trees.nbody(2), [M.arg(p, M.MW_COPY), M.arg(torch.empty_like(p), M.MW_COPY)])


def test_single_pixel_and_single_row_images():
    for H, W in ((1, 1), (1, 4096), (4096, 1)):
        img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
        dst = torch.empty((H, W, 4), dtype=torch.uint8, device=DEV)
        run(ctx(2, [0.5, 0.5]), trees.filter_pipeline(), [M.arg(dev(img)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), oracle_filter(img))
        gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
        want, D = oracle_hyst(gray)
        for cc in (ctx(1), ctx(2, [0.5, 0.5])):
            out = torch.empty((H, W), dtype=torch.uint8, device=DEV)
            r = run(cc, trees.hysteresis(), [M.arg(dev(gray)), M.arg(out)])
            assert np.array_equal(out.cpu().numpy(), want) and r["executions"] == D + 1


# ----------------------------------------------------------------- tuning knobs
def test_tuning_knobs_bit_identical():
    """Every tuning value (the profile builder's search space) gives the same bytes."""
    c = ctx(1)
    img = synth.np_rgba(3, 0, 6 * 8192).reshape(6, 8192, 4)
    want = oracle_filter(img)
    src = dev(img)
    for tma in range(9):
        for unroll in (2, 4, 8):
            M.mw_ctx_set_tuning(c, M.MW_TUNE_RGBA_TMA, tma)
            M.mw_ctx_set_tuning(c, M.MW_TUNE_RGBA_UNROLL, unroll)
            dst = torch.empty_like(src)
            run(c, trees.filter_pipeline(), [M.arg(src), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), want), (tma, unroll)
            if tma:
                break
    gray = synth.np_u8_stream(8, 0, 300 * 257).reshape(300, 257)
    want_h, D = oracle_hyst(gray)
    for planes, T, R in ((0, 8, 40), (1, 4, 32), (1, 6, 32), (1, 8, 32), (1, 8, 40), (1, 12, 40),
                         (1, 6, 48), (1, 8, 48)):
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_PLANES, planes)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, 8)   # valid with every row count
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_ROWS, R)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, T)
        out = torch.empty((300, 257), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(out)])
        assert np.array_equal(out.cpu().numpy(), want_h) and r["executions"] == D + 1, (planes, T, R)
    pos, vel = synth.np_nbody(9, 0, 1024, 2.0 ** -10)
    outs = []
    for split in (0, 1):
        M.mw_ctx_set_tuning(c, M.MW_TUNE_NBODY_SPLIT, split)
        acc = torch.empty((1024, 4), dtype=torch.float32, device=DEV)
        run(c, M.mw_kernel_nbody_accel(1e-4), [M.arg(dev(pos), M.MW_COPY), M.arg(acc)])
        outs.append(acc.cpu().numpy())
    acc_o, cond = K.nbody_accel(pos, 1e-4)
    for o in outs:
        _nb_check(o[:, :3].astype(np.float64), acc_o, cond)
    with pytest.raises(M.MwError):
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_T, 5)


# ----------------------------------------------------------------- profile building (NEXT-2)
def test_autotune_filter_and_nbody(tmp_path):
    kb = M.mw_kb_open(str(tmp_path / "kb.txt"))
    c = ctx(1)
    img = synth.np_rgba(3, 0, 64 * 8192).reshape(64, 8192, 4)
    src, dst = dev(img), torch.empty((64, 8192, 4), dtype=torch.uint8, device=DEV)
    tree = trees.filter_pipeline()
    tune, ms = M.mw_autotune(c, tree, [M.arg(src), M.arg(dst)], reps=2, kb=kb)
    assert ms > 0 and [M.mw_ctx_get_tuning(c, k) for k in range(M.MW_TUNE_COUNT)] == tune
    assert np.array_equal(dst.cpu().numpy(), oracle_filter(img))
    assert M.mw_kb_lookup(kb, tree, [64, 8192, 4])[0] == M.MW_KB_EXACT
    # in-place state is restored after tuning
    pos, vel = synth.np_nbody(9, 0, 2048, 2.0 ** -11)
    p, v = dev(pos), dev(vel)
    M.mw_autotune(c, trees.nbody(1), [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)], reps=1, kb=kb)
    assert np.array_equal(p.cpu().numpy(), pos) and np.array_equal(v.cpu().numpy(), vel)
    assert M.mw_kb_count(kb) == 2
    kb.close()


def test_u8_tma_and_lsu_paths_identical():
    c = ctx(2, [0.4, 0.6])
    for shape in ((9, 64, 256), (3, 100, 100), (40, 1024, 16)):
        vol = synth.np_u8_stream(7, 0, int(np.prod(shape))).reshape(shape)
        want = K.segment(vol, 85, 170)
        for v in (0, 1):
            M.mw_ctx_set_tuning(c, M.MW_TUNE_U8_TMA, v)
            dst = torch.empty(shape, dtype=torch.uint8, device=DEV)
            run(c, trees.segmentation(), [M.arg(dev(vol)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), want), (shape, v)


# ----------------------------------------------------------------- C-ABI from C
def test_c_program_through_the_abi():
    """examples/filter_c.c drives the C-ABI with no Python; its output checksum
    must equal the oracle's for the same input."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "filter_c")
    H, W = 61, 96
    i = np.arange(H * W, dtype=np.int64)
    img = np.stack([(i * 7) % 256, (i * 13) % 256, (i * 29) % 256, np.full_like(i, 255)], -1)
    want = oracle_filter(img.astype(np.uint8).reshape(H, W, 4))
    fnv = 1469598103934665603
    for b in want.tobytes():
        fnv = ((fnv ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    for parts in (1, 3):
        out = subprocess.run([exe, str(H), str(W), str(parts)], capture_output=True, text=True, check=True)
        assert out.stdout.split()[1] == f"{fnv:016x}", out.stdout


def test_ctx_destroy_while_future_and_graph_alive():
    c = ctx()
    x = dev(synth.np_f32_um11(1, 0, 4096))
    y = dev(synth.np_f32_um11(2, 0, 4096))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = M.mw_graph_capture(c, trees.saxpy(1.0), [M.arg(x), M.arg(y)], s)
    f = M.mw_run(c, trees.mapreduce(False), [M.arg(x)])
    raw = c.ptr
    c.destroy()                      # deferred: the future and the graph still hold the ctx
    f.wait()
    assert abs(f.result()["reduced"] - K.sum_(x.cpu().numpy())) <= 1e-12 * 4096
    with torch.cuda.stream(s):
        g.launch(s)
    s.synchronize()
    st = M.lib().mw_run(raw, trees.saxpy(1.0).ptr, None, 0, None, None)
    assert st == M.MW_E_INVALID_SPEC or st == M.MW_E_STATE
    del f, g                         # last references: the teardown runs here
    torch.cuda.synchronize()


# ----------------------------------------------------------------- FFT (NEXT-3)
from oracle import fft as FF  # noqa: E402

SEED_FFT = 11


def _fft_tree(log2n, dirs):
    leaves = [M.mw_kernel_fft(log2n, d == "I") for d in dirs]
    return leaves[0] if len(leaves) == 1 else M.mw_pipeline(leaves)


def _fft_in(B, N, start=0):
    return synth.np_f32_um11(SEED_FFT, start, 2 * B * N).reshape(B, N, 2)


def _fft_check(got, x, dirs):
    N = x.shape[1]
    want = FF.fft_chain(FF.as_complex(x), dirs)
    err = FF.rel_l2(FF.as_complex(got), want)
    assert np.all(np.isfinite(err)) and err.max() <= FF.tolerance(N, len(dirs)), (dirs, err.max())
    return err.max()


@pytest.mark.parametrize("log2n", [13, 14, 15, 16])
@pytest.mark.parametrize("dirs", ["F", "I", "FI", "IF", "FF", "FIIF"])
def test_fft_chain_parity(log2n, dirs):
    N = 1 << log2n
    B = 3
    x = _fft_in(B, N, 77)
    src = dev(x)
    dst = torch.empty_like(src)
    run(ctx(), _fft_tree(log2n, dirs), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy(), x, dirs)
    assert torch.equal(src, dev(x))   # input untouched


@pytest.mark.parametrize("four", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("dirs", ["FI", "FIFI", "IFI"])
def test_fft_fused_pair_paths(four, dirs):
    """The fused pipeline(fft, ifft) at 2^16 on every implementation — the
    16 x 4096 four-step path as one persistent dataflow launch
    (MW_TUNE_FFT_4STEP = 1, default) and as three launches (4), the 256 x 256
    one as three launches (3) and as a dataflow launch (2), and
    one thread-block cluster per transform (0) — within the bound of the
    oracle, also inside longer chains and after an inverse leaf."""
    N, B = 1 << 16, 5
    x = _fft_in(B, N, 123)
    src = dev(x)
    dst = torch.empty_like(src)
    c = ctx()
    M.mw_ctx_set_tuning(c, M.MW_TUNE_FFT_4STEP, four)
    run(c, _fft_tree(16, dirs), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy(), x, dirs)
    assert torch.equal(src, dev(x))


@pytest.mark.parametrize("launches,flow", [(3, 2), (4, 1)])
@pytest.mark.parametrize("B", [1, 2, 17, 40, 300])
def test_fft_4step_dataflow_bitwise(B, launches, flow):
    """The dataflow launches (MW_TUNE_FFT_4STEP = 2 for 256 x 256, 1 for
    16 x 4096: work items claimed from an atomic ticket, passes of a
    transform ordered by readiness counters) run the same arithmetic per
    element as the three launches of the same decomposition (3, 4):
    bit-identical outputs for batches shorter and longer than the pipelining
    lag (64), within the oracle's bound, and on a repeated run of the same
    ctx (the counters are re-zeroed per launch)."""
    N = 1 << 16
    x = _fft_in(B, N, 900 + B)
    src = dev(x)
    ref = torch.empty_like(src)
    c1 = ctx()
    M.mw_ctx_set_tuning(c1, M.MW_TUNE_FFT_4STEP, launches)
    run(c1, trees.fft_pipeline(16), [M.arg(src), M.arg(ref)])
    c2 = ctx()
    M.mw_ctx_set_tuning(c2, M.MW_TUNE_FFT_4STEP, flow)
    for _ in range(2):
        dst = torch.full_like(src, float("nan"))
        run(c2, trees.fft_pipeline(16), [M.arg(src), M.arg(dst)])
        assert torch.equal(dst, ref)
    if B <= 40:
        _fft_check(dst.cpu().numpy(), x, "FI")
    assert torch.equal(src, dev(x))   # input untouched


def test_fft_pipeline_partitions_bitwise_and_batch():
    """The benchmark tree over a batch split into partitions (whole FFTs per
    partition, zero shares, ragged splits): every FFT is computed the same way
    wherever it lands, so the output is bit-identical across distributions."""
    log2n, B = 16, 37
    N = 1 << log2n
    x = _fft_in(B, N)
    src = dev(x)
    ref = torch.empty_like(src)
    run(ctx(), trees.fft_pipeline(log2n), [M.arg(src), M.arg(ref)])
    _fft_check(ref.cpu().numpy(), x, "FI")
    rng = np.random.default_rng(5)
    for k, d in [(3, x_) for x_ in dists(3, rng, 2) + [[0.0, 1.0, 0.0]]] + [(5, [0.1, 0.2, 0.0, 0.3, 0.4])]:
        dst = torch.empty_like(src)
        run(ctx(k, d), trees.fft_pipeline(log2n), [M.arg(src), M.arg(dst)])
        assert torch.equal(dst, ref), d


def test_fft_closed_forms_on_device():
    """Delta and single-tone inputs (closed forms, no oracle library): the
    forward transform of a delta at n0 is the twiddle row exp(-2 pi i n0 k/N)."""
    N = 1 << 16
    x = np.zeros((2, N, 2), np.float32)
    x[0, 5, 0] = 1.0
    x[1, 0, 0] = 1.0   # delta at 0 -> all ones
    src = dev(x)
    dst = torch.empty_like(src)
    run(ctx(), M.mw_kernel_fft(16, False), [M.arg(src), M.arg(dst)])
    g = dst.cpu().numpy().astype(np.float64)
    k = np.arange(N)
    want = np.exp(-2j * np.pi * ((5 * k) % N) / N)
    assert np.max(np.abs(g[0, :, 0] + 1j * g[0, :, 1] - want)) < 4e-6
    assert np.array_equal(g[1], np.stack([np.ones(N), np.zeros(N)], -1))


def test_fft_edge_cases():
    c = ctx(2)
    e = torch.empty((0, 1 << 13, 2), dtype=torch.float32, device=DEV)
    run(c, trees.fft_pipeline(13), [M.arg(e), M.arg(torch.empty_like(e))])   # empty batch
    x = _fft_in(1, 1 << 13)
    src = dev(x)
    dst = torch.empty_like(src)
    run(c, trees.fft_pipeline(13), [M.arg(src), M.arg(dst)])   # one FFT, two partitions
    _fft_check(dst.cpu().numpy(), x, "FI")
    # loop_for(fft, 0) is the identity; loop_for(pipeline(fft, ifft), 3) fuses to 3 launches
    run(c, M.mw_loop_for(M.mw_kernel_fft(13, False), 0), [M.arg(src), M.arg(dst)])
    assert torch.equal(dst, src)
    run(c, M.mw_loop_for(trees.fft_pipeline(13), 3), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy(), x, "FIFIFI")
    with pytest.raises(M.MwError):   # leaf size != row length
        run(c, trees.fft_pipeline(14), [M.arg(src), M.arg(dst)])


@pytest.mark.parametrize("four", [1, 2, 3, 4])
def test_fft_2p16_edge_cases(four):
    """The four-step forms at 2^16: an empty batch, one FFT on three
    partitions (two of them empty), loop_for(pipeline(fft, ifft), 3) (three
    fused pairs, each a dataflow launch or three launches in place on the
    output)."""
    c = ctx(3, [0.0, 1.0, 0.0])
    M.mw_ctx_set_tuning(c, M.MW_TUNE_FFT_4STEP, four)
    e = torch.empty((0, 1 << 16, 2), dtype=torch.float32, device=DEV)
    run(c, trees.fft_pipeline(16), [M.arg(e), M.arg(torch.empty_like(e))])
    x = _fft_in(1, 1 << 16, 21)
    src = dev(x)
    dst = torch.empty_like(src)
    run(c, trees.fft_pipeline(16), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy(), x, "FI")
    run(c, M.mw_loop_for(trees.fft_pipeline(16), 3), [M.arg(src), M.arg(dst)])
    _fft_check(dst.cpu().numpy(), x, "FIFIFI")


@pytest.mark.parametrize("B", [40, 300])
def test_fft_host_staged_and_graph(B):
    """Host-staged runs (chunks of the batch) and a captured graph (replayed
    twice: the dataflow launch's readiness counters are re-zeroed by the
    captured memset) equal the device run."""
    log2n = 16
    x = _fft_in(B, 1 << log2n, 3)
    src = dev(x)
    ref = torch.empty_like(src)
    c = ctx()
    run(c, trees.fft_pipeline(log2n), [M.arg(src), M.arg(ref)])
    hin = torch.from_numpy(x).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    run(c, trees.fft_pipeline(log2n), [M.arg(hin), M.arg(hout)])
    assert torch.equal(hout, ref.cpu())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = torch.empty_like(src)
        g = M.mw_graph_capture(c, trees.fft_pipeline(log2n), [M.arg(src), M.arg(out)], s)
        for _ in range(2):
            out.fill_(float("nan"))
            g.launch(s)
            s.synchronize()
            assert torch.equal(out, ref)


# ----------------------------------------------------------------- NEXT-4 variants
def _merge_ref(op, parts):
    acc = parts[0]
    for r in parts[1:]:
        acc = (acc - r if op == M.MW_MERGE_SUB else acc * r if op == M.MW_MERGE_MUL
               else acc / r if op == M.MW_MERGE_DIV else op(acc, r))
    return acc


@pytest.mark.parametrize("dot", [False, True])
def test_mapreduce_merge_functions(dot):
    """P:705-707 merging functions (R26): per-partition partials merged in
    partition order; each compared with the oracle's partition-aware
    evaluation within a first-order propagated fp64 bound."""
    n = 7 * (1 << 16) + 311
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    xd, yd = dev(x), dev(y)
    args = [M.arg(xd), M.arg(yd)] if dot else [M.arg(xd)]
    stage = M.mw_kernel_map_product() if dot else M.mw_kernel_map_identity()
    ostage = sct.Leaf("map_product" if dot else "map_identity")
    user = lambda a, r: 0.5 * a + r   # noqa: E731  (order-sensitive)
    for d in ([0.5, 0.25, 0.25], [0.2, 0.0, 0.8], [1.0, 0.0, 0.0]):
        c = ctx(3, d)
        off, lens = M.mw_partition(c, stage, n)
        for op in (M.MW_MERGE_SUB, M.MW_MERGE_MUL, M.MW_MERGE_DIV, user):
            node = M.mw_map_reduce_user(stage, op) if callable(op) else M.mw_map_reduce(stage, op)
            got = run(c, node, args)["reduced"]
            oop = op if callable(op) else {M.MW_MERGE_SUB: "-", M.MW_MERGE_MUL: "*", M.MW_MERGE_DIV: "/"}[op]
            want = sct.evaluate(sct.MapReduce(ostage, oop), (x, y) if dot else (x,), lengths=lens).reduced
            # first-order bound: partial p is within 1e-13 * sum|terms_p| of exact
            parts, tol, o = [], [], 0
            for ln in lens:
                if ln:
                    sl = slice(o, o + ln)
                    terms = x[sl].astype(np.float64) * (y[sl].astype(np.float64) if dot else 1.0)
                    parts.append(float(np.sum(terms)))
                    tol.append(1e-13 * float(np.sum(np.abs(terms))))
                o += ln
            bound = 0.0
            for p in range(len(parts)):
                h = tol[p]
                q = list(parts)
                q[p] += h
                bound += abs(_merge_ref(op, q) - _merge_ref(op, parts)) if h else 0.0
            assert abs(got - want) <= 2 * bound + 1e-300, (d, op, got, want, bound)
        c.destroy()
    # ADD keeps the canonical, distribution-independent sum
    r1 = run(ctx(3, [0.2, 0.0, 0.8]), M.mw_map_reduce(stage, M.MW_MERGE_ADD), args)["reduced"]
    r2 = run(ctx(1), M.mw_map_reduce(stage, M.MW_MERGE_ADD), args)["reduced"]
    assert r1 == r2


def test_loop_host_condition():
    """condition (stage 1) and state update (stage 3) on the host;
    a loop stopped at k by its host condition equals loop_for(body, k)."""
    img = synth.np_rgba(3, 0, 40 * 256).reshape(40, 256, 4)
    src = dev(img)
    for k, dist in ((0, [1.0]), (1, [0.5, 0.5]), (3, [0.3, 0.7])):
        c = ctx(len(dist), dist)
        calls = []
        dst = torch.empty_like(src)
        r = run(c, M.mw_loop_host(trees.filter_pipeline(), 50, lambda i: (calls.append(i), i < k)[1]),
                [M.arg(src), M.arg(dst)])
        ref = torch.empty_like(src)
        run(c, M.mw_loop_for(trees.filter_pipeline(), k), [M.arg(src), M.arg(ref)])
        assert torch.equal(dst, ref) and r["executions"] == k and r["converged"], k
        assert calls == list(range(k + 1))
        want = sct.evaluate(sct.LoopFor(sct.Pipeline([sct.Leaf("gauss_noise", {"seed": 4, "scale": 8}),
                                                       sct.Leaf("solarize", {"threshold": 128}),
                                                       sct.Leaf("mirror")]), k), img).value
        assert np.array_equal(dst.cpu().numpy(), want)
    # in-place state (saxpy): the host update reads the device state each iteration
    c = ctx(2)
    x = dev(synth.np_f32_um11(1, 0, 4099))
    y0 = synth.np_f32_um11(2, 0, 4099)
    y = dev(y0)
    seen = []

    def cond(i):
        seen.append(float(y[7]))   # stage 3: state read on the host between iterations
        return i < 4
    r = run(c, M.mw_loop_host(trees.saxpy(0.5), 100, cond), [M.arg(x), M.arg(y)])
    want = y0
    for _ in range(4):
        want = K.saxpy(0.5, synth.np_f32_um11(1, 0, 4099), want)
    assert np.array_equal(y.cpu().numpy(), want) and r["executions"] == 4 and len(seen) == 5
    # max_iters reached -> not converged; a hysteresis step body (stencil, ping-pong)
    gray = synth.np_u8_stream(8, 0, 60 * 90).reshape(60, 90)
    L = K.segment(gray, 173, 250)
    dst = torch.empty((60, 90), dtype=torch.uint8, device=DEV)
    r = run(ctx(3), M.mw_loop_host(M.mw_kernel_hysteresis_step(), 4, lambda i: True), [M.arg(dev(L)), M.arg(dst)])
    assert np.array_equal(dst.cpu().numpy(), K.hyst_bfs(L, 4)[0]) and r["executions"] == 4 and not r["converged"]
    # not capturable; not nestable
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with pytest.raises(M.MwError):
            M.mw_graph_capture(ctx(1), M.mw_loop_host(trees.saxpy(0.5), 3, lambda i: True), [M.arg(x), M.arg(y)], s)
    # a host loop as a pipeline stage runs (test_host_condition_loop_inside_a_pipeline):
    # mirror twice in the loop, once after it = one mirror
    out = torch.empty_like(src)
    r = run(ctx(1), M.mw_pipeline([M.mw_loop_host(M.mw_kernel_mirror(), 2, lambda i: True), M.mw_kernel_mirror()]),
            [M.arg(src), M.arg(out)])
    assert np.array_equal(out.cpu().numpy(), K.mirror(src.cpu().numpy())) and r["executions"] == 2


def test_released_futures_and_arglist():
    """Futures dropped without waiting are reclaimed by later runs (release
    never blocks); a prebuilt ArgList gives the same bytes as a list; a ctx
    destroyed with runs in flight drains them first."""
    H, W = 256, 512
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = oracle_filter(img)
    c = ctx(2, [0.5, 0.5])
    src = dev(img)
    outs = [torch.empty((H, W, 4), dtype=torch.uint8, device=DEV) for _ in range(4)]
    lists = [M.ArgList([M.arg(src), M.arg(o)]) for o in outs]
    for i in range(300):
        M.mw_run(c, trees.filter_pipeline(), lists[i % 4] if i % 2 else [M.arg(src), M.arg(outs[i % 4])])
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), want)
    tail = M.mw_run(c, trees.filter_pipeline(), lists[0])
    M.mw_ctx_destroy(c)
    tail.wait()
    assert np.array_equal(outs[0].cpu().numpy(), want)


def test_plan_cache_errors_not_cached():
    """The per-node plan cache publishes only successful plans: a tree that
    cannot run reports its error on every run, and a shared subtree planned
    inside several roots gives the same bytes each time."""
    c = ctx()
    bad = M.mw_kernel_reduce(M.MW_REDUCE_MAX)   # a reduction stage runs only inside map_reduce_sct
    x = torch.ones(100, device=DEV)
    for _ in range(2):
        with pytest.raises(M.MwError) as e:
            run(c, bad, [M.arg(x)])
        assert e.value.status == M.MW_E_INVALID_SPEC
    m = M.mw_kernel_map_identity()
    t1 = M.mw_map_reduce_sct(m, M.mw_kernel_reduce(M.MW_REDUCE_MAX))
    t2 = M.mw_map_reduce(m, M.MW_MERGE_ADD)
    xs = dev(synth.np_f32_um11(5, 0, 5000))
    for _ in range(3):
        assert run(c, t1, [M.arg(xs)])["reduced"] == K.fold_extreme(xs.cpu().numpy())
        assert run(c, t2, [M.arg(xs)])["reduced"] == K.sum_(xs.cpu().numpy())


def test_dropped_future_keeps_temporaries_alive():
    """A future dropped while its run is in flight, together with the only
    reference to a temporary input, on a side stream: the caching allocator
    must not hand the input's memory to a new tensor before the run read it."""
    H, W = 2048, 2048
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = oracle_filter(img)
    c = ctx()
    side = torch.cuda.Stream()
    dst = torch.empty((H, W, 4), dtype=torch.uint8, device=DEV)
    for _ in range(5):
        tmp = dev(img)                     # allocated on the default stream
        side.wait_stream(torch.cuda.current_stream())
        M.mw_run(c, trees.filter_pipeline(), [M.arg(tmp), M.arg(dst)], stream=side)
        del tmp                            # future and input dropped at once
        junk = torch.full((H, W, 4), 7, dtype=torch.uint8, device=DEV)   # may reuse the block
        del junk
    torch.cuda.synchronize()
    assert np.array_equal(dst.cpu().numpy(), want)


@pytest.mark.parametrize("lohi", [(0, 0), (0, 256), (256, 256), (100, 100), (3, 129), (130, 200),
                                  (0, 90), (200, 256), (127, 128)])
def test_hysteresis_threshold_modes(lohi):
    """Every compile-time compare-mode pair of the plane pack (lo / hi below
    128, at or above 128, <= 0, >= 256), one and three partitions."""
    H, W = 130, 300
    gray = synth.np_u8_stream(8, 11, H * W).reshape(H, W)
    want, D = oracle_hyst(gray, *lohi)
    for k, d in ((1, None), (3, [0.3, 0.3, 0.4])):
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(pctx(k, d, 1), trees.hysteresis(*lohi), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want), (lohi, k)
        assert r["executions"] == D + 1, (lohi, k)


# ----------------------------------------------------------------- hysteresis: fused multi-partition loop
@pytest.mark.parametrize("fused", [1, 0])
def test_hysteresis_partitions_fused_and_per_pass(fused):
    """Several partitions of one rank: the whole loop in one cooperative kernel
    (in-kernel halo stores into the neighbours' halo rows, device loop
    condition) or one launch per partition and pass — identical output, E."""
    rng = np.random.default_rng(11)
    H, W = 777, 1300
    gray = synth.np_u8_stream(8, 9, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)
    L = K.segment(gray, 173, 250)
    for k, d in [(8, None), (8, [0.3, 0.01, 0.0, 0.2, 0.09, 0.2, 0.0, 0.2]), (2, [0.999, 0.001])] + \
            [(5, x) for x in dists(5, rng, 2)]:
        c = pctx(k, d, 1)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_FUSED, fused)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want), d
        assert r["executions"] == D + 1 and r["converged"]
        for n in (D - 2, 3):
            dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
            r = run(c, trees.hysteresis(max_iters=n), [M.arg(dev(gray)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(K.hyst_bfs(L, n)[0]))
            assert r["executions"] == n and not r["converged"]
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        run(c, M.mw_loop_for(M.mw_kernel_hysteresis_step(), 13), [M.arg(dev(L)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), K.hyst_bfs(L, 13)[0])


def _path_image(H, W, pts):
    """Gray image: 0 everywhere (below lo), weak (200) on the path, strong
    (255) at its first point: the fronts run along the path one pixel per
    execution, so the last change lands at a chosen execution."""
    g = np.zeros((H, W), dtype=np.uint8)
    for (y, x) in pts:
        g[y, x] = 200
    g[pts[0]] = 255
    return g


def _serpentine(H, W, legs, run, drop):
    """Right `run` px, down `drop` rows, left `run` px, ... `legs` legs, then
    the total length is known exactly (8-connected, no shortcuts: legs are
    `drop` >= 2 rows apart)."""
    pts, y, x, d = [], 1, 1, 1
    for leg in range(legs):
        for _ in range(run):
            pts.append((y, x))
            x += d
        for _ in range(drop):
            pts.append((y, x))
            y += 1
        d = -d
    return pts


@pytest.mark.parametrize("ppr", [1, 3])
def test_hysteresis_fronts_across_tiles_and_passes(ppr):
    """Fronts crossing warp-tile boundaries (32-row strips, 960-pixel column
    blocks) and ending at every position of a pass (the first, a middle and
    the last of the T = 8 executions): exercises the per-tile early stop,
    the push-model activity stamps (self and 3x3, across partitions at ppr = 3)
    and the exact E at pass boundaries."""
    H, W = 300, 2100
    cases = []
    for L in (7, 8, 9, 15, 16, 17, 40):   # horizontal across the 960-px block edge
        cases.append([(150, 955 - L // 2 + i) for i in range(L + 1)])
    for L in (8, 9, 31, 33):               # vertical across strip edges
        cases.append([(20 + i, 500) for i in range(L + 1)])
    cases.append([(5 + i, 940 + i) for i in range(70)])   # diagonal through a tile corner
    cases.append(_serpentine(H, W, 5, 1500, 3))           # long snake, E in the thousands
    c = pctx(ppr, None, 1)
    for k, pts in enumerate(cases):
        gray = _path_image(H, W, pts)
        want, D = oracle_hyst(gray)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want), k
        assert r["executions"] == D + 1 and r["converged"], (k, r, D)
        L = K.segment(gray, 173, 250)
        for n in (D - 1, D, 8 * (D // 8)):
            if n < 1:
                continue
            dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
            r = run(c, trees.hysteresis(max_iters=n), [M.arg(dev(gray)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), K.hyst_finalize(K.hyst_bfs(L, n)[0])), (k, n)


@pytest.mark.parametrize("ppr", [1, 4])
def test_hysteresis_repeated_runs_one_ctx(ppr):
    """Runs of one ctx reuse the plane buffers: the image-edge halo rows and
    the loop flags are set up once per buffer set (the loop kernels leave their
    flags ready) and the per-tile activity stamps are never cleared.  A
    sequence of different inputs, trees (while / max_iters / loop_for) and
    paths (fused, per-pass, slowed partition) on the same buffers must match
    the oracle at every run."""
    H, W = 391, 700
    c = pctx(ppr, None, 1)
    L0 = None
    seq = [(1, 0, None), (1, 0, 5), (0, 0, None), (1, 0, None), (1, 2.0, None), (1, 0, 7), (1, 0, None)]
    for i, (fused, slow, n) in enumerate(seq):
        gray = synth.np_u8_stream(8, 100 + i, H * W).reshape(H, W)
        L = K.segment(gray, 173, 250)
        M.mw_ctx_set_tuning(c, M.MW_TUNE_HYST_FUSED, fused)
        if ppr > 1:
            M.mw_ctx_set_slowdown(c, 1, slow if slow else 1.0)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        if n is None:
            want, D = oracle_hyst(gray)
            r = run(c, trees.hysteresis(), [M.arg(dev(gray)), M.arg(dst)])
            assert r["executions"] == D + 1 and r["converged"], (i, r, D)
        else:
            want = K.hyst_finalize(K.hyst_bfs(L, n)[0])
            r = run(c, trees.hysteresis(max_iters=n), [M.arg(dev(gray)), M.arg(dst)])
            assert r["executions"] == n, (i, r)
        assert np.array_equal(dst.cpu().numpy(), want), i
        # a loop_for over the labels on the same buffers in between
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        run(c, M.mw_loop_for(M.mw_kernel_hysteresis_step(), 9), [M.arg(dev(L)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), K.hyst_bfs(L, 9)[0]), i


def test_hysteresis_fused_partitions_graph_capture():
    """The fused multi-partition loop decides its condition on the device, so
    the while-loop tree can be captured and replayed."""
    H, W = 500, 640
    gray = synth.np_u8_stream(8, 4, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)
    c = pctx(4, [0.1, 0.4, 0.2, 0.3], 1)
    s = torch.cuda.Stream()
    src = dev(gray)
    dst = torch.zeros_like(src)
    torch.cuda.synchronize()
    g = M.mw_graph_capture(c, trees.hysteresis(), [M.arg(src), M.arg(dst)], stream=s)
    for _ in range(2):
        dst.zero_()
        torch.cuda.synchronize()
        g.launch(s)
        s.synchronize()
        assert np.array_equal(dst.cpu().numpy(), want)
        r = g.result()
        assert r["executions"] == D + 1 and r["converged"]


# ----------------------------------------------------------------- general SCT composition
@pytest.mark.parametrize("m", [2, 3])
def test_while_loop_with_multi_step_body(m):
    """loop_while_changed(pipeline(step x m)): E counts BODY executions (a body
    changed iff one of its steps did), as the oracle's LoopWhileChanged."""
    H, W = 257, 300
    gray = synth.np_u8_stream(8, 2, H * W).reshape(H, W)
    body = sct.Pipeline([sct.Leaf("hysteresis_step")] * m)
    otree = sct.Pipeline([sct.Leaf("segment", {"lo": 173, "hi": 250}),
                          sct.LoopWhileChanged(body, 1000), sct.Leaf("hysteresis_finalize")])
    want = sct.evaluate(otree, gray)
    mb = M.mw_pipeline([M.mw_kernel_hysteresis_step() for _ in range(m)])
    tree = M.mw_pipeline([M.mw_kernel_segment(173, 250), M.mw_loop_while_changed(mb, 1000, 1),
                          M.mw_kernel_hysteresis_finalize()])
    for k, d, planes in [(1, None, 1), (3, [0.3, 0.3, 0.4], 1), (3, [0.5, 0.0, 0.5], 0), (2, None, 0)]:
        c = pctx(k, d, planes)
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(c, tree, [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want.value), (k, planes)
        assert r["executions"] == want.executions and r["converged"], (r, want.executions)
    # max body executions below the fixed point
    n = max(1, want.executions - 3)
    otree2 = sct.Pipeline([sct.Leaf("segment", {"lo": 173, "hi": 250}), sct.LoopWhileChanged(body, n)])
    w2 = sct.evaluate(otree2, gray)
    tree2 = M.mw_pipeline([M.mw_kernel_segment(173, 250), M.mw_loop_while_changed(mb, n, 1)])
    for k, planes in ((1, 1), (3, 1), (2, 0)):
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(pctx(k, None, planes), tree2, [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), w2.value) and r["executions"] == n and not r["converged"]


def test_loop_for_mixed_bodies():
    """loop_for over bodies mixing kinds: the loop is its body unrolled (state
    carried between executions), against the oracle's depth-first evaluation."""
    H, W = 130, 170
    gray = synth.np_u8_stream(8, 6, H * W).reshape(H, W)
    lab = K.segment(gray, 173, 250)
    cases = [
        (sct.LoopFor(sct.Pipeline([sct.Leaf("segment", {"lo": 100, "hi": 200}),
                                   sct.Leaf("hysteresis_step")]), 3),
         M.mw_loop_for(M.mw_pipeline([M.mw_kernel_segment(100, 200), M.mw_kernel_hysteresis_step()]), 3),
         gray),
        (sct.LoopFor(sct.LoopWhileChanged(sct.Leaf("hysteresis_step"), 500), 2),
         M.mw_loop_for(M.mw_loop_while_changed(M.mw_kernel_hysteresis_step(), 500), 2), lab),
        (sct.LoopFor(sct.LoopFor(sct.Leaf("hysteresis_step"), 3), 4),
         M.mw_loop_for(M.mw_loop_for(M.mw_kernel_hysteresis_step(), 3), 4), lab),
    ]
    for otree, tree, inp in cases:
        want = sct.evaluate(otree, inp)
        for k, d in ((1, None), (3, [0.2, 0.5, 0.3])):
            dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
            r = run(ctx(k, d), tree, [M.arg(dev(inp)), M.arg(dst)])
            assert np.array_equal(dst.cpu().numpy(), want.value)
            assert r["executions"] == want.executions
    # N-body loop over two steps of different dt (not merged: unrolled)
    N = 700
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -9)
    tree = M.mw_loop_for(M.mw_pipeline([M.mw_kernel_nbody_step(1e-3, 1e-4), M.mw_kernel_nbody_step(5e-4, 1e-4)]), 2)
    p1, v1 = dev(pos), dev(vel)
    run(ctx(2), tree, [M.arg(p1, M.MW_COPY), M.arg(v1, M.MW_COPY)])
    p2, v2 = dev(pos), dev(vel)
    c1 = ctx(1)
    for _ in range(2):
        run(c1, trees.nbody(1, dt=1e-3), [M.arg(p2, M.MW_COPY), M.arg(v2, M.MW_COPY)])
        run(c1, trees.nbody(1, dt=5e-4), [M.arg(p2, M.MW_COPY), M.arg(v2, M.MW_COPY)])
    assert torch.equal(p1, p2) and torch.equal(v1, v2)


def test_mapreduce_fused_saxpy_map_stage():
    """map_reduce(pipeline(saxpy chain, map_product)): the chain is fused into
    the reduction kernel (y' never stored), against the oracle; the canonical
    sum is bit-identical for every distribution and y is left untouched."""
    n = 6 * (1 << 16) + 999
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    for chain in ([0.75], [2.5, -1.25, 0.5]):
        otree = sct.MapReduce(sct.Pipeline([sct.Leaf("saxpy", {"a": a}) for a in chain] +
                                           [sct.Leaf("map_product")]), "+")
        want = sct.evaluate(otree, (x, y)).reduced
        tree = M.mw_map_reduce(M.mw_pipeline([M.mw_kernel_saxpy(a) for a in chain] +
                                             [M.mw_kernel_map_product()]))
        got = []
        for k, d in ((1, None), (3, [0.5, 0.1, 0.4]), (4, [0.0, 0.5, 0.25, 0.25])):
            yd = dev(y)
            got.append(run(ctx(k, d), tree, [M.arg(dev(x)), M.arg(yd)])["reduced"])
            assert np.array_equal(yd.cpu().numpy(), y)
        assert all(g == got[0] for g in got)
        yp = y
        for a in chain:
            yp = K.saxpy(a, x, yp)
        assert abs(got[0] - want) <= 1e-12 * K.abs_sum(x, yp)
    # with the device reduction stage (max of the terms): bit-exact
    tree = M.mw_map_reduce_sct(M.mw_pipeline([M.mw_kernel_saxpy(0.75), M.mw_kernel_map_product()]),
                               M.mw_kernel_reduce(M.MW_REDUCE_MAX))
    r = run(ctx(3, [0.3, 0.3, 0.4]), tree, [M.arg(dev(x)), M.arg(dev(y))])["reduced"]
    assert r == (x.astype(np.float64) * K.saxpy(0.75, x, y).astype(np.float64)).max()


def test_host_condition_loop_inside_a_pipeline():
    """pipeline(..., loop_host(body, cond), ...): the Fig. 1 shape with the
    paper's host-side loop condition as a stage, not the root."""
    H, W = 140, 190
    gray = synth.np_u8_stream(8, 11, H * W).reshape(H, W)
    calls = []

    def cond(i):
        calls.append(i)
        return i < 6

    otree = sct.Pipeline([sct.Leaf("segment", {"lo": 173, "hi": 250}),
                          sct.LoopHost(sct.Leaf("hysteresis_step"), 100, cond=lambda i: i < 6),
                          sct.Leaf("hysteresis_finalize")])
    want = sct.evaluate(otree, gray)
    tree = M.mw_pipeline([M.mw_kernel_segment(173, 250),
                          M.mw_loop_host(M.mw_kernel_hysteresis_step(), 100, cond),
                          M.mw_kernel_hysteresis_finalize()])
    for k, d in ((1, None), (3, [0.3, 0.0, 0.7])):
        calls.clear()
        dst = torch.empty((H, W), dtype=torch.uint8, device=DEV)
        r = run(ctx(k, d), tree, [M.arg(dev(gray)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), want.value)
        assert r["executions"] == want.executions == 6 and r["converged"] and calls == list(range(7))
    # RGBA: the loop between two fused chains; loop first / last
    img = synth.np_rgba(3, 0, 33 * 64).reshape(33, 64, 4)
    for pre, post in (([M.mw_kernel_gauss_noise(4, 8)], [M.mw_kernel_mirror()]), ([], [M.mw_kernel_mirror()]),
                      ([M.mw_kernel_gauss_noise(4, 8), M.mw_kernel_mirror()], [])):
        tree = M.mw_pipeline(pre + [M.mw_loop_host(M.mw_kernel_solarize(100), 10, lambda i: i < 3)] + post)
        v = img
        if pre:
            v = K.gauss_noise(v, 4, 8)
            if len(pre) == 2:
                v = K.mirror(v)
        for _ in range(3):
            v = K.solarize(v, 100)
        if post:
            v = K.mirror(v)
        dst = torch.empty_like(dev(img))
        r = run(ctx(2, [0.6, 0.4]), tree, [M.arg(dev(img)), M.arg(dst)])
        assert np.array_equal(dst.cpu().numpy(), v) and r["executions"] == 3
    # in place (saxpy): every part on the same arguments
    n = 4099
    x = synth.np_f32_um11(1, 0, n)
    y0 = synth.np_f32_um11(2, 0, n)
    yd = dev(y0)
    tree = M.mw_pipeline([M.mw_kernel_saxpy(0.5), M.mw_loop_host(M.mw_kernel_saxpy(0.25), 10, lambda i: i < 4),
                          M.mw_kernel_saxpy(2.0)])
    run(ctx(2), tree, [M.arg(dev(x)), M.arg(yd)])
    want = K.saxpy(0.5, x, y0)
    for _ in range(4):
        want = K.saxpy(0.25, x, want)
    assert np.array_equal(yd.cpu().numpy(), K.saxpy(2.0, x, want))


def test_reduction_stage_sct():
    """map_reduce_sct(map stage, pipeline(term maps, reduce(op), scalar maps)):
    the L1 / L2 / L-inf norms, a mean and a sum of squared products, on the
    device, against the oracle; every distribution gives the same bits."""
    n = 5 * (1 << 16) + 4321
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)

    def both(tmaps, op, smaps, dot=False):
        ot = [sct.Leaf("term_map", {"map": t}) for t in tmaps] + [sct.Leaf("reduce", {"op": op})] + \
             [sct.Leaf("scalar_map", {"map": k, "c": c}) for k, c in smaps]
        otree = sct.MapReduce(sct.Leaf("map_product" if dot else "map_identity"),
                              ot[0] if len(ot) == 1 else sct.Pipeline(ot))
        codes = {"abs": M.MW_TERM_ABS, "square": M.MW_TERM_SQUARE}
        ops = {"sum": M.MW_REDUCE_SUM, "max": M.MW_REDUCE_MAX, "min": M.MW_REDUCE_MIN}
        sk = {"sqrt": M.MW_SCALAR_SQRT, "scale": M.MW_SCALAR_SCALE}
        st = [M.mw_kernel_term_map(codes[t]) for t in tmaps] + [M.mw_kernel_reduce(ops[op])] + \
             [M.mw_kernel_scalar_map(sk[k], c) for k, c in smaps]
        tree = M.mw_map_reduce_sct(M.mw_kernel_map_product() if dot else M.mw_kernel_map_identity(),
                                   st[0] if len(st) == 1 else M.mw_pipeline(st))
        return otree, tree

    cases = [(["abs"], "sum", []), (["square"], "sum", [("sqrt", 0.0)]), (["abs"], "max", []),
             ([], "sum", [("scale", 1.0 / n)]), (["square"], "sum", [], True), (["abs"], "min", [], True),
             (["abs", "square"], "sum", [("sqrt", 0.0), ("scale", 0.5)])]
    for case in cases:
        tm, op, sm = case[:3]
        dot = len(case) > 3
        otree, tree = both(tm, op, sm, dot)
        want = sct.evaluate(otree, (x, y) if dot else x).reduced
        args = [M.arg(dev(x))] + ([M.arg(dev(y))] if dot else [])
        got = [run(ctx(k, d), tree, args)["reduced"]
               for k, d in ((1, None), (3, [0.2, 0.5, 0.3]), (4, [0.0, 0.25, 0.5, 0.25]))]
        assert all(g == got[0] for g in got), case
        if op == "sum":
            assert abs(got[0] - want) <= 1e-12 * abs(want), (case, got[0], want)
        else:
            assert got[0] == want, case
    # the map/reduce structure is validated
    with pytest.raises(M.MwError):
        M.mw_map_reduce_sct(M.mw_kernel_map_identity(),
                            M.mw_pipeline([M.mw_kernel_term_map(0), M.mw_kernel_term_map(1)]))
    with pytest.raises(M.MwError):
        run(ctx(), M.mw_kernel_term_map(0), [M.arg(dev(x))])
