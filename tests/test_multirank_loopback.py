"""Cross-rank code paths of libmarrow, executed on ONE GPU.

Each rank is a host thread with its own ctx, stream and buffers (holding only
its own rows of every PARTITION argument, as a process on its own GPU would),
created with MW_TRANSPORT_LOOPBACK: the executor's cross-rank branches — halo
send/recv groups, the MapReduce merge all-reduce, the
loop-condition all-reduce, the COPY re-replication allgather-v
 and the timings all-gather of the monitor — run
exactly as they do over NCCL, only the transport is device copies between the
threads' buffers.  Every output is compared with the oracle (bit-exact for
integer work) and with the one-rank result.
"""
import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import kernels as K  # noqa: E402
from oracle import sct  # noqa: E402
from paper_1510_06585_b200 import marrow as M  # noqa: E402
from paper_1510_06585_b200 import trees  # noqa: E402

DEV = "cuda:0"


def run_ranks(nranks, ppr, dist, fn, tune=()):
    """fn(rank, ctx, stream) on nranks loopback threads; returns their results."""
    gid = os.urandom(128)
    out, err = [None] * nranks, [None] * nranks

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                c = M.mw_ctx_create(0, r, nranks, ppr, gid, transport=M.MW_TRANSPORT_LOOPBACK)
                if dist is not None:
                    M.mw_set_distribution(c, dist)
                for k, v in tune:
                    M.mw_ctx_set_tuning(c, k, v)
                out[r] = fn(r, c, s)
                s.synchronize()
                c.destroy()
        except BaseException as e:  # noqa: BLE001 - re-raised in the main thread
            err[r] = e

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
        assert not t.is_alive(), "loopback rank hung"
    for e in err:
        if e is not None:
            raise e
    return out


def local_rows(c, node, L, rank):
    """This rank's contiguous row range [s0, s1) (its ppr partitions)."""
    info = M.mw_ctx_info(c)
    off, ln = M.mw_partition(c, node, L)
    f, p = info["first_part"], info["parts_per_rank"]
    return off[f], off[f + p - 1] + ln[f + p - 1], (off, ln)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def assemble(parts, shape, dtype):
    """Concatenate the ranks' (s0, array) row slices into the global array."""
    out = np.zeros(shape, dtype)
    for s0, a in parts:
        out[s0:s0 + len(a)] = a
    return out


CASES = [(2, 1, None), (2, 1, [0.3, 0.7]), (3, 1, [0.5, 0.0, 0.5]), (3, 1, [0.0, 0.6, 0.4]),
         (2, 2, [0.1, 0.4, 0.0, 0.5]), (3, 2, None)]


def _partitioned_map(node_fn, src, out_dtype, nranks, ppr, dist, tune=()):
    H = src.shape[0]

    def fn(r, c, s):
        node = node_fn()
        s0, s1, _ = local_rows(c, node, H, r)
        x = dev(src[s0:s1])
        y = torch.empty((s1 - s0,) + src.shape[1:], dtype=out_dtype, device=DEV)
        f = M.mw_run(c, node, [M.arg(x, local_offset=s0, global_shape=src.shape),
                               M.arg(y, local_offset=s0, global_shape=src.shape)])
        f.wait()
        return s0, y.cpu().numpy()

    return run_ranks(nranks, ppr, dist, fn, tune)


# ----------------------------------------------------------------- Map / Pipeline (no collective)
@pytest.mark.parametrize("nranks,ppr,dist", CASES)
def test_filter_ranks_bitwise(nranks, ppr, dist):
    H, W = 301, 640
    img = synth.np_rgba(3, 0, H * W).reshape(H, W, 4)
    want = K.mirror(K.solarize(K.gauss_noise(img, 4, 8), 128))
    parts = _partitioned_map(trees.filter_pipeline, img, torch.uint8, nranks, ppr, dist)
    assert np.array_equal(assemble(parts, img.shape, np.uint8), want)


@pytest.mark.parametrize("nranks,ppr,dist", CASES)
def test_segmentation_ranks_bitwise(nranks, ppr, dist):
    shape = (37, 64, 96)
    vol = synth.np_u8_stream(7, 0, int(np.prod(shape))).reshape(shape)
    want = K.segment(vol, 85, 170)
    parts = _partitioned_map(trees.segmentation, vol, torch.uint8, nranks, ppr, dist)
    assert np.array_equal(assemble(parts, shape, np.uint8), want)


# ----------------------------------------------------------------- MapReduce (merge all-reduce)
@pytest.mark.parametrize("nranks,ppr,dist", CASES)
def test_mapreduce_ranks_bit_identical(nranks, ppr, dist):
    n = 7 * (1 << 16) + 1234
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    trees_of = {"sum": lambda: trees.mapreduce(False), "dot": lambda: trees.mapreduce(True),
                "max": lambda: trees.mapreduce_sct(M.MW_REDUCE_MAX, True),
                "min": lambda: trees.mapreduce_sct(M.MW_REDUCE_MIN, True),
                "l2": lambda: M.mw_map_reduce_sct(M.mw_kernel_map_identity(), M.mw_pipeline(
                    [M.mw_kernel_term_map(M.MW_TERM_SQUARE), M.mw_kernel_reduce(M.MW_REDUCE_SUM),
                     M.mw_kernel_scalar_map(M.MW_SCALAR_SQRT)]))}
    single = {}
    c1 = M.mw_ctx_create(0, 0, 1, 1)
    for key, t in trees_of.items():
        args = [M.arg(dev(x))] + ([M.arg(dev(y))] if key not in ("sum", "l2") else [])
        single[key] = M.mw_run(c1, t(), args).wait().result()["reduced"]

    def fn(r, c, s):
        res = {}
        for key, t in trees_of.items():
            node = t()
            s0, s1, _ = local_rows(c, node, n, r)
            args = [M.arg(dev(x[s0:s1]), local_offset=s0, global_shape=(n,))]
            if key not in ("sum", "l2"):
                args.append(M.arg(dev(y[s0:s1]), local_offset=s0, global_shape=(n,)))
            res[key] = M.mw_run(c, node, args).wait().result()["reduced"]
        return res

    for res in run_ranks(nranks, ppr, dist, fn):
        for key, v in res.items():
            assert v == single[key], key   # the canonical sum: bit-identical for every split
    assert abs(single["sum"] - K.sum_(x)) <= 1e-12 * K.abs_sum(x)
    assert abs(single["dot"] - K.dot(x, y)) <= 1e-12 * K.abs_sum(x, y)
    prods = x.astype(np.float64) * y.astype(np.float64)
    assert single["max"] == prods.max() and single["min"] == prods.min()


def test_mapreduce_ranks_merge_sub():
    """A non-ADD merging function folds the per-partition partials in global
    partition order (R26); every rank forms the same value."""
    n = 5 * (1 << 16)
    x = synth.np_f32_um11(5, 0, n)
    dist = [0.4, 0.0, 0.2, 0.4]

    def fn(r, c, s):
        node = M.mw_map_reduce(M.mw_kernel_map_identity(), M.MW_MERGE_SUB)
        s0, s1, (off, ln) = local_rows(c, node, n, r)
        v = M.mw_run(c, node, [M.arg(dev(x[s0:s1]), local_offset=s0, global_shape=(n,))]).wait()
        return v.result()["reduced"], off, ln

    res = run_ranks(2, 2, dist, fn)
    off, ln = res[0][1], res[0][2]
    partials = [K.sum_(x[o:o + m]) for o, m in zip(off, ln) if m > 0]
    want = partials[0]
    for p in partials[1:]:
        want -= p
    for v, _, _ in res:
        assert v == res[0][0] and abs(v - want) <= 1e-12 * K.abs_sum(x)


# ----------------------------------------------------------------- hysteresis (halo + loop condition)
def oracle_hyst(gray, lo=173, hi=250):
    L = K.segment(gray, lo, hi)
    fixed, D = K.hyst_bfs(L)
    return K.hyst_finalize(fixed), D


@pytest.mark.parametrize("planes,fused", [(1, 1), (1, 0), (0, 0)])
@pytest.mark.parametrize("nranks,ppr,dist", CASES)
def test_hysteresis_ranks_bitwise_and_E(planes, fused, nranks, ppr, dist):
    """planes + fused: one cooperative kernel per rank for the whole loop, halo
    rows stored into the neighbouring ranks' planes, a rank barrier per pass;
    planes alone: per-pass kernels + transport halos + lagged all-reduce;
    bytes: the byte stencil."""
    H, W = 333, 515
    gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
    want, D = oracle_hyst(gray)

    def fn(r, c, s):
        got = []
        for ce in (1, 4):
            node = trees.hysteresis(check_every=ce)
            s0, s1, _ = local_rows(c, node, H, r)
            dst = torch.empty((s1 - s0, W), dtype=torch.uint8, device=DEV)
            src = dev(gray[s0:s1])
            l0 = M.mw_ctx_launch_count(c)
            res = M.mw_run(c, node, [M.arg(src, local_offset=s0, global_shape=(H, W)),
                                     M.arg(dst, local_offset=s0, global_shape=(H, W))]).wait().result()
            got.append((s0, dst.cpu().numpy(), res["executions"], res["converged"],
                        M.mw_ctx_launch_count(c) - l0))
        return got

    res = run_ranks(nranks, ppr, dist, fn, tune=[(M.MW_TUNE_HYST_PLANES, planes), (M.MW_TUNE_HYST_FUSED, fused)])
    for i in range(2):
        out = assemble([(g[i][0], g[i][1]) for g in res], (H, W), np.uint8)
        assert np.array_equal(out, want)
        for g in res:
            assert g[i][2] == D + 1 and g[i][3]
            if planes and fused:   # the whole loop is one launch per rank (+ pack/unpack/setup)
                assert g[i][4] <= 8, g[i][4]


def test_hysteresis_ranks_max_iters():
    H, W = 200, 300
    gray = synth.np_u8_stream(8, 5, H * W).reshape(H, W)
    L = K.segment(gray, 173, 250)
    _, D = K.hyst_bfs(L)
    n = max(1, D - 4)

    def fn(r, c, s):
        node = trees.hysteresis(max_iters=n)
        s0, s1, _ = local_rows(c, node, H, r)
        dst = torch.empty((s1 - s0, W), dtype=torch.uint8, device=DEV)
        res = M.mw_run(c, node, [M.arg(dev(gray[s0:s1]), local_offset=s0, global_shape=(H, W)),
                                 M.arg(dst, local_offset=s0, global_shape=(H, W))]).wait().result()
        return s0, dst.cpu().numpy(), res

    res = run_ranks(3, 1, [0.3, 0.3, 0.4], fn)
    out = assemble([(a, b) for a, b, _ in res], (H, W), np.uint8)
    assert np.array_equal(out, K.hyst_finalize(K.hyst_bfs(L, n)[0]))
    assert all(x["executions"] == n and not x["converged"] for _, _, x in res)


@pytest.mark.parametrize("nranks,ppr", [(2, 1), (3, 2)])
def test_hysteresis_ranks_fronts_across_rank_boundaries(nranks, ppr):
    """Fronts running along constructed paths across the rank boundaries
    (vertical lines through the row split, a serpentine through every
    partition): the fused cross-rank loop's forced boundary strips, the push
    stamps of the partitions and the device barrier's loop condition must
    give the oracle's iterates and E."""
    H, W = 240, 1100
    paths = [[(10 + i, 300) for i in range(200)],                      # vertical, crosses every split
             [(5 + i, 900 + (i % 2)) for i in range(223)]]              # zig-zag column
    # serpentine, legs 3 rows apart, through every rank (E = 8611 < max_iters)
    pts, y, x, d = [], 1, 1, 1
    for leg in range(70):
        for _ in range(120):
            pts.append((y, x))
            x += d
        for _ in range(3):
            pts.append((y, x))
            y += 1
        d = -d
        if y + 4 >= H:
            break
    paths.append(pts)
    for k, p in enumerate(paths):
        gray = np.zeros((H, W), dtype=np.uint8)
        for (yy, xx) in p:
            gray[yy, xx] = 200
        gray[p[0]] = 255
        want, D = oracle_hyst(gray)

        def fn(r, c, s):
            node = trees.hysteresis()
            s0, s1, _ = local_rows(c, node, H, r)
            dst = torch.empty((s1 - s0, W), dtype=torch.uint8, device=DEV)
            res = M.mw_run(c, node, [M.arg(dev(gray[s0:s1]), local_offset=s0, global_shape=(H, W)),
                                     M.arg(dst, local_offset=s0, global_shape=(H, W))]).wait().result()
            return s0, dst.cpu().numpy(), res

        res = run_ranks(nranks, ppr, None, fn)
        out = assemble([(a, b) for a, b, _ in res], (H, W), np.uint8)
        assert np.array_equal(out, want), k
        assert all(x["executions"] == D + 1 and x["converged"] for _, _, x in res), (k, D)


# ----------------------------------------------------------------- N-body (COPY re-replication)
@pytest.mark.parametrize("nranks,ppr,dist", CASES)
def test_nbody_ranks_replicated_bitwise(nranks, ppr, dist):
    N = 2048 + 256
    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -11)
    c1 = M.mw_ctx_create(0, 0, 1, 1)
    p1, v1 = dev(pos), dev(vel)
    M.mw_run(c1, trees.nbody(3), [M.arg(p1, M.MW_COPY), M.arg(v1, M.MW_COPY)]).wait()
    p1, v1 = p1.cpu().numpy(), v1.cpu().numpy()

    def fn(r, c, s):
        p, v = dev(pos), dev(vel)
        M.mw_run(c, trees.nbody(3), [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)]).wait()
        return p.cpu().numpy(), v.cpu().numpy()

    for p, v in run_ranks(nranks, ppr, dist, fn):
        # every rank holds the whole replicated state, identical to one rank's
        assert np.array_equal(p.view(np.uint32), p1.view(np.uint32))
        assert np.array_equal(v.view(np.uint32), v1.view(np.uint32))
    po, vo, _ = K.nbody_step(pos, vel, 1e-4, 1e-3)   # first step against the fp64 oracle
    c1b = M.mw_ctx_create(0, 0, 1, 1)
    pp, vv = dev(pos), dev(vel)
    M.mw_run(c1b, trees.nbody(1), [M.arg(pp, M.MW_COPY), M.arg(vv, M.MW_COPY)]).wait()
    assert np.allclose(pp.cpu().numpy()[:, :3], po[:, :3], rtol=0, atol=1e-6)


# ----------------------------------------------------------------- monitoring / rebalance (timings all-gather)
def test_timings_allgather_and_identical_rebalance():
    """mw_last_timings all-gathers every partition's compute time; the
    balance step then takes the same decision on every rank."""
    N = 4096

    pos, vel = synth.np_nbody(9, 0, N, 2.0 ** -12)

    def fn(r, c, s):
        M.mw_ctx_set_slowdown(c, 2, 6.0)   # partition 2 (rank 1's first) is slow
        p, v = dev(pos), dev(vel)
        node = trees.nbody(1)
        hist = []
        for step in range(5):
            M.mw_run(c, node, [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)]).wait()
            ms, wall = M.mw_last_timings(c)
            trig = M.mw_rebalance(c)
            hist.append((ms, trig, M.mw_get_distribution(c)))
        return hist, p.cpu().numpy()

    res = run_ranks(2, 2, None, fn)
    h0, h1 = res[0][0], res[1][0]
    for (ms0, t0, d0), (ms1, t1, d1) in zip(h0, h1):
        assert ms0 == ms1 and t0 == t1 and d0 == d1   # the same gathered vector, same decision
        assert all(m > 0 for m in ms0)
    assert [t for _, t, _ in h0].index(True) == 2     # third unbalanced run triggers
    assert h0[-1][2][2] < 0.5 * h0[-1][2][0]
    assert np.array_equal(res[0][1], res[1][1])


def test_loopback_group_mismatch_is_an_error():
    """Ranks issuing different collectives surface MW_E_NCCL instead of
    corrupting data (mw_run on a MapReduce on one rank only would hang NCCL;
    the loopback transport times out — here we only check the id/nranks
    validation, which fails fast)."""
    gid = os.urandom(128)
    errs = []

    def w(r, n):
        try:
            M.mw_ctx_create(0, r, n, 1, gid, transport=M.MW_TRANSPORT_LOOPBACK)
        except M.MwError as e:
            errs.append(e.status)

    t1 = threading.Thread(target=w, args=(0, 2))
    t1.start()
    import time
    time.sleep(0.5)
    w(0, 3)   # a second rank 0 with another nranks: rejected at once
    assert M.MW_E_INVALID_SPEC in errs
    w(1, 2)   # completes the group so thread 1 returns
    t1.join(timeout=60)


# ----------------------------------------------------------------- full config sizes, several ranks
@pytest.mark.slow
def test_config_hysteresis_16384_ranks_E48():
    """BASELINE config C5a through the cross-rank path: 3 ranks with a zero
    share, and 2 ranks x 4 partitions; every rank generates only its rows."""
    n = 16384
    gray = synth.host_u8_stream(synth.SEED_HYST, 0, n * n).reshape(n, n)
    want, D = oracle_hyst(gray)
    assert D + 1 == 48
    del gray
    for nranks, ppr, dist in ((3, 1, [0.5, 0.0, 0.5]), (2, 4, None)):
        def fn(r, c, s):
            node = trees.hysteresis()
            s0, s1, _ = local_rows(c, node, n, r)
            src = torch.empty((s1 - s0, n), dtype=torch.uint8, device=DEV)
            if s1 > s0:
                synth.dev_fill_u8_stream(src, synth.SEED_HYST, s0 * n, stream=s)
            dst = torch.empty_like(src)
            res = M.mw_run(c, node, [M.arg(src, local_offset=s0, global_shape=(n, n)),
                                     M.arg(dst, local_offset=s0, global_shape=(n, n))]).wait().result()
            return s0, s1, bool(np.array_equal(dst.cpu().numpy(), want[s0:s1])), res
        for s0, s1, ok, res in run_ranks(nranks, ppr, dist, fn):
            assert ok, (nranks, ppr, s0, s1)
            assert res["executions"] == 48 and res["converged"]


@pytest.mark.slow
def test_config_mapreduce_2p30_ranks_exact():
    n = 1 << 30
    exact_s = -383760319397 / 2.0 ** 23
    exact_d = 643773335475643653 / 2.0 ** 46

    def fn(r, c, s):
        out = []
        for dot in (False, True):
            node = trees.mapreduce(dot)
            s0, s1, _ = local_rows(c, node, n, r)
            x = torch.empty(s1 - s0, dtype=torch.float32, device=DEV)
            synth.dev_fill_f32_um11(x, synth.SEED_MR_X, s0, stream=s)
            args = [M.arg(x, local_offset=s0, global_shape=(n,))]
            if dot:
                y = torch.empty(s1 - s0, dtype=torch.float32, device=DEV)
                synth.dev_fill_f32_um11(y, synth.SEED_MR_Y, s0, stream=s)
                args.append(M.arg(y, local_offset=s0, global_shape=(n,)))
            out.append(M.mw_run(c, node, args).wait().result()["reduced"])
            del args
        return out

    res = run_ranks(3, 1, [0.25, 0.0, 0.75], fn)
    for s_, d_ in res:
        assert s_ == res[0][0] and d_ == res[0][1]
        assert abs(s_ - exact_s) <= 1e-12 * abs(exact_s) and abs(d_ - exact_d) <= 1e-12 * abs(exact_d)


@pytest.mark.slow
def test_config_nbody_2p20_ranks_step_bitwise():
    """One N-body step of the 2^20 config on 2 ranks (x 2 partitions, one
    empty) equals the one-rank step bit for bit on every rank (COPY
    re-replication through the transport's allgather-v)."""
    N = 1 << 20
    pos = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    vel = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    synth.dev_fill_nbody(pos, vel, synth.SEED_NBODY, 0, 2.0 ** -20)
    p1, v1 = pos.clone(), vel.clone()
    c1 = M.mw_ctx_create(0, 0, 1, 1)
    M.mw_run(c1, trees.nbody(1), [M.arg(p1, M.MW_COPY), M.arg(v1, M.MW_COPY)]).wait()
    torch.cuda.synchronize()

    def fn(r, c, s):
        p, v = pos.clone(), vel.clone()
        M.mw_run(c, trees.nbody(1), [M.arg(p, M.MW_COPY), M.arg(v, M.MW_COPY)]).wait()
        return bool(torch.equal(p, p1)) and bool(torch.equal(v, v1))

    assert all(run_ranks(2, 2, [0.3, 0.0, 0.3, 0.4], fn))
