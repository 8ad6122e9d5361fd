"""Pins of the oracle to things other than itself (CPU only).

Each test pins one oracle function to what the paper or mathematics fixes:
closed forms, invariants, library routines (PIL, scipy, mpmath, fractions),
brute force on tiny inputs, and independently computed reference values
(tests/golden/, cited).  A plausible mistake (dropped term, wrong sign or
index, transposed operand) fails at least one of them.
"""
import math
import random
import struct
import zlib
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import balance as B
from oracle import brute
from oracle import kernels as K
from oracle import partition as P
from oracle import sct
from tests.golden_io import config_reference, filter_w4h2

REF = config_reference()


def f32bits(v):
    return struct.unpack("<I", struct.pack("<f", v))[0]


# ----------------------------------------------------------------- generators
def test_splitmix64_published_vector():
    # SplitMix64 seed 0 reference outputs (the standard test vector)
    want = [int(v, 16) for v in REF["splitmix64_seed0"]]
    got = [int(v) for v in synth.np_splitmix64(0, np.arange(3))]
    assert got == want
    assert synth.host_lib().synth_splitmix64(0, 0) == want[0]
    assert int(synth.np_splitmix64(8, [0])[0]) == int(REF["splitmix64_seed8_i0"][0], 16)
    assert list(synth.host_u8_stream(8, 0, 8)) == [int(v) for v in REF["hyst_first_bytes"]]


def test_synth_numpy_matches_c():
    for seed in (1, 3, 9):
        assert np.array_equal(synth.np_f32_um11(seed, 1000, 777), synth.host_f32_um11(seed, 1000, 777))
        assert np.array_equal(synth.np_f32_u01(seed, 5, 333), synth.host_f32_u01(seed, 5, 333))
        assert np.array_equal(synth.np_u8_stream(seed, 13, 1001), synth.host_u8_stream(seed, 13, 1001))
        assert np.array_equal(synth.np_rgba(seed, 7, 300), synth.host_rgba(seed, 7, 300))
        p1, _ = synth.np_nbody(seed, 11, 50, 2.0 ** -20)
        p2, v2 = synth.host_nbody(seed, 11, 50, 2.0 ** -20)
        assert np.array_equal(p1, p2) and not v2.any()


def test_synth_f32_exact_grid():
    x = synth.host_f32_um11(5, 0, 1 << 16)
    u = (synth.np_splitmix64(5, np.arange(1 << 16)) >> np.uint64(40)).astype(np.int64)
    # exact: x == u * 2^-23 - 1 with integer u < 2^24
    assert np.array_equal(x.astype(np.float64) * 2.0 ** 23, (u - (1 << 23)).astype(np.float64))


# ----------------------------------------------------------------- saxpy
def test_saxpy_special_cases():
    y = synth.np_f32_um11(2, 0, 1000)
    x = synth.np_f32_um11(1, 0, 1000)
    assert np.array_equal(K.saxpy(0.0, x, y).view(np.uint32), y.view(np.uint32))
    assert np.array_equal(K.saxpy(2.5, np.zeros_like(x), y).view(np.uint32), y.view(np.uint32))
    assert K.saxpy(2.0, np.float32([3.0]), np.float32([1.0]))[0] == 7.0


def test_saxpy_single_rounding_pin():
    # fma gives exactly 2^-24; a separately rounded product gives 0 (reading R8)
    a = np.float32(1 + 2.0 ** -12)
    y = np.float32(-(1 + 2.0 ** -11))
    assert K.saxpy(float(a), np.float32([a]), np.float32([y]))[0] == 2.0 ** -24
    assert np.float32(a * a) + y == 0.0


def test_saxpy_vs_exact_rational_rounding():
    rng = random.Random(7)
    xs = [struct.unpack("<f", struct.pack("<f", rng.uniform(-1, 1) * 2.0 ** rng.randint(-30, 30)))[0]
          for _ in range(400)]
    ys = [struct.unpack("<f", struct.pack("<f", rng.uniform(-1, 1) * 2.0 ** rng.randint(-30, 30)))[0]
          for _ in range(400)]
    a = struct.unpack("<f", struct.pack("<f", 1.7320508))[0]
    got = K.saxpy(a, np.float32(xs), np.float32(ys))
    want = brute.saxpy_exact(a, xs, ys)
    assert [f32bits(float(g)) for g in got] == [f32bits(w) for w in want]


def test_saxpy_config_reference():
    n = 1 << 20
    x = synth.host_f32_um11(synth.SEED_SAXPY_X, 0, n)
    y = synth.host_f32_um11(synth.SEED_SAXPY_Y, 0, n)
    yp = K.saxpy(2.5, x, y)
    assert float(x[0]) == float(REF["saxpy_x0"][0])
    assert float(y[0]) == float(REF["saxpy_y0"][0])
    assert float(yp[0]) == float(REF["saxpy_yp0"][0])
    assert zlib.crc32(yp.tobytes()) == int(REF["saxpy_crc32"][0], 16)


# ----------------------------------------------------------------- noise
def test_lowbias32_vectors_and_brute():
    assert [K.lowbias32(v) for v in (1, 2, 3)] == [int(h, 16) for h in REF["lowbias32_1_2_3"]]
    rng = random.Random(1)
    for _ in range(2000):
        v = rng.getrandbits(32)
        assert K.lowbias32(v) == brute.lowbias32(v)


def test_noise_scale_zero_is_identity():
    img = synth.np_rgba(3, 0, 64 * 33).reshape(33, 64, 4)
    assert np.array_equal(K.gauss_noise(img, 4, 0), img)


def test_noise_matches_brute_and_clamps():
    rng = np.random.default_rng(0)
    H, W = 9, 13
    img = rng.integers(0, 256, size=(H, W, 4), dtype=np.uint8)
    img[0, :, :3] = 250   # top clamp corner
    img[1, :, :3] = 5     # bottom clamp corner
    for seed, S in ((4, 8), (123456, 13), (0xFFFFFFFF, 40)):
        out = K.gauss_noise(img, seed, S, y0=5)
        for y in range(H):
            for x in range(W):
                want = brute.noise_pixel(tuple(int(v) for v in img[y, x]), (5 + y) * W + x, seed, S)
                assert tuple(int(v) for v in out[y, x]) == want
    out = K.gauss_noise(img, 4, 40)
    assert out[0, :, :3].max() == 255 and out[1, :, :3].min() == 0
    assert np.array_equal(out[..., 3], img[..., 3])


def test_noise_binomial_statistics():
    # n_c = (Bin(10,1/2) - 5) * S: mean 0, variance 2.5 S^2 (closed form), channels independent
    S = 8
    img = np.full((1024, 1024, 4), 128, dtype=np.uint8)
    n = K.gauss_noise(img, 4, S).astype(np.int64)[..., :3] - 128
    N = n.shape[0] * n.shape[1]
    for c in range(3):
        v = n[..., c].ravel()
        assert abs(v.mean()) < 5 * math.sqrt(2.5 * S * S / N)
        assert abs(v.var() / (2.5 * S * S) - 1) < 0.01
        assert set(np.unique(v)) <= {S * (k - 5) for k in range(11)}
    assert abs(np.corrcoef(n[..., 0].ravel(), n[..., 1].ravel())[0, 1]) < 0.01


def test_noise_partition_offset_trait():
    img = synth.np_rgba(3, 0, 20 * 7).reshape(20, 7, 4)
    whole = K.gauss_noise(img, 9, 8)
    parts = [K.gauss_noise(img[a:b], 9, 8, y0=a) for a, b in ((0, 3), (3, 4), (4, 20))]
    assert np.array_equal(np.concatenate(parts), whole)


# ----------------------------------------------------------------- solarize / mirror
def test_solarize_matches_pil():
    from PIL import Image, ImageOps
    v = np.arange(256, dtype=np.uint8)
    rgb = np.stack([v, v[::-1], np.roll(v, 77)], axis=-1).reshape(16, 16, 3)
    rgba = np.concatenate([rgb, np.full((16, 16, 1), 9, np.uint8)], axis=-1)
    for T in (0, 1, 128, 200, 255):
        want = np.asarray(ImageOps.solarize(Image.fromarray(rgb, "RGB"), threshold=T))
        got = K.solarize(rgba, T)
        assert np.array_equal(got[..., :3], want), T
        assert np.array_equal(got[..., 3], rgba[..., 3])


def test_mirror_matches_pil_and_involution():
    from PIL import Image, ImageOps
    img = synth.np_rgba(11, 0, 5 * 9).reshape(5, 9, 4)
    want = np.asarray(ImageOps.mirror(Image.fromarray(img, "RGBA")))
    assert np.array_equal(K.mirror(img), want)
    assert np.array_equal(K.mirror(K.mirror(img)), img)
    one = img[:, :1].copy()
    assert np.array_equal(K.mirror(one), one)


def test_filter_pipeline_golden_vector():
    Kg, hg, rows = filter_w4h2()
    assert K.lowbias32(4 ^ 0x9E3779B9) == Kg
    for i, h in hg.items():
        assert K.lowbias32(i ^ Kg) == h
    W, H = 4, 2
    img = np.array([[(16 * i) % 256, (255 - 16 * i) % 256, (37 * i) % 256, 200]
                    for i in range(W * H)], dtype=np.uint8).reshape(H, W, 4)
    tree = sct.Pipeline([sct.Leaf("gauss_noise", {"seed": 4, "scale": 8}),
                         sct.Leaf("solarize", {"threshold": 128}), sct.Leaf("mirror")])
    out = sct.evaluate(tree, img).value
    assert [[tuple(int(c) for c in px) for px in row] for row in out] == rows
    # the composed function written independently (brute) agrees
    lists = [[tuple(int(c) for c in img[y, x]) for x in range(W)] for y in range(H)]
    assert brute.filter_pipeline(lists, 4, 8, 128) == rows


def test_pipeline_equals_composition_random():
    img = synth.np_rgba(3, 0, 17 * 23).reshape(17, 23, 4)
    tree = sct.Pipeline([sct.Leaf("gauss_noise", {"seed": 4, "scale": 8}),
                         sct.Leaf("solarize", {"threshold": 128}), sct.Leaf("mirror")])
    out = sct.evaluate(tree, img).value
    lists = [[tuple(int(c) for c in img[y, x]) for x in range(23)] for y in range(17)]
    assert [[tuple(int(c) for c in px) for px in row] for row in out] == \
        brute.filter_pipeline(lists, 4, 8, 128)


@pytest.mark.slow
def test_filter_config_reference():
    H = W = 8192
    img = synth.host_rgba(synth.SEED_IMAGE, 0, H * W).reshape(H, W, 4)
    out = K.mirror(K.solarize(K.gauss_noise(img, synth.SEED_NOISE, 8), 128))
    assert tuple(int(v) for v in out[0, 0]) == tuple(int(v) for v in REF["filter_out_0_0"])
    assert tuple(int(v) for v in out[0, W - 1]) == tuple(int(v) for v in REF["filter_out_0_8191"])
    assert zlib.crc32(out.tobytes()) == int(REF["filter_crc32"][0], 16)


# ----------------------------------------------------------------- segmentation
def test_segment_boundaries_and_histogram():
    v = np.arange(256, dtype=np.uint8)
    out = K.segment(v, 85, 170)
    assert [int(out[i]) for i in (0, 84, 85, 169, 170, 255)] == [0, 0, 128, 128, 255, 255]
    assert np.all(np.diff(out.astype(int)) >= 0)
    assert set(np.unique(out)) == {0, 128, 255}
    a = synth.np_u8_stream(7, 0, 1 << 16)
    s = K.segment(a, 85, 170)
    assert (s == 0).sum() == (a < 85).sum()
    assert (s == 128).sum() == ((a >= 85) & (a < 170)).sum()
    assert (s == 255).sum() == (a >= 170).sum()
    assert np.array_equal(K.segment(a, 0, 256), np.full_like(a, 128))


@pytest.mark.slow
def test_segment_config_reference():
    n = 1024 * 1024 * 512
    a = synth.host_u8_stream(synth.SEED_SEGMENT, 0, n)
    s = K.segment(a, 85, 170)
    counts = np.bincount(s, minlength=256)
    assert [int(counts[0]), int(counts[128]), int(counts[255])] == [int(c) for c in REF["segment_counts"]]
    assert zlib.crc32(s.data) == int(REF["segment_crc32"][0], 16)


# ----------------------------------------------------------------- hysteresis (R11)
def _labels(rng, H, W, p_strong=0.03, p_weak=0.47):
    r = rng.random((H, W))
    return np.where(r < p_strong, 255, np.where(r < p_strong + p_weak, 128, 0)).astype(np.uint8)


def test_hyst_step_exhaustive_3x3_vs_brute():
    for code in range(3 ** 9):
        vals, c = [], code
        for _ in range(9):
            vals.append((0, 128, 255)[c % 3])
            c //= 3
        L = np.array(vals, dtype=np.uint8).reshape(3, 3)
        got, ch = K.hyst_step(L)
        want, wch = brute.hyst_step(L.tolist())
        assert got.tolist() == want and ch == wch


def test_hyst_bfs_equals_jacobi_and_scipy():
    from scipy import ndimage
    rng = np.random.default_rng(3)
    for trial in range(60):
        H, W = rng.integers(1, 40, size=2)
        L = _labels(rng, H, W)
        # literal Jacobi loop (while changed)
        cur, e, changed = L, 0, True
        levels = [L]
        while changed:
            cur, changed = K.hyst_step(cur)
            e += 1
            levels.append(cur)
        fixed, D = K.hyst_bfs(L)
        assert np.array_equal(fixed, cur) and e == D + 1
        # Loop_for(step, n) == promotion of BFS levels <= n
        for n in (0, 1, 2, D):
            assert np.array_equal(K.hyst_bfs(L, n)[0], levels[min(n, len(levels) - 1)])
        # library cross-check: final strong set = 8-connected components of (L>0) holding a 255
        lab, _ = ndimage.label(L > 0, structure=np.ones((3, 3)))
        keep = np.unique(lab[L == 255])
        want = np.isin(lab, keep[keep > 0]) & (L > 0)
        assert np.array_equal(fixed == 255, want)


def test_hyst_closed_forms():
    for H, W in ((5, 9), (7, 3), (4, 4), (1, 1)):
        L = np.full((H, W), 128, np.uint8)
        L[0, 0] = 255
        _, D = K.hyst_bfs(L)
        assert D + 1 == max(H, W) or (H == W == 1 and D == 0)
    for ell in (1, 5, 20):
        L = np.zeros((3, ell + 1), np.uint8)
        L[1, 0] = 255
        L[1, 1:] = 128
        _, D = K.hyst_bfs(L)
        assert D + 1 == ell + 1
    L = np.where(np.arange(30).reshape(5, 6) % 2, 128, 0).astype(np.uint8)  # no strong pixel
    out, D = K.hyst_bfs(L)
    assert D == 0 and np.array_equal(out, L)
    assert np.array_equal(K.hyst_finalize(np.uint8([0, 128, 255, 7])), np.uint8([0, 0, 255, 7]))


def test_hysteresis_tree_loop_semantics():
    rng = np.random.default_rng(5)
    gray = rng.integers(0, 256, size=(31, 29), dtype=np.uint8)
    step = sct.Leaf("hysteresis_step")
    tree = sct.Pipeline([sct.Leaf("segment", {"lo": 173, "hi": 250}),
                         sct.LoopWhileChanged(step, 10000),
                         sct.Leaf("hysteresis_finalize")])
    r = sct.evaluate(tree, gray)
    L = K.segment(gray, 173, 250)
    fixed, D = K.hyst_bfs(L)
    assert np.array_equal(r.value, K.hyst_finalize(fixed))
    loop = sct.evaluate(sct.LoopWhileChanged(step, 10000), L)
    assert loop.executions == D + 1 and loop.converged
    # Loop equals its unrolled body
    for n in (1, 2, 3):
        a = sct.evaluate(sct.LoopFor(step, n), L).value
        b = sct.evaluate(sct.Pipeline([step] * n), L).value if n >= 2 else sct.evaluate(step, L).value
        assert np.array_equal(a, b)
    # max_iters caps executions and reports non-convergence
    capped = sct.evaluate(sct.LoopWhileChanged(step, 1), L)
    assert capped.executions == 1 and (D == 0 or not capped.converged)


@pytest.mark.slow
def test_hysteresis_config_reference():
    n = 16384
    gray = synth.host_u8_stream(synth.SEED_HYST, 0, n * n).reshape(n, n)
    L = K.segment(gray, 173, 250)
    c = np.bincount(L.ravel(), minlength=256)
    assert [int(c[255]), int(c[128]), int(c[0])] == [int(v) for v in REF["hyst_initial"]]
    fixed, D = K.hyst_bfs(L)
    assert D == int(REF["hyst_D"][0])
    assert int((fixed == 255).sum()) == int(REF["hyst_final255"][0])
    assert int((fixed == 255).sum()) - int(c[255]) == int(REF["hyst_promoted"][0])
    assert zlib.crc32(K.hyst_finalize(fixed).data) == int(REF["hyst_crc32"][0], 16)


# ----------------------------------------------------------------- N-body
def test_nbody_special_cases():
    eps2 = 1e-4
    p1 = np.float32([[0.3, -0.2, 0.1, 1.0]])
    acc, _ = K.nbody_accel(p1, eps2)
    assert np.all(acc == 0.0)
    p2 = np.float32([[0.1, 0.2, 0.3, 0.5], [-0.4, 0.25, 0.7, 0.5]])
    acc, _ = K.nbody_accel(p2, eps2)
    assert np.array_equal(acc[1], -acc[0]) and np.any(acc[0] != 0)
    # body 0 feels body 1 along +d01 (attraction) with magnitude m r (r^2+eps2)^-3/2
    d = p2[1, :3].astype(np.float64) - p2[0, :3]
    r2 = float(d @ d)
    assert np.allclose(acc[0], 0.5 * d / (r2 + np.float64(np.float32(eps2))) ** 1.5, rtol=1e-14)


def test_nbody_symmetric_shell_and_momentum():
    eps2 = 1e-4
    dirs = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    pos = np.float32([[0, 0, 0, 1.0]] + [[0.5 * a, 0.5 * b, 0.5 * c, 0.25] for a, b, c in dirs])
    acc, cond = K.nbody_accel(pos, eps2, targets=np.int64([0]))
    assert np.abs(acc[0]).max() < 1e-15 * cond[0] + 1e-300
    p, _ = synth.np_nbody(9, 0, 300, 2.0 ** -8)
    p[:, 3] = synth.np_f32_u01(12, 0, 300) + np.float32(0.5)
    acc, _ = K.nbody_accel(p, eps2)
    mom = (p[:, 3:4].astype(np.float64) * acc).sum(axis=0)
    scale = (p[:, 3:4].astype(np.float64) * np.abs(acc)).sum()
    assert np.abs(mom).max() < 1e-13 * scale


def test_nbody_vs_mpmath():
    import mpmath
    mpmath.mp.dps = 40
    p, _ = synth.np_nbody(9, 0, 16, 2.0 ** -4)
    eps2 = np.float32(1e-4)
    acc, _ = K.nbody_accel(p, float(eps2))
    for i in range(16):
        a = [mpmath.mpf(0)] * 3
        for j in range(16):
            d = [mpmath.mpf(float(p[j, c])) - mpmath.mpf(float(p[i, c])) for c in range(3)]
            r2 = d[0] ** 2 + d[1] ** 2 + d[2] ** 2 + mpmath.mpf(float(eps2))
            s = mpmath.mpf(float(p[j, 3])) / r2 ** mpmath.mpf(1.5)
            a = [a[c] + d[c] * s for c in range(3)]
        ref = np.array([float(v) for v in a])
        assert np.abs(acc[i] - ref).max() <= 1e-13 * np.abs(ref).max()


def test_nbody_step_free_particles_closed_form():
    """Symplectic Euler (R12) with a = 0 — one body, or bodies of mass 0 —
    is uniform motion: v' = v and, with exactly representable p, v and dt,
    p_k = p_0 + k v dt exactly after k steps (closed form, no fp64 detour)."""
    dt = 2.0 ** -10
    p = np.float32([[0.5, -0.25, 0.125, 1.0]])
    v = np.float32([[0.25, 0.5, -1.0, 0.0]])
    for k in range(1, 6):
        p, v, acc = K.nbody_step(p, v, 1e-4, dt)
        assert np.all(acc == 0.0) and np.array_equal(v[0, :3], np.float32([0.25, 0.5, -1.0]))
        want = [0.5 + k * 0.25 * dt, -0.25 + k * 0.5 * dt, 0.125 - k * dt]
        assert [Fraction(float(c)) for c in p[0, :3]] == [Fraction(w) for w in want]
        assert p[0, 3] == 1.0
    # many bodies, all massless: every body moves on its own straight line
    pos, _ = synth.np_nbody(9, 0, 50, 0.0)
    vel = np.zeros_like(pos)
    vel[:, :3] = np.float32(2.0 ** -4)
    po, vo, acc = K.nbody_step(pos, vel, 1e-4, dt)
    assert np.all(acc == 0.0) and np.array_equal(vo, vel)
    want = [[Fraction(float(c)) + Fraction(1, 2 ** 14) for c in row[:3]] for row in pos]
    got = [[Fraction(float(c)) for c in row[:3]] for row in po]
    for g, w, row in zip(got, want, pos):   # exact when representable, else one rounding
        for gc, wc in zip(g, w):
            assert abs(gc - wc) <= Fraction(abs(float(np.spacing(np.float32(float(wc)))))) / 2


def test_nbody_step_antisymmetric_pair_closed_form():
    """Two equal masses at rest at (+-x, 0, 0): each is pulled toward the
    other with a = m (2x) / ((2x)^2 + eps^2)^(3/2) (closed form, mpmath), then
    v' = a dt, p' = p + v' dt, rounded once to binary32 (R12): the pair stays
    mirror-symmetric bit for bit, and the values agree with the closed form
    to half an fp32 ulp."""
    import mpmath
    mpmath.mp.dps = 50
    x, m, eps2, dt = 0.375, 0.5, np.float32(1e-4), np.float32(1e-3)
    pos = np.float32([[x, 0, 0, m], [-x, 0, 0, m]])
    vel = np.zeros_like(pos)
    po, vo, acc = K.nbody_step(pos, vel, float(eps2), float(dt))
    d = mpmath.mpf(2 * x)
    a = mpmath.mpf(m) * d / (d ** 2 + mpmath.mpf(float(eps2))) ** mpmath.mpf(1.5)
    v1 = a * mpmath.mpf(float(dt))
    p1 = mpmath.mpf(x) - v1 * mpmath.mpf(float(dt))
    assert abs(acc[0, 0] - float(-a)) <= 1e-15 * float(a) and acc[0, 1] == acc[0, 2] == 0.0
    assert abs(float(vo[0, 0]) - float(-v1)) <= float(np.spacing(np.float32(float(v1)))) / 2
    assert abs(float(po[0, 0]) - float(p1)) <= float(np.spacing(np.float32(float(p1)))) / 2
    assert vo[1, 0] == -vo[0, 0] and po[1, 0] == -po[0, 0]
    assert np.all(vo[:, 1:3] == 0) and np.all(po[:, 1:3] == 0) and np.all(po[:, 3] == m)


@pytest.mark.slow
def test_nbody_config_reference():
    N = 1 << 20
    pos, _ = synth.host_nbody(synth.SEED_NBODY, 0, N, 2.0 ** -20)
    samples = synth.nbody_sample_indices(N, 4)
    assert [int(s) for s in samples] == [int(v) for v in REF["nbody_samples_k0_3"]]
    r2 = (pos[:, :3].astype(np.float64) ** 2).sum(axis=1)
    assert int(np.argmin(r2)) == int(REF["nbody_nearest_origin"][0])
    bodies = sorted(REF["nbody_acc"])
    acc, cond = K.nbody_accel(pos, 1e-4, targets=np.int64(bodies))
    for k, b in enumerate(bodies):
        want, wc = REF["nbody_acc"][b]
        # serial fp64 fold over 2^20 terms vs the reference's pairwise fold:
        # agreement within the fold's error bound N*eps*C_i (~2.3e-10 * C_i)
        assert np.abs(acc[k] - want).max() <= 2.3e-10 * cond[k]
        assert abs(cond[k] / np.linalg.norm(acc[k]) - wc) < 0.06


# ----------------------------------------------------------------- MapReduce
def test_abs_sum_pins():
    """sum |terms| (the conditioning scale of the MapReduce tolerance, SURVEY
    §8(c) c.5): +-1 sequences sum |.| to n exactly whatever their signed sum;
    exact rational brute force (fractions) for random fp32 inputs (sum and
    dot terms); sign flips of x or y do not change it; it dominates |sum|."""
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 1000, 4097):
        s = np.where(rng.integers(0, 2, n) == 1, 1.0, -1.0).astype(np.float32)
        assert K.abs_sum(s) == float(n)
        assert K.abs_sum(s, s) == float(n) and K.abs_sum(s, -s) == float(n)
        assert K.sum_(s) == float(np.sum(s.astype(np.int64)))
    for n in (1, 10, 333, 2000):
        x = synth.np_f32_um11(21, 0, n) * np.float32(2.0 ** rng.integers(-20, 20))
        y = synth.np_f32_um11(22, 0, n)
        ex = sum(abs(Fraction(float(v))) for v in x)
        exd = sum(abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, y))
        assert abs(Fraction(K.abs_sum(x)) - ex) <= ex * Fraction(1, 2 ** 52)
        assert abs(Fraction(K.abs_sum(x, y)) - exd) <= exd * Fraction(1, 2 ** 52)
        assert K.abs_sum(-x) == K.abs_sum(x) and K.abs_sum(x, -y) == K.abs_sum(x, y)
        assert K.abs_sum(x) >= abs(K.sum_(x)) and K.abs_sum(x, y) >= abs(K.dot(x, y))
        assert K.abs_sum(np.abs(x)) == K.sum_(np.abs(x))   # one sign: abs_sum = sum


def test_mapreduce_closed_forms():
    n = (1 << 25) + 3
    ones = np.ones(n, np.float32)
    assert K.sum_(ones) == float(n)                        # fp32 fold would stall at 2^24
    x = (np.arange(1 << 20) % 1024).astype(np.float32) / np.float32(1024)
    assert K.sum_(x) == 523776.0                           # 1024 * sum_{k<1024} k/1024
    y = synth.np_f32_um11(6, 0, 1000)
    for k in (0, 17, 999):
        e = np.zeros(1000, np.float32)
        e[k] = 1
        assert K.dot(y, e) == float(y[k])
    assert K.sum_(np.zeros(0, np.float32)) == 0.0


def test_mapreduce_vs_exact_fractions():
    for seed in range(4):
        x = synth.np_f32_um11(5 + seed, 0, 3001)
        y = synth.np_f32_um11(6 + seed, 0, 3001)
        xs = [float(v) for v in x]
        ys = [float(v) for v in y]
        es, ed = brute.exact_sum(xs), brute.exact_dot(xs, ys)
        assert abs(Fraction(K.sum_(x)) - es) <= abs(es) * Fraction(1, 10 ** 14) + Fraction(1, 10 ** 300)
        assert abs(Fraction(K.dot(x, y)) - ed) <= abs(ed) * Fraction(1, 10 ** 14) + Fraction(1, 10 ** 300)


def test_fold_chunks_equal_single_fold():
    x = synth.np_f32_um11(5, 0, 100000)
    y = synth.np_f32_um11(6, 0, 100000)
    f = K.Fold()
    for a in range(0, 100000, 7919):
        f.add(x[a:a + 7919], y[a:a + 7919])
    assert f.value == K.dot(x, y)
    tree = sct.MapReduce(sct.Leaf("map_product"))
    assert sct.evaluate(tree, (x, y)).reduced == K.dot(x, y)


@pytest.mark.slow
def test_mapreduce_config_exact():
    n, chunk = 1 << 30, 1 << 25
    fs, fd = K.Fold(), K.Fold()
    usum, dsum = 0, 0
    for a in range(0, n, chunk):
        ux = (synth.np_splitmix64(5, np.arange(a, a + chunk, dtype=np.uint64)) >> np.uint64(40)).astype(np.int64)
        uy = (synth.np_splitmix64(6, np.arange(a, a + chunk, dtype=np.uint64)) >> np.uint64(40)).astype(np.int64)
        usum += int(ux.sum())
        # exact integer dot of (ux - 2^23)(uy - 2^23): split to stay inside int64
        dx, dy = ux - (1 << 23), uy - (1 << 23)
        dsum += int((dx * dy).sum(dtype=np.int64))
        x = (dx.astype(np.float32) * np.float32(2.0 ** -23))
        y = (dy.astype(np.float32) * np.float32(2.0 ** -23))
        fs.add(x)
        fd.add(x, y)
    exact_sum = Fraction(usum - n * (1 << 23), 1 << 23)
    exact_dot = Fraction(dsum, 1 << 46)
    assert exact_sum == Fraction(int(REF["mapreduce_sum_num"][0]), 1 << int(REF["mapreduce_sum_den_log2"][0]))
    assert exact_dot == Fraction(int(REF["mapreduce_dot_num"][0]), 1 << int(REF["mapreduce_dot_den_log2"][0]))
    assert abs(Fraction(fs.value) - exact_sum) <= abs(exact_sum) * Fraction(1, 10 ** 13)
    assert abs(Fraction(fd.value) - exact_dot) <= abs(exact_dot) * Fraction(1, 10 ** 13)


# ----------------------------------------------------------------- tree semantics
def test_kernel_execution_order_fig1():
    fig1 = sct.Pipeline([sct.Leaf("segment", {"lo": 1, "hi": 2}),
                         sct.LoopWhileChanged(sct.Leaf("hysteresis_step"), 100),
                         sct.Leaf("hysteresis_finalize")])
    assert sct.kernel_execution_order(fig1, [3]) == [0, 1, 1, 1, 2]      # S:80 / P:130
    assert sct.kernel_execution_order(sct.Leaf("mirror"), []) == [0]
    assert sct.kernel_execution_order(sct.Map(sct.Pipeline([sct.Leaf("mirror"), sct.Leaf("solarize")])), []) == [0, 1]
    with pytest.raises(KeyError):
        sct.kernel_execution_order(fig1, [])
    tree = sct.Pipeline([sct.LoopFor(sct.Leaf("mirror"), 2), sct.Leaf("solarize")])
    assert sct.kernel_execution_order(tree, []) == [0, 0, 1]


def test_tree_typing():
    with pytest.raises(ValueError):
        sct.Pipeline([sct.Leaf("mirror")])
    with pytest.raises(ValueError):
        sct.sig(sct.Pipeline([sct.Leaf("mirror"), sct.Leaf("segment", {"lo": 1, "hi": 2})]))
    assert sct.sig(sct.MapReduce(sct.Leaf("map_product"))) == (sct.VEC2, "scalar")
    img = synth.np_rgba(3, 0, 6 * 10).reshape(6, 10, 4)
    assert np.array_equal(sct.evaluate(sct.LoopFor(sct.Leaf("mirror"), 2), img).value, img)


# ----------------------------------------------------------------- partitioner
def test_granule_spec_examples():
    assert P.granule([(4, 2), (4, 1)], align=16) == 16
    assert P.granule([(1, 1)], align=1) == 1
    with pytest.raises(P.EpuNuError):
        P.granule([(3, 2)])
    assert P.granule([(6, 1), (4, 1)], align=1) == 12


def test_partition_examples():
    assert P.partition(1024, 16, [0.75, 0.25]) == ([0, 768], [768, 256])
    assert P.partition(8192, 1, [1 / 3, 1 / 3, 1 / 3])[1] == [2731, 2731, 2730]
    assert P.partition(8192, 1, [0.5, 0.3, 0.2, 0.0])[1] == [4096, 2458, 1638, 0]
    assert P.partition(100, 1, [1.0]) == ([0], [100])
    assert P.partition(8, 16, [0.5, 0.5]) == ([0, 0], [0, 8])                     # tail rule
    with pytest.raises(P.InvalidSpec):
        P.partition(8, 16, [0.5, 0.5], strict=True)
    for bad in ([0.5, 0.6], [-0.1, 1.1], [0.0, 0.0], []):
        with pytest.raises(P.InvalidSpec):
            P.partition(10, 1, bad)


def test_partition_brute_force_optimality():
    rng = random.Random(11)
    for _ in range(1500):
        k = rng.randint(1, 4)
        U = rng.randint(0, 12)
        g = rng.choice([1, 2, 4])
        w = [rng.choice([0, 1, 2, 3, 5, 8]) for _ in range(k)]
        if not any(w):
            w[0] = 1
        d = [x / sum(w) for x in w]
        tail = rng.randint(0, g - 1)
        L = U * g + tail
        off, ln = P.partition(L, g, d)
        assert sum(ln) == L and off == [sum(ln[:i]) for i in range(k)]
        units = [(n - (tail if i == max(j for j in range(k) if d[j] > 0) else 0)) // g
                 for i, n in enumerate(ln)]
        assert all(n % g == 0 for n in [u * g for u in units])
        assert all(u == 0 for u, x in zip(units, d) if x == 0)
        # largest remainder minimises max |u - dU| and sum |u - dU| over all splits
        best_max = best_l1 = float("inf")

        def rec(i, left, acc):
            nonlocal best_max, best_l1
            if i == k - 1:
                c = acc + [left]
                if any(c[j] > 0 and d[j] == 0 for j in range(k)):
                    return
                best_max = min(best_max, max(abs(c[j] - d[j] * U) for j in range(k)))
                best_l1 = min(best_l1, sum(abs(c[j] - d[j] * U) for j in range(k)))
                return
            for u in range(left + 1):
                rec(i + 1, left - u, acc + [u])

        rec(0, U, [])
        assert max(abs(units[j] - d[j] * U) for j in range(k)) <= best_max + 1e-9
        assert sum(abs(units[j] - d[j] * U) for j in range(k)) <= best_l1 + 1e-9


# ----------------------------------------------------------------- balancer
def test_lbt_sequence_and_trigger():
    p, s = B.Params(), B.State()
    seq = []
    for _ in range(3):
        _, trig = B.step(p, s, [1.0, 2.0], [10, 10], [0.5, 0.5])
        seq.append((round(s.lbt, 4), trig))
    # 0.6667, 0.8889 then the 3rd unbalanced run crosses 0.95 (0.9630) and triggers
    assert seq[0] == (0.6667, False) and seq[1] == (0.8889, False) and seq[2][1] is True
    lbt = 0.0
    for _ in range(3):
        lbt = B.lbt_update(lbt, 1, 2 / 3)
    assert abs(lbt - 0.962962962) < 1e-8


def test_lbt_alternating_bound_and_decay():
    lbt, hi = 0.0, 0.0
    for n in range(200):
        lbt = B.lbt_update(lbt, n % 2 == 0, 2 / 3)
        hi = max(hi, lbt)
    w = 2 / 3
    assert hi <= w / (1 - (1 - w) ** 2) + 1e-12 and hi > 0.749   # sup = 0.75 (corrects S:467)
    lbt = 0.9
    for n in range(1, 6):
        lbt = B.lbt_update(lbt, 0, w)
        assert abs(lbt - 0.9 * (1 - w) ** n) < 1e-15


def test_deviation_direction():
    assert B.deviation([2.0, 1.0], [5, 5]) == 0.5
    assert B.deviation([2.0, 0.0], [5, 0]) == 1.0
    # dev 0.86 >= maxDev 0.85 is balanced (reading R15: "within 85% of the best")
    p, s = B.Params(), B.State()
    for _ in range(10):
        _, trig = B.step(p, s, [0.86, 1.0], [1, 1], [0.5, 0.5])
        assert not trig and s.lbt == 0.0


def test_proportional_converges_in_one_step():
    rates = [1.0, 1.0, 1.0, 0.5]                     # partition 3 runs at half speed
    L, g = 1 << 20, 256
    d = [0.25] * 4
    p, s = B.Params(), B.State()
    trig_at = None
    for run in range(8):
        off, ln = P.partition(L, g, d)
        t = [ln[i] / rates[i] for i in range(4)]    # linear cost model
        nd, trig = B.step(p, s, t, ln, d)
        if trig and trig_at is None:
            trig_at = run
        d = nd
    assert trig_at == 2
    _, ln = P.partition(L, g, d)
    want = [r / sum(rates) * L for r in rates]
    assert all(abs(ln[i] - want[i]) <= g for i in range(4))
    assert B.deviation([ln[i] / rates[i] for i in range(4)], ln) >= 0.85


def test_abs_doubling_rule():
    # three shifts in one direction at 0.05, the fourth uses 0.10
    p, s = B.Params(mode=B.ABS), B.State(active=1, abs_t=0.05)
    d = [0.1, 0.9]
    steps = []
    for _ in range(4):
        nd, trig = B.step(p, s, [1.0, 3.0], [1, 1], d)
        assert trig
        steps.append(round(nd[0] - d[0], 12))
        d = nd
    assert steps == [0.05, 0.05, 0.05, 0.10]
    # a reversal halves the step (binary-search refinement)
    nd, _ = B.step(p, s, [3.0, 1.0], [1, 1], d)
    assert round(d[0] - nd[0], 12) == 0.05


def test_abs_converges_two_classes():
    rate = [1.0, 3.0]
    d, p, s = [0.5, 0.5], B.Params(mode=B.ABS), B.State()
    for run in range(40):
        t = [d[0] / rate[0], d[1] / rate[1]]
        d, _ = B.step(p, s, t, [1 if d[0] > 0 else 0, 1 if d[1] > 0 else 0], d)
    t = [d[0] / rate[0], d[1] / rate[1]]
    assert B.deviation(t, [1, 1]) >= 0.85


# ----------------------------------------------------------------- FFT (NEXT-3)
from oracle import fft as FF  # noqa: E402


@pytest.mark.parametrize("N", [1, 2, 8, 64, 512, 4096])
def test_fft_chain_vs_brute_force_dft(N):
    """The oracle's library step agrees with the direct definition (sign of
    the exponent, 1/N on the inverse only, natural output order)."""
    x = synth.np_f32_um11(11, 0, 2 * N).reshape(N, 2)
    xc = FF.as_complex(x)
    assert xc[0] == complex(float(x[0, 0]), float(x[0, 1]))
    for d, inv in (("F", False), ("I", True)):
        got = FF.fft_chain(xc, d)
        want = FF.dft_brute(xc, inv)
        assert FF.rel_l2(got, want) < 1e-12 * max(1.0, math.log2(N))


def test_fft_closed_forms_at_65536():
    N = 1 << 16
    n = np.arange(N)
    # delta at n0 -> X[k] = exp(-2 pi i n0 k / N)  (exponent reduced mod N exactly)
    for n0 in (0, 1, 12345):
        d = np.zeros(N, np.complex128)
        d[n0] = 1.0
        want = np.exp(-2j * np.pi * ((n0 * n) % N) / N)
        assert np.max(np.abs(FF.fft_chain(d, "F") - want)) < 1e-11
    # pure tone m -> N delta_{k,m}; constant -> N delta_{k,0}
    m = 777
    tone = np.exp(2j * np.pi * ((m * n) % N) / N)
    X = FF.fft_chain(tone, "F")
    assert abs(X[m] - N) < 1e-7 and np.max(np.abs(np.delete(X, m))) < 1e-7
    X = FF.fft_chain(np.ones(N), "F")
    assert X[0] == N and np.max(np.abs(X[1:])) < 1e-9
    # inverse of a delta at k0 = (1/N) exp(+2 pi i k0 n / N)
    d = np.zeros(N, np.complex128)
    d[3] = 1.0
    assert np.max(np.abs(FF.fft_chain(d, "I") - np.exp(2j * np.pi * 3 * n / N) / N)) < 1e-16


def test_fft_invariants_batch():
    B, N = 3, 1 << 13
    x = FF.as_complex(synth.np_f32_um11(11, 0, 2 * B * N).reshape(B, N, 2))
    X = FF.fft_chain(x, "F")
    # Parseval: sum |X|^2 = N sum |x|^2, per transform of the batch
    assert np.allclose(np.sum(np.abs(X) ** 2, -1), N * np.sum(np.abs(x) ** 2, -1), rtol=1e-12)
    # round trip (the benchmark's pipeline(fft, ifft)) and its reverse
    assert np.max(FF.rel_l2(FF.fft_chain(x, "FI"), x)) < 1e-14
    assert np.max(FF.rel_l2(FF.fft_chain(x, "IF"), x)) < 1e-14
    # batch rows are independent: row 1 alone gives the same transform
    assert np.array_equal(FF.fft_chain(x[1], "F"), X[1])
    # shift theorem: x[(n - s) mod N] -> X[k] exp(-2 pi i s k / N)
    s = 100
    k = np.arange(N)
    Xs = FF.fft_chain(np.roll(x[0], s), "F")
    assert np.max(np.abs(Xs - X[0] * np.exp(-2j * np.pi * ((s * k) % N) / N))) < 1e-9
    # F F x = N x[-n mod N]
    FFx = FF.fft_chain(x[0], "FF")
    assert np.max(np.abs(FFx - N * x[0][(-k) % N])) < 1e-8
    # brute force on one full 8192-point row
    assert FF.rel_l2(X[2], FF.dft_brute(x[2])) < 1e-12


def test_fft_tolerance_formula():
    # Higham Thm 24.2 shape: grows with log2 N and the number of stages
    assert FF.tolerance(1 << 16, 1) < FF.tolerance(1 << 16, 2) < 2 * FF.tolerance(1 << 16, 1) + 1e-7
    assert FF.tolerance(1 << 13, 1) < FF.tolerance(1 << 16, 1) < 1e-5


def test_fft_tolerance_value_vs_higham_constants():
    """The VALUE of the bound, recomputed in 50-digit arithmetic from the
    constants of Higham (2002) Thm 24.2 as printed there: unit roundoff of
    binary32 u = 2^-24, gamma_n = n u / (1 - n u), computed weights with
    |w^ - w| <= mu, eta = mu + gamma_4 (sqrt 2 + mu), relative error of the
    radix-2 FFT <= log2(N) eta / (1 - log2(N) eta); R25 takes
    mu = 4u (a tabulated fp32 root times one complex product) and adds u for
    the final rounding to fp32 per chain."""
    import mpmath
    mpmath.mp.dps = 50
    u = mpmath.mpf(2) ** -24

    def gamma(n):
        return n * u / (1 - n * u)

    mu = 4 * u
    eta = mu + gamma(4) * (mpmath.sqrt(2) + mu)
    for log2n in (13, 14, 15, 16):
        per = log2n * eta / (1 - log2n * eta)
        for stages in (1, 2, 6):
            want = float(stages * per + u)
            assert abs(FF.tolerance(1 << log2n, stages) - want) <= 1e-12 * want
    # the number DESIGN.md R25 quotes: 9.3e-6 per stage at N = 65536
    assert 9.2e-6 < FF.tolerance(1 << 16, 1) < 9.3e-6


def test_fft_tolerance_bounds_a_real_fp32_fft():
    """The bound is a bound: an iterative radix-2 FFT carried out in complex64
    (numpy, every butterfly rounded to binary32, twiddles rounded to binary32)
    stays within tolerance(N, 1) of the fp64 transform, and the bound is not
    vacuous (within 200x of the observed worst error)."""
    rng = np.random.default_rng(7)
    for log2n in (8, 10, 12):
        N = 1 << log2n
        worst = 0.0
        for trial in range(4):
            x = (rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)).astype(np.complex64)
            # bit-reversal permutation, then log2n butterfly levels in complex64
            rev = np.array([int(format(i, f"0{log2n}b")[::-1], 2) for i in range(N)])
            y = x[rev].copy()
            h = 1
            while h < N:
                k = np.arange(h)
                w = np.exp(-2j * np.pi * k / (2 * h)).astype(np.complex64)
                y = y.reshape(-1, 2 * h)
                a, b = y[:, :h].copy(), (y[:, h:] * w).astype(np.complex64)
                y[:, :h], y[:, h:] = a + b, a - b
                y = y.reshape(N)
                h *= 2
            err = FF.rel_l2(y.astype(np.complex128), np.fft.fft(x.astype(np.complex128)))
            worst = max(worst, float(err))
        tol = FF.tolerance(N, 1)
        assert worst <= tol and tol <= 200 * worst, (N, worst, tol)


# ----------------------------------------------------------------- NEXT-4 variants
def test_merge_functions_pinned_to_exact_partials():
    """P:705-707 merging functions over per-partition partials (R26): each
    partial is pinned to math.fsum (exactly rounded), then merged in order."""
    n = 5 * (1 << 16) + 123
    x = synth.np_f32_um11(5, 0, n)
    y = synth.np_f32_um11(6, 0, n)
    lengths = [2 << 16, 0, 1 << 16, (2 << 16) + 123]
    xs = x.astype(np.float64)
    ex, ed, o = [], [], 0
    for ln in lengths:
        if ln:
            ex.append(math.fsum(xs[o:o + ln]))
            ed.append(math.fsum(xs[o:o + ln] * y[o:o + ln].astype(np.float64)))
        o += ln
    ident = sct.Leaf("map_identity")
    prod = sct.Leaf("map_product")
    for op, f in (("-", lambda a, b: a - b), ("*", lambda a, b: a * b), ("/", lambda a, b: a / b),
                  (lambda a, b: 2 * a + b, lambda a, b: 2 * a + b)):
        want_s, want_d = ex[0], ed[0]
        for a, b in zip(ex[1:], ed[1:]):
            want_s, want_d = f(want_s, a), f(want_d, b)
        got_s = sct.evaluate(sct.MapReduce(ident, op), (x,), lengths=lengths).reduced
        got_d = sct.evaluate(sct.MapReduce(prod, op), (x, y), lengths=lengths).reduced
        assert abs(got_s - want_s) <= 1e-12 * max(1.0, abs(want_s))
        assert abs(got_d - want_d) <= 1e-12 * max(1.0, abs(want_d))
    # '+' ignores the partitioning (the canonical sum)
    assert abs(sct.evaluate(sct.MapReduce(ident, "+"), (x,)).reduced - math.fsum(xs)) < 1e-9


def test_reduction_stage_extremes_pinned():
    """Device reduction stage MAX / MIN (NEXT-4, reading R28): the
    oracle's serial maxNum/minNum fold is pinned to (a) Python's built-in
    max/min over the terms as Python floats (fp64; fp32 x*y is exact there) on
    tiny inputs, (b) closed forms, (c) invariants: max = -min of the negated
    terms, the fold over a concatenation = the fold of the pieces' folds
    (any partitioning), NaN terms ignored, empty -> -inf / +inf."""
    rng = np.random.default_rng(28)
    for n in (1, 2, 7, 33):
        x = synth.np_f32_um11(5, 0, n)
        y = synth.np_f32_um11(6, 0, n)
        tx = [float(a) for a in x]
        td = [float(a) * float(b) for a, b in zip(x, y)]
        assert K.fold_extreme(x) == max(tx) and K.fold_extreme(x, is_min=True) == min(tx)
        assert K.fold_extreme(x, y) == max(td) and K.fold_extreme(x, y, True) == min(td)
    # closed forms: x_i = i - k over n elements; x*y with y = -x peaks at 0
    n, k = 1000, 377
    x = (np.arange(n) - k).astype(np.float32)
    assert K.fold_extreme(x) == n - 1 - k and K.fold_extreme(x, is_min=True) == -k
    assert K.fold_extreme(x, -x) == 0.0 and K.fold_extreme(x, -x, True) == -float(n - 1 - k) ** 2
    # exact product: (1 + 2^-23)^2 needs 47 bits, kept exactly in fp64
    a = np.array([1 + 2.0 ** -23], np.float32)
    assert K.fold_extreme(a, a) == (1 + 2.0 ** -23) ** 2 != float(np.float32(a[0] * a[0]))
    # invariants
    x = synth.np_f32_um11(5, 0, 5000)
    y = synth.np_f32_um11(6, 0, 5000)
    assert K.fold_extreme(x) == -K.fold_extreme(-x, is_min=True)
    cuts = np.sort(rng.integers(0, 5000, size=5))
    pieces = np.split(np.arange(5000), cuts)
    for is_min in (False, True):
        parts = [K.fold_extreme(x[p], y[p], is_min) for p in pieces]
        agg = min(parts) if is_min else max(parts)
        assert agg == K.fold_extreme(x, y, is_min)
    z = np.array([np.nan, -2.0, np.nan, 3.0], np.float32)
    assert K.fold_extreme(z) == 3.0 and K.fold_extreme(z, is_min=True) == -2.0
    assert K.fold_extreme(np.zeros(0, np.float32)) == -math.inf
    assert K.fold_extreme(np.zeros(0, np.float32), is_min=True) == math.inf
    # through the interpreter: reduce('sum') is the '+' fold
    ident, prod = sct.Leaf("map_identity"), sct.Leaf("map_product")
    assert sct.evaluate(sct.MapReduce(ident, sct.Leaf("reduce", {"op": "sum"})), (x,)).reduced == \
        sct.evaluate(sct.MapReduce(ident, "+"), (x,)).reduced
    assert sct.evaluate(sct.MapReduce(prod, sct.Leaf("reduce", {"op": "max"})), (x, y)).reduced == \
        max(float(a) * float(b) for a, b in zip(x, y))
    assert sct.kernel_execution_order(sct.MapReduce(prod, sct.Leaf("reduce", {"op": "min"})), []) == [0, 1]


def test_loop_host_reduces_to_loop_for():
    """a host condition that stops at k equals loop_for(body, k)."""
    img = synth.np_rgba(3, 0, 8 * 16).reshape(8, 16, 4)
    body = sct.Pipeline([sct.Leaf("gauss_noise", {"seed": 4, "scale": 8}),
                         sct.Leaf("mirror")])
    seen = []
    for k in (0, 1, 3):
        seen.clear()
        r = sct.evaluate(sct.LoopHost(body, 10, lambda i: (seen.append(i), i < k)[1]), img)
        want = sct.evaluate(sct.LoopFor(body, k), img).value
        assert np.array_equal(r.value, want) and r.executions == k and r.converged
        assert seen == list(range(k + 1))
    r = sct.evaluate(sct.LoopHost(body, 2, lambda i: True), img)
    assert r.executions == 2 and not r.converged
    assert sct.kernel_execution_order(sct.LoopHost(body, 9, None), [2]) == [0, 1, 0, 1]


# ----------------------------------------------------------------- composite map stage (general SCT composition)
def test_mapreduce_composite_map_stage_closed_forms():
    """map_reduce(pipeline(saxpy(a), map_product)): the map stage transforms
    (x, y) -> (x, fma(a, x, y)) before the terms x * y' are formed (P:162,
    P:191 map_reduce(SCT map_stage, ...)).  Pinned by closed forms that a
    wrong composition (terms from y instead of y', the reduction before the
    saxpy, a dropped fma) fails: a = 0 gives the pinned dot(x, y); y = 0 and
    a = 1 give sum x^2 exactly (fractions); a = 2, y = -x give y' = x exactly."""
    n = 3000
    x = synth.np_f32_um11(31, 0, n)
    y = synth.np_f32_um11(32, 0, n)
    comp = lambda a: sct.MapReduce(sct.Pipeline([sct.Leaf("saxpy", {"a": a}),   # noqa: E731
                                                 sct.Leaf("map_product")]), "+")
    assert sct.sig(comp(1.0)) == (sct.SAXPY, "scalar")
    assert sct.evaluate(comp(0.0), (x, y)).reduced == K.dot(x, y)
    sq = sum(Fraction(float(v)) ** 2 for v in x)
    z = np.zeros_like(x)
    assert abs(Fraction(sct.evaluate(comp(1.0), (x, z)).reduced) - sq) <= sq * Fraction(1, 2 ** 52)
    assert abs(Fraction(sct.evaluate(comp(2.0), (x, -x)).reduced) - sq) <= sq * Fraction(1, 2 ** 52)
    # and the composition is not the plain dot when a != 0
    assert sct.evaluate(comp(0.5), (x, y)).reduced != K.dot(x, y)


def test_interpreter_reports_while_executions_through_composites():
    """E (marrow.h out[2]) is the total of the while-loops' body executions
    anywhere in the tree: through a pipeline (Fig. 1 shape) it is D + 1 of the
    BFS depth (scipy-pinned hyst_bfs); a body of m steps changes iff one of its
    steps does, so E_m = floor((D - 1) / m) + 2; loop_for(while, 2) adds one
    more (an execution that changes nothing)."""
    gray = synth.np_u8_stream(8, 2, 120 * 150).reshape(120, 150)
    lab = K.segment(gray, 173, 250)
    _, D = K.hyst_bfs(lab)
    assert D >= 3
    step = sct.Leaf("hysteresis_step")
    fig1 = lambda body: sct.Pipeline([sct.Leaf("segment", {"lo": 173, "hi": 250}),   # noqa: E731
                                      sct.LoopWhileChanged(body, 1000), sct.Leaf("hysteresis_finalize")])
    assert sct.evaluate(fig1(step), gray).executions == D + 1
    for m in (2, 3):
        r = sct.evaluate(fig1(sct.Pipeline([step] * m)), gray)
        assert r.executions == (D - 1) // m + 2 and r.converged
        r2 = sct.evaluate(fig1(sct.LoopFor(step, m)), gray)
        assert r2.executions == r.executions and np.array_equal(r2.value, r.value)
    r = sct.evaluate(sct.LoopFor(sct.LoopWhileChanged(step, 1000), 2), lab)
    assert r.executions == D + 2


def test_reduction_stage_sct_closed_forms():
    """Reduction-stage SCT (NEXT-4): term maps before the fold, scalar
    maps after it.  Pins: the L2 norm of a +-1 vector is sqrt(n) exactly; the
    L1 fold equals abs_sum (pinned above); sum of squares against exact
    rational brute force; max |x| against a brute-force scan; mean = sum / n
    with the scale applied after the fold (not per term); abs o square =
    square."""
    def red(ops, op="sum"):
        tm = [sct.Leaf("term_map", {"map": t}) for t in ops[0]]
        sm = [sct.Leaf("scalar_map", {"map": k, "c": c}) for k, c in ops[1]]
        stages = tm + [sct.Leaf("reduce", {"op": op})] + sm
        return sct.MapReduce(sct.Leaf("map_identity"), stages[0] if len(stages) == 1 else sct.Pipeline(stages))
    rng = np.random.default_rng(5)
    n = 4097
    s = np.where(rng.integers(0, 2, n) == 1, 1.0, -1.0).astype(np.float32)
    assert sct.evaluate(red((["square"], [("sqrt", 0.0)])), s).reduced == math.sqrt(n)
    x = synth.np_f32_um11(33, 0, 2000)
    assert sct.evaluate(red((["abs"], [])), x).reduced == K.abs_sum(x)
    sq = sum(Fraction(float(v)) ** 2 for v in x)
    got = Fraction(sct.evaluate(red((["square"], [])), x).reduced)
    assert abs(got - sq) <= sq * Fraction(1, 2 ** 52)
    assert sct.evaluate(red((["abs"], []), "max"), x).reduced == max(abs(float(v)) for v in x)
    assert sct.evaluate(red(([], [("scale", 1.0 / 2000)])), x).reduced == K.sum_(x) * (1.0 / 2000)
    assert sct.evaluate(red((["abs", "square"], [])), x).reduced == sct.evaluate(red((["square"], [])), x).reduced
    assert sct.sig(red((["square"], [("sqrt", 0.0)]))) == (sct.VEC1, "scalar")
