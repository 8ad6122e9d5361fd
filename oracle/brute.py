"""Pure-Python brute force for tiny inputs (ORACLE — test infrastructure only).

Independent second implementation of the definitions in oracle.c, written
with Python integers / fractions and no numpy arithmetic, so that the tests
can pin the C oracle against it on tiny inputs (exact rationals for sums,
literal neighbour loops for the stencil, bit loops for the hash).
"""
from __future__ import annotations

import struct
from fractions import Fraction

M32 = 0xFFFFFFFF


def lowbias32(v: int) -> int:
    v &= M32
    v ^= v >> 16
    v = (v * 0x7FEB352D) & M32
    v ^= v >> 15
    v = (v * 0x846CA68B) & M32
    v ^= v >> 16
    return v


def popcount(v: int) -> int:
    return bin(v).count("1")


def noise_pixel(px, idx: int, seed: int, S: int):
    K = lowbias32(seed ^ 0x9E3779B9)
    h = lowbias32(idx ^ K)
    out = []
    for c in range(3):
        n = (popcount((h >> (10 * c)) & 0x3FF) - 5) * S
        out.append(min(255, max(0, px[c] + n)))
    out.append(px[3])
    return tuple(out)


def solarize_pixel(px, T: int):
    return tuple([(255 - v if v >= T else v) for v in px[:3]] + [px[3]])


def filter_pipeline(img, seed, S, T):
    """img: list of rows of RGBA tuples.  noise -> solarize -> mirror."""
    H, W = len(img), len(img[0])
    out = []
    for y in range(H):
        row = []
        for x in range(W):
            xs = W - 1 - x
            row.append(solarize_pixel(noise_pixel(img[y][xs], y * W + xs, seed, S), T))
        out.append(row)
    return out


def segment_value(v: int, lo: int, hi: int) -> int:
    return 0 if v < lo else (128 if v < hi else 255)


def hyst_step(L):
    H, W = len(L), len(L[0])
    out = [list(r) for r in L]
    changed = False
    for y in range(H):
        for x in range(W):
            if L[y][x] != 128:
                continue
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if (dy or dx) and 0 <= y + dy < H and 0 <= x + dx < W and L[y + dy][x + dx] == 255:
                        out[y][x] = 255
            changed |= out[y][x] != L[y][x]
    return out, changed


def f32(v: float) -> float:
    return struct.unpack("<f", struct.pack("<f", v))[0]


def exact_sum(xs) -> Fraction:
    return sum((Fraction(float(v)) for v in xs), Fraction(0))


def exact_dot(xs, ys) -> Fraction:
    return sum((Fraction(float(a)) * Fraction(float(b)) for a, b in zip(xs, ys)), Fraction(0))


def round_f32(q: Fraction) -> float:
    """Round an exact rational once to binary32, round-half-even (finite range)."""
    if q == 0:
        return 0.0
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    quantum = Fraction(2) ** (max(e, -126) - 23)
    m = a / quantum
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * float(fl * quantum)


def saxpy_exact(a, x, y):
    """Correctly rounded binary32 of the exact a*x + y (one rounding)."""
    A = Fraction(float(a))
    return [round_f32(A * Fraction(float(xi)) + Fraction(float(yi))) for xi, yi in zip(x, y)]
