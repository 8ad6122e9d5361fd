"""ORACLE (test infrastructure only) — the FFT workload (NEXT-3).

PAPER.md P:729-732 (§4 Benchmarks): "FFT is a set of Fast-Fourier
Transformations adapted from the SHOC Benchmark Suite, where FFT is
pipelined with its inversion.  The elementary partitioning unit is the size
of each FFT which is 512 KBytes."  Readings (R23-R25): one FFT is
N = 65536 complex single-precision points (512 KiB, interleaved re/im), a
batch of B such FFTs is partitioned by whole FFTs, the pipeline is
pipeline(fft, ifft), and the inverse carries the 1/N factor:

    forward  X[k] = sum_n x[n] exp(-2 pi i n k / N)
    inverse  x[n] = (1/N) sum_k X[k] exp(+2 pi i n k / N)

The method reaches these plain definitions up to rounding, so the oracle is
the definition evaluated in fp64 with a library FFT as the step (numpy's
pocketfft); tests/test_oracle_pins.py pins it against a brute-force DFT and
closed forms, independently of that library.
"""
from __future__ import annotations

import numpy as np


def as_complex(a: np.ndarray) -> np.ndarray:
    """float32 [..., N, 2] (re, im) -> complex128 [..., N], exact."""
    a = np.asarray(a)
    return a[..., 0].astype(np.float64) + 1j * a[..., 1].astype(np.float64)


def fft_chain(x: np.ndarray, dirs) -> np.ndarray:
    """Apply the FFT leaves of a pipeline in order (the output of
    stage i is the input of stage i+1) along the last axis.  dirs: sequence
    of 'F' (forward) / 'I' (inverse, with 1/N).  Returns complex128."""
    y = np.asarray(x, dtype=np.complex128)
    for d in dirs:
        if d == "F":
            y = np.fft.fft(y, axis=-1)
        elif d == "I":
            y = np.fft.ifft(y, axis=-1)   # includes the 1/N factor
        else:
            raise ValueError(d)
    return y


def dft_brute(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Direct O(N^2) DFT of one vector (pin only): exponent n*k reduced mod N
    in integers before the angle is formed, rows in blocks."""
    x = np.asarray(x, dtype=np.complex128)
    N = x.shape[-1]
    n = np.arange(N, dtype=np.int64)
    out = np.empty(N, np.complex128)
    sgn = 1.0 if inverse else -1.0
    for k0 in range(0, N, 256):
        k = np.arange(k0, min(N, k0 + 256), dtype=np.int64)
        e = (k[:, None] * n[None, :]) % N
        w = np.exp(sgn * 2j * np.pi * e / N)
        out[k0:k0 + len(k)] = w @ x
    return out / N if inverse else out


def rel_l2(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Per-transform relative L2 error ||got - want|| / ||want|| (last axis)."""
    num = np.sqrt(np.sum(np.abs(got - want) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(want) ** 2, axis=-1))
    return num / np.maximum(den, np.finfo(np.float64).tiny)


def tolerance(N: int, stages: int) -> float:
    """Bound on rel_l2 for an fp32 radix-2 (Cooley-Tukey / Stockham) FFT
    chain (Higham, Accuracy and Stability of Numerical Algorithms, Thm 24.2):
    log2(N) eta / (1 - log2(N) eta) per transform, eta = mu + gamma_4 (sqrt2
    + mu), u = 2^-24, twiddle error mu <= 4u (a tabulated fp32 root, one
    complex product), plus the final rounding to fp32 (u).  DESIGN.md R25."""
    u = 2.0 ** -24
    mu = 4 * u
    g4 = 4 * u / (1 - 4 * u)
    eta = mu + g4 * (np.sqrt(2.0) + mu)
    L = np.log2(N)
    per = L * eta / (1 - L * eta)
    return stages * per + u
