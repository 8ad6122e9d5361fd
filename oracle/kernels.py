"""ctypes binding of oracle.c (ORACLE — test infrastructure only).

Each wrapper takes/returns numpy arrays; the arithmetic is in oracle.c, whose
functions cite the paper passage they follow.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() first")
        L = ctypes.CDLL(path)
        i64, vp, f32, f64, u32, i32 = (ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                       ctypes.c_double, ctypes.c_uint32, ctypes.c_int32)
        sig = {
            "orc_saxpy": (None, [i64, f32, vp, vp]),
            "orc_lowbias32": (u32, [u32]),
            "orc_gauss_noise": (None, [i64, i64, vp, vp, u32, i32, i64]),
            "orc_fold_chunk": (None, [i64, vp, vp, vp]),
            "orc_solarize": (None, [i64, vp, vp, i32]),
            "orc_mirror": (None, [i64, i64, vp, vp]),
            "orc_segment": (None, [i64, vp, vp, i32, i32]),
            "orc_hyst_step": (ctypes.c_int, [i64, i64, vp, vp]),
            "orc_hyst_finalize": (None, [i64, vp, vp]),
            "orc_hyst_bfs": (i64, [i64, i64, vp, vp, i64]),
            "orc_nbody_accel": (None, [i64, vp, f32, i64, vp, vp, vp]),
            "orc_nbody_step": (None, [i64, vp, vp, f32, f32, vp, vp, vp]),
            "orc_sum": (f64, [i64, vp]),
            "orc_dot": (f64, [i64, vp, vp]),
            "orc_abs_sum": (f64, [i64, vp, vp]),
            "orc_fold_extreme": (f64, [i64, vp, vp, i32]),
            "orc_sum_f64": (f64, [i64, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def saxpy(a: float, x, y):
    x = _c(x, np.float32)
    y = _c(y, np.float32).copy()
    lib().orc_saxpy(x.size, ctypes.c_float(a), _p(x), _p(y))
    return y


def lowbias32(v: int) -> int:
    return int(lib().orc_lowbias32(v & 0xFFFFFFFF))


def gauss_noise(img, seed: int, S: int, y0: int = 0):
    """y0 = global row of img[0] (Offset trait); 0 for a whole image."""
    img = _c(img, np.uint8)
    H, W = img.shape[0], img.shape[1]
    out = np.empty_like(img)
    lib().orc_gauss_noise(H, W, _p(img), _p(out), seed & 0xFFFFFFFF, S, y0)
    return out


def solarize(img, T: int):
    img = _c(img, np.uint8)
    out = np.empty_like(img)
    lib().orc_solarize(img.size // 4, _p(img), _p(out), T)
    return out


def mirror(img):
    img = _c(img, np.uint8)
    out = np.empty_like(img)
    lib().orc_mirror(img.shape[0], img.shape[1], _p(img), _p(out))
    return out


def segment(a, lo: int, hi: int):
    a = _c(a, np.uint8)
    out = np.empty_like(a)
    lib().orc_segment(a.size, _p(a), _p(out), lo, hi)
    return out


def hyst_step(L):
    L = _c(L, np.uint8)
    out = np.empty_like(L)
    changed = lib().orc_hyst_step(L.shape[0], L.shape[1], _p(L), _p(out))
    return out, bool(changed)


def hyst_finalize(L):
    L = _c(L, np.uint8)
    out = np.empty_like(L)
    lib().orc_hyst_finalize(L.size, _p(L), _p(out))
    return out


def hyst_bfs(L, max_level: int = -1):
    """Returns (labels after promoting BFS levels <= max_level, D)."""
    L = _c(L, np.uint8)
    out = np.empty_like(L)
    D = lib().orc_hyst_bfs(L.shape[0], L.shape[1], _p(L), _p(out), max_level)
    if D < 0:
        raise MemoryError("orc_hyst_bfs allocation failed")
    return out, int(D)


def nbody_accel(pos4, eps2: float, targets=None):
    """fp64 accelerations (nt,3) and conditioning sums C_i (nt,)."""
    pos4 = _c(pos4, np.float32)
    N = pos4.shape[0]
    if targets is None:
        nt, tp = N, None
    else:
        targets = _c(targets, np.int64)
        nt, tp = targets.size, targets
    acc = np.empty((nt, 3), dtype=np.float64)
    cond = np.empty(nt, dtype=np.float64)
    lib().orc_nbody_accel(N, _p(pos4), ctypes.c_float(eps2), nt, _p(tp), _p(acc), _p(cond))
    return acc, cond


def nbody_step(pos4, vel4, eps2: float, dt: float):
    pos4 = _c(pos4, np.float32)
    vel4 = _c(vel4, np.float32)
    N = pos4.shape[0]
    po, vo = np.empty_like(pos4), np.empty_like(vel4)
    acc = np.empty((N, 3), dtype=np.float64)
    lib().orc_nbody_step(N, _p(pos4), _p(vel4), ctypes.c_float(eps2), ctypes.c_float(dt),
                         _p(po), _p(vo), _p(acc))
    return po, vo, acc


def sum_(x):
    x = _c(x, np.float32)
    return float(lib().orc_sum(x.size, _p(x)))


def dot(x, y):
    x, y = _c(x, np.float32), _c(y, np.float32)
    assert x.size == y.size
    return float(lib().orc_dot(x.size, _p(x), _p(y)))


class Fold:
    """Serial Neumaier fold continued across chunks (== one fold over all)."""

    def __init__(self):
        self.sc = np.zeros(2, dtype=np.float64)

    def add(self, x, y=None):
        x = _c(x, np.float32)
        if y is not None:
            y = _c(y, np.float32)
            assert y.size == x.size
        lib().orc_fold_chunk(x.size, _p(x), _p(y), _p(self.sc))
        return self

    @property
    def value(self) -> float:
        return float(self.sc[0] + self.sc[1])


def fold_extreme(x, y=None, is_min=False):
    """Reduction stage MAX / MIN (NEXT-4, R28): serial fold of the terms x
    (or x*y, exact in fp64) with maxNum / minNum; empty -> -inf / +inf."""
    x = _c(x, np.float32)
    if y is not None:
        y = _c(y, np.float32)
        assert y.size == x.size
    return float(lib().orc_fold_extreme(x.size, _p(x), _p(y), int(bool(is_min))))


def abs_sum(x, y=None):
    x = _c(x, np.float32)
    if y is not None:
        y = _c(y, np.float32)
    return float(lib().orc_abs_sum(x.size, _p(x), _p(y)))


def sum_f64(t):
    """Serial Neumaier fold of fp64 terms (reduction stage with term maps)."""
    t = _c(t, np.float64)
    return float(lib().orc_sum_f64(t.size, _p(t)))
