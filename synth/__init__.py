"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the SplitMix64 counter generator
and the per-workload input recipes (SURVEY.md §8(d)
d.0/d.1).  Three implementations of the same streams:

* ``np_*``      — numpy, for tiny inputs and as a cross-check of the C one;
* ``host_*``    — plain C (``libsynth_host.so``), for large host inputs;
* ``dev_*``     — CUDA (``libsynth_dev.so``), fills device memory for a rank's
                  own slice (keyed by the global element index).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# Seeds and parameters of the configs.
SEED_SAXPY_X, SEED_SAXPY_Y = 1, 2
SEED_IMAGE, SEED_NOISE = 3, 4
SEED_MR_X, SEED_MR_Y = 5, 6
SEED_SEGMENT = 7
SEED_HYST = 8
SEED_NBODY = 9
SEED_NBODY_SAMPLES = 10


# --------------------------------------------------------------------------- numpy
def np_splitmix64(seed: int, idx) -> np.ndarray:
    """SplitMix64 outputs z_i for the given indices (uint64 wraparound)."""
    with np.errstate(over="ignore"):
        i = np.asarray(idx, dtype=np.uint64)
        z = np.uint64(seed) + (i + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def np_f32_um11(seed: int, start: int, count: int) -> np.ndarray:
    z = np_splitmix64(seed, np.arange(start, start + count, dtype=np.uint64))
    return ((z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23)
            - np.float32(1.0)).astype(np.float32)


def np_f32_u01(seed: int, start: int, count: int) -> np.ndarray:
    z = np_splitmix64(seed, np.arange(start, start + count, dtype=np.uint64))
    return ((z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def np_u8_stream(seed: int, start: int, count: int) -> np.ndarray:
    v = np.arange(start, start + count, dtype=np.uint64)
    z = np_splitmix64(seed, v >> np.uint64(3))
    return ((z >> (np.uint64(8) * (v & np.uint64(7)))) & np.uint64(0xFF)).astype(np.uint8)


def np_rgba(seed: int, start_px: int, count: int) -> np.ndarray:
    z = np_splitmix64(seed, np.arange(start_px, start_px + count, dtype=np.uint64))
    out = np.empty((count, 4), dtype=np.uint8)
    for c in range(3):
        out[:, c] = ((z >> np.uint64(8 * c)) & np.uint64(0xFF)).astype(np.uint8)
    out[:, 3] = 255
    return out


def np_nbody(seed: int, start: int, count: int, mass: float):
    b = np.arange(start, start + count, dtype=np.uint64)
    pos = np.empty((count, 4), dtype=np.float32)
    for c in range(3):
        z = np_splitmix64(seed, np.uint64(3) * b + np.uint64(c))
        pos[:, c] = (z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
    pos[:, 3] = np.float32(mass)
    return pos, np.zeros((count, 4), dtype=np.float32)


def nbody_sample_indices(n_bodies: int, count: int = 2048) -> np.ndarray:
    """Pinned N-body parity sample: SplitMix64(seed 10, k) mod N."""
    return (np_splitmix64(SEED_NBODY_SAMPLES, np.arange(count, dtype=np.uint64))
            % np.uint64(n_bodies)).astype(np.int64)


# --------------------------------------------------------------------------- C host
_host = None
_dev = None


def _load(name):
    path = os.path.join(_HERE, name)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run __graft_entry__.build() first")
    return ctypes.CDLL(path)


def host_lib():
    global _host
    if _host is None:
        lib = _load("libsynth_host.so")
        u64, vp = ctypes.c_uint64, ctypes.c_void_p
        lib.synth_splitmix64.restype = u64
        lib.synth_splitmix64.argtypes = [u64, u64]
        for fn in ("synth_u64", "synth_f32_um11", "synth_f32_u01", "synth_u8_stream", "synth_rgba"):
            getattr(lib, fn).argtypes = [u64, u64, u64, vp]
            getattr(lib, fn).restype = None
        lib.synth_nbody.argtypes = [u64, u64, u64, ctypes.c_float, vp, vp]
        lib.synth_nbody.restype = None
        _host = lib
    return _host


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def host_f32_um11(seed, start, count):
    out = np.empty(count, dtype=np.float32)
    host_lib().synth_f32_um11(seed, start, count, _ptr(out))
    return out


def host_f32_u01(seed, start, count):
    out = np.empty(count, dtype=np.float32)
    host_lib().synth_f32_u01(seed, start, count, _ptr(out))
    return out


def host_u8_stream(seed, start, count):
    out = np.empty(count, dtype=np.uint8)
    host_lib().synth_u8_stream(seed, start, count, _ptr(out))
    return out


def host_rgba(seed, start_px, count):
    out = np.empty((count, 4), dtype=np.uint8)
    host_lib().synth_rgba(seed, start_px, count, _ptr(out))
    return out


def host_nbody(seed, start, count, mass):
    pos = np.empty((count, 4), dtype=np.float32)
    vel = np.empty((count, 4), dtype=np.float32)
    host_lib().synth_nbody(seed, start, count, ctypes.c_float(mass), _ptr(pos), _ptr(vel))
    return pos, vel


# --------------------------------------------------------------------------- device
def dev_lib():
    global _dev
    if _dev is None:
        lib = _load("libsynth_dev.so")
        u64, vp = ctypes.c_uint64, ctypes.c_void_p
        for fn in ("synth_dev_f32_um11", "synth_dev_f32_u01", "synth_dev_u8_stream", "synth_dev_rgba"):
            getattr(lib, fn).argtypes = [u64, u64, u64, vp, vp]
            getattr(lib, fn).restype = ctypes.c_int
        lib.synth_dev_nbody.argtypes = [u64, u64, u64, ctypes.c_float, vp, vp, vp]
        lib.synth_dev_nbody.restype = ctypes.c_int
        _dev = lib
    return _dev


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with cudaError {rc}")


def dev_fill_f32_um11(t, seed, start, stream=None):
    _check(dev_lib().synth_dev_f32_um11(seed, start, t.numel(), ctypes.c_void_p(t.data_ptr()),
                                        _stream_ptr(stream)), "synth_dev_f32_um11")


def dev_fill_f32_u01(t, seed, start, stream=None):
    _check(dev_lib().synth_dev_f32_u01(seed, start, t.numel(), ctypes.c_void_p(t.data_ptr()),
                                       _stream_ptr(stream)), "synth_dev_f32_u01")


def dev_fill_u8_stream(t, seed, start, stream=None):
    _check(dev_lib().synth_dev_u8_stream(seed, start, t.numel(), ctypes.c_void_p(t.data_ptr()),
                                         _stream_ptr(stream)), "synth_dev_u8_stream")


def dev_fill_rgba(t, seed, start_px, stream=None):
    assert t.numel() % 4 == 0
    _check(dev_lib().synth_dev_rgba(seed, start_px, t.numel() // 4, ctypes.c_void_p(t.data_ptr()),
                                    _stream_ptr(stream)), "synth_dev_rgba")


def dev_fill_nbody(pos, vel, seed, start, mass, stream=None):
    _check(dev_lib().synth_dev_nbody(seed, start, pos.numel() // 4, ctypes.c_float(mass),
                                     ctypes.c_void_p(pos.data_ptr()),
                                     ctypes.c_void_p(vel.data_ptr()) if vel is not None else None,
                                     _stream_ptr(stream)), "synth_dev_nbody")
