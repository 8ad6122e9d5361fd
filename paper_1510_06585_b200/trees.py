"""The benchmark skeleton trees of the paper (§4) and of
BASELINE.json, built bottom-up from libmarrow's built-in kernels."""
from __future__ import annotations

from . import marrow as M

# Defaults (R1, R2, R6, R11, R12)
NOISE_SEED, NOISE_SCALE, SOLARIZE_T = 4, 8, 128
SEG_LO, SEG_HI = 85, 170
HYST_LO, HYST_HI = 173, 250
NBODY_DT, NBODY_EPS2 = 1e-3, 1e-4
SAXPY_A = 2.5


def saxpy(a=SAXPY_A):
    """map(saxpy) — P:740-742."""
    return M.mw_map(M.mw_kernel_saxpy(a))


def filter_pipeline(seed=NOISE_SEED, scale=NOISE_SCALE, threshold=SOLARIZE_T):
    """pipeline(gaussian noise, solarize, mirror) — P:725-728."""
    return M.mw_pipeline([M.mw_kernel_gauss_noise(seed, scale), M.mw_kernel_solarize(threshold),
                          M.mw_kernel_mirror()])


def segmentation(lo=SEG_LO, hi=SEG_HI):
    """map(segmentation) — P:743."""
    return M.mw_map(M.mw_kernel_segment(lo, hi))


def mapreduce(dot=True):
    """map_reduce(map stage, +) — P:165."""
    m = M.mw_kernel_map_product() if dot else M.mw_kernel_map_identity()
    return M.mw_map_reduce(m, M.MW_MERGE_ADD)


def mapreduce_sct(op, dot=True):
    """map_reduce(map stage, reduce(op)) with a device reduction stage
    (NEXT-4): op = M.MW_REDUCE_SUM / MAX / MIN."""
    m = M.mw_kernel_map_product() if dot else M.mw_kernel_map_identity()
    return M.mw_map_reduce_sct(m, M.mw_kernel_reduce(op))


def hysteresis(lo=HYST_LO, hi=HYST_HI, max_iters=10000, check_every=1):
    """pipeline(threshold, loop(step), finalize) — the Fig. 1 shape."""
    return M.mw_pipeline([M.mw_kernel_segment(lo, hi),
                          M.mw_loop_while_changed(M.mw_kernel_hysteresis_step(), max_iters,
                                                  check_every),
                          M.mw_kernel_hysteresis_finalize()])


def nbody(steps, dt=NBODY_DT, eps2=NBODY_EPS2):
    """loop(nbody step, steps) with COPY positions — P:734-737."""
    return M.mw_loop_for(M.mw_kernel_nbody_step(dt, eps2), steps)


def fft_pipeline(log2n=16):
    """The FFT benchmark: "FFT is pipelined with its inversion";
    pipeline(fft, ifft) over a batch of 2^log2n-point complex64 transforms
    (512 KiB each at log2n = 16, reading R23)."""
    return M.mw_pipeline([M.mw_kernel_fft(log2n, False), M.mw_kernel_fft(log2n, True)])
