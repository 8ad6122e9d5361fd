"""THE ORACLE — test infrastructure only.

A plain, slow, obviously correct CPU implementation of what the hot path
computes (arxiv 1510.06585, Marrow).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import it.
It shares no code with the CUDA path (``paper_1510_06585_b200``) and never
imports it; the two meet only through the seeded inputs of ``synth``.

Modules:
  kernels   — ctypes binding of oracle.c (fp64 / exact integer built-in kernels)
  sct       — recursive skeleton-tree interpreter (depth-first, one partition)
  partition — granule / largest-remainder partitioner (integer)
  balance   — lbt monitor, proportional re-derivation, Adaptive Binary Search
  brute     — pure-Python brute force of the kernels for tiny inputs
  fft       — FFT / inverse FFT pipeline (NEXT-3) in fp64 with its tolerance

"parity unpinned": fidelity of the noise / solarize / segmentation / N-body
*definitions* to the paper's own (unpublished) OpenCL kernels.  Everything
else is pinned in tests/test_oracle_pins.py; see DESIGN.md §Oracle.
"""
