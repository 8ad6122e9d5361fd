"""Locality-aware domain decomposition (ORACLE — test infrastructure only).

P:355-372 (§3.1 constraint display): every vector V communicated between
kernels is split into the same p partitions V^j with
    epu(V) mod nu(V,K) = 0,   #V^j mod (epu(V)/nu(V,K)) = 0,   #V^j mod wgs_j(K) = 0.
Reading R14/R5: the B200 kernels bound-check their tails, so
wgs = 1 and the hardware unit becomes an alignment granule `align`
(16 B vectors, one row, one slab, 256 bodies, one 2^16 reduction chunk).
The granule is the least g satisfying every divisibility: lcm of all
epu/nu and align ("granule").

Apportionment (reading R13, P:587-589 admits imbalance without a rule):
U = floor(L/g) granules; raw_i = d_i*U; base_i = floor(raw_i); the
U - sum(base) leftover granules go one each to the largest fractional
parts (Hamilton / largest remainder), ties to the larger d_i then the lower
index, only to partitions with d_i > 0.  The L mod g tail goes to the last
partition with d_i > 0 (documented deviation from P:368's divisibility,
needed for odd sizes).  Offsets are prefix sums (contiguous, rank order).
All arithmetic is IEEE fp64 exactly as written here.
"""
from __future__ import annotations

import math


class EpuNuError(ValueError):
    pass


class InvalidSpec(ValueError):
    pass


def granule(pairs, align: int = 1) -> int:
    """pairs: iterable of (epu, nu) for every kernel touching the vector."""
    g = int(align)
    if g < 1:
        raise InvalidSpec("align must be >= 1")
    for epu, nu in pairs:
        if epu < 1 or nu < 1:
            raise InvalidSpec("epu and nu must be >= 1")
        if epu % nu != 0:
            raise EpuNuError(f"epu {epu} mod nu {nu} != 0")
        g = g * (epu // nu) // math.gcd(g, epu // nu)
    return g


def check_distribution(d):
    if len(d) == 0:
        raise InvalidSpec("empty distribution")
    if any(not (x >= 0.0) for x in d):
        raise InvalidSpec("negative or NaN fraction")
    if not any(x > 0.0 for x in d):
        raise InvalidSpec("no positive fraction")
    s = 0.0
    for x in d:
        s += x
    if abs(s - 1.0) > 1e-9:
        raise InvalidSpec(f"fractions sum to {s}")


def partition(L: int, g: int, d, strict: bool = False):
    """Returns (offsets, lengths) in domain units for each partition."""
    check_distribution(d)
    k = len(d)
    U = L // g
    tail = L - U * g
    if strict and tail:
        raise InvalidSpec(f"infeasible partition: {L} mod {g} != 0")
    raw = [float(d[i]) * float(U) for i in range(k)]
    base = [math.floor(r) for r in raw]
    left = U - sum(base)
    cand = [i for i in range(k) if d[i] > 0.0]
    cand.sort(key=lambda i: (-(raw[i] - base[i]), -d[i], i))
    for j in range(left):
        base[cand[j % len(cand)]] += 1
    # sum(d) may exceed 1 by <= 1e-9: then take back from the smallest parts
    j = len(cand) - 1
    while left < 0:
        i = cand[j % len(cand)]
        if base[i] > 0:
            base[i] -= 1
            left += 1
        j -= 1
    lengths = [b * g for b in base]
    last = max(i for i in range(k) if d[i] > 0.0)
    lengths[last] += tail
    offsets, acc = [], 0
    for n in lengths:
        offsets.append(acc)
        acc += n
    assert acc == L
    return offsets, lengths
