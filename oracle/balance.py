"""Dynamic load balancing (ORACLE — test infrastructure only).

P:610-638 (§3.3 "Dynamic Load Balancing"):
    lbt(n) = isUnbalanced(dev) * weight + lbt(n-1) * (1 - weight)
with default weight 2/3 and a trigger when lbt(n) ~ 1.
Readings (R15-R17):
  * dev = min_i t_i / max_i t_i over partitions with work; a run is
    unbalanced iff dev / cFactor < maxDev (the P:624 inequality read
    literally contradicts §4's "within 80% to 85% of the best");
  * lbt(0) = 0, "~1" means lbt >= 0.95 (exactly the 3rd consecutive
    unbalanced run triggers: 0.667, 0.889, 0.963);
  * PROPORTIONAL (default for identical GPUs, P:388's "relative
    performance" rule fed with measured rates): r_i = len_i / t_i,
    d_i' = r_i / sum(r), zero-work partitions stay 0; one shot, lbt <- 0;
  * ABS (Adaptive Binary Search, two device classes = two
    partitions): on trigger an episode starts and takes one step per run
    until a balanced run ends it (lbt <- 0, state reset).  Step: move
    `transferable` (initially 1/8) of the domain from the slower to the
    faster partition; a reversal of direction halves it (binary search);
    when more than 2 moves were already made in the same direction it
    doubles first (the interval "shifts sideways" and grows),
    capped at 1; the share is clamped to [0, 1].
All arithmetic is IEEE fp64, in exactly this order.
"""
from __future__ import annotations

from dataclasses import dataclass

PROPORTIONAL, ABS = 0, 1


@dataclass
class Params:
    weight: float = 2.0 / 3.0
    max_dev: float = 0.85
    c_factor: float = 1.0
    trigger: float = 0.95
    mode: int = PROPORTIONAL


@dataclass
class State:
    lbt: float = 0.0
    active: int = 0
    abs_t: float = 0.0
    abs_last_dir: int = 0
    abs_count: int = 0
    runs: int = 0


def deviation(times, lens) -> float:
    act = [float(t) for t, n in zip(times, lens) if n > 0]
    if len(act) <= 1:
        return 1.0
    hi = max(act)
    if hi <= 0.0:
        return 1.0
    return min(act) / hi


def lbt_update(prev: float, unbalanced: int, weight: float) -> float:
    return float(unbalanced) * weight + prev * (1.0 - weight)


def step(p: Params, s: State, times, lens, cur):
    """One monitoring step after a run.  Returns (next_distribution, triggered)."""
    k = len(cur)
    dev = deviation(times, lens)
    unb = 1 if dev / p.c_factor < p.max_dev else 0
    s.lbt = lbt_update(s.lbt, unb, p.weight)
    s.runs += 1
    nxt = [float(c) for c in cur]
    if s.active and not unb:           # a balanced run ends an ABS episode
        s.active, s.lbt = 0, 0.0
        s.abs_t, s.abs_last_dir, s.abs_count = 0.0, 0, 0
        return nxt, False
    if not s.active and s.lbt < p.trigger:
        return nxt, False
    if p.mode == PROPORTIONAL:
        r = [0.0] * k
        tot = 0.0
        for i in range(k):
            if lens[i] > 0:
                t = float(times[i])
                r[i] = float(lens[i]) / (t if t > 0.0 else 1e-30)
                tot += r[i]
        nxt = [r[i] / tot for i in range(k)]
        s.lbt = 0.0
        return nxt, True
    # ABS, two classes
    if k != 2:
        raise ValueError("ABS mode needs exactly two partitions")
    s.active = 1
    d = 1 if float(times[0]) < float(times[1]) else -1   # toward the faster one
    if s.abs_t == 0.0:
        s.abs_t = 0.125
    if d == s.abs_last_dir:
        if s.abs_count > 2:
            s.abs_t = min(2.0 * s.abs_t, 1.0)
            s.abs_count = 0
        s.abs_count += 1
    else:
        if s.abs_last_dir != 0:
            s.abs_t = s.abs_t / 2.0
        s.abs_count = 1
    s.abs_last_dir = d
    s0 = float(cur[0]) + float(d) * s.abs_t
    s0 = 0.0 if s0 < 0.0 else (1.0 if s0 > 1.0 else s0)
    s.lbt = 0.0
    return [s0, 1.0 - s0], True
