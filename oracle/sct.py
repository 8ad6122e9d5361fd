"""Skeleton computation tree interpreter (ORACLE — test infrastructure only).

The plain definition the method must reproduce is the *sequential,
single-device, depth-first evaluation of the tree over the whole domain as
one partition* (§2 "executed sequentially, according to a
depth-first evaluation of the tree"; §3.1 SPMD model: each
partition runs the SCT "according to the single device execution model").
So the oracle never splits: Map's independence is what makes the
method's splitting legal, and the tests check the method against this
unsplit evaluation.

Node semantics (DESIGN.md "Readings" R9, R10, R16):
  Leaf(kind, **params)        a built-in kernel (oracle.kernels)
  Pipeline(s1..sn)            s1, ..., sn in order; output of s_i is the input
                              of s_{i+1}
  Map(t)                      t over the whole domain
  MapReduce(m, '+')           m per element, then a serial left fold in
                              Neumaier-compensated fp64
  MapReduce(m, Leaf('reduce', op=...))  the reduction stage is an SCT
                              (NEXT-4, R28): 'sum' = the '+' fold,
                              'max' / 'min' = serial maxNum / minNum fold
  LoopFor(b, n)               state_{k+1} = b(state_k), k < n
  LoopWhileChanged(b, max)    condition before each iteration; stop when the
                              body changed nothing or max executions reached
                              (P:221-224); reports executions E
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import fft as FF
from . import kernels as K

# value kinds flowing along tree edges
SAXPY, RGBA, U8, U8_2D, NBODY, VEC1, VEC2, TERMS, ACCEL, TRAITS, CPLX = (
    "saxpy", "rgba", "u8", "u8_2d", "nbody", "vec1", "vec2", "terms", "accel", "traits", "cplx")

# leaf kind -> (input value kind, output value kind)
LEAF_SIG = {
    "saxpy": (SAXPY, SAXPY),
    "gauss_noise": (RGBA, RGBA),
    "solarize": (RGBA, RGBA),
    "mirror": (RGBA, RGBA),
    "segment": (U8, U8),
    "hysteresis_finalize": (U8, U8),
    "hysteresis_step": (U8_2D, U8_2D),
    "nbody_step": (NBODY, NBODY),
    "nbody_accel": (NBODY, ACCEL),
    "map_identity": (VEC1, TERMS),
    "map_product": (VEC2, TERMS),
    "debug_traits": (TRAITS, TRAITS),
    "fft": (CPLX, CPLX),
    "reduce": (TERMS, "scalar"),
    "term_map": (TERMS, TERMS),        # reduction-stage SCT: |t| or t*t before the fold
    "scalar_map": ("scalar", "scalar"),  # reduction-stage SCT: sqrt or scale of the result
}


class Node:
    pass


@dataclass
class Leaf(Node):
    kind: str
    params: dict = field(default_factory=dict)


@dataclass
class Pipeline(Node):
    stages: list

    def __post_init__(self):
        if len(self.stages) < 2:
            raise ValueError("Pipeline needs >= 2 stages (SPEC S:68)")


@dataclass
class Map(Node):
    tree: Node


@dataclass
class MapReduce(Node):
    """op: '+' (the canonical sum of all terms) or, NEXT-4 (P:705-707,
    DESIGN.md R26), '-', '*', '/' or a callable fn(acc, partial): the
    per-partition partial results r_p (partitions with work, global order)
    merged left to right — evaluate() then needs the partition lengths."""
    map_stage: Node
    op: object = "+"


@dataclass
class LoopFor(Node):
    body: Node
    n: int


@dataclass
class LoopWhileChanged(Node):
    body: Node
    max_iters: int


@dataclass
class LoopHost(Node):
    """NEXT-4 (P:374-378 stages 1 and 3 on the host, R27): before iteration i
    cond(i) is evaluated on the host; False ends the loop."""
    body: Node
    max_iters: int
    cond: object = None


@dataclass
class Result:
    value: object
    changed: bool = False          # did the last body change anything
    executions: int = 0            # while-loop body executions (E)
    converged: bool = True
    reduced: float | None = None   # MapReduce fp64 result


def _compat(a, b):
    # a saxpy value is the pair (x, y) of fp32 vectors: what map_product takes
    return a == b or {a, b} == {U8, U8_2D} or {a, b} == {SAXPY, VEC2}


def sig(node: Node):
    """(input kind, output kind) of a tree; raises ValueError if ill-typed."""
    if isinstance(node, Leaf):
        return LEAF_SIG[node.kind]
    if isinstance(node, Pipeline):
        sigs = [sig(s) for s in node.stages]
        for (_, o), (i, _) in zip(sigs, sigs[1:]):
            if not _compat(o, i):
                raise ValueError(f"pipeline stage kinds do not chain: {o} -> {i}")
        return sigs[0][0], sigs[-1][1]
    if isinstance(node, Map):
        return sig(node.tree)
    if isinstance(node, MapReduce):
        i, o = sig(node.map_stage)
        if o != TERMS:
            raise ValueError("MapReduce map stage must produce terms")
        return i, "scalar"
    if isinstance(node, (LoopFor, LoopWhileChanged, LoopHost)):
        i, o = sig(node.body)
        if not _compat(i, o):
            raise ValueError("loop body must preserve its value kind")
        return i, o
    raise TypeError(node)


def _leaf(node: Leaf, v):
    p = node.params
    k = node.kind
    if k == "saxpy":
        x, y = v
        return Result((x, K.saxpy(p["a"], x, y)))
    if k == "gauss_noise":
        return Result(K.gauss_noise(v, p["seed"], p["scale"]))
    if k == "solarize":
        return Result(K.solarize(v, p["threshold"]))
    if k == "mirror":
        return Result(K.mirror(v))
    if k == "segment":
        return Result(K.segment(v, p["lo"], p["hi"]))
    if k == "hysteresis_finalize":
        return Result(K.hyst_finalize(v))
    if k == "hysteresis_step":
        out, changed = K.hyst_step(v)
        return Result(out, changed=changed)
    if k == "nbody_step":
        pos, vel = v
        po, vo, _ = K.nbody_step(pos, vel, p["eps2"], p["dt"])
        return Result((po, vo))
    if k == "nbody_accel":
        pos = v[0] if isinstance(v, tuple) else v
        acc, _ = K.nbody_accel(pos, p["eps2"])
        return Result(acc)
    if k in ("map_identity", "map_product"):
        return Result(v)  # terms are formed inside the fold (exact in fp64)
    if k == "fft":
        # one transform per row (R23/R24); complex128 flows between
        # FFT stages, fp32 [.., N, 2] in
        x = v if np.iscomplexobj(v) else FF.as_complex(v)
        return Result(FF.fft_chain(x, "I" if p["inverse"] else "F"))
    if k == "debug_traits":
        # one partition: SIZE = L, OFFSET = 0 for every element
        L = int(v)
        out = np.empty((L, 2), dtype=np.int64)
        out[:, 0] = L
        out[:, 1] = 0
        return Result(out)
    raise ValueError(k)


def _merge(op, parts):
    acc = parts[0]
    for r in parts[1:]:
        if op == "-":
            acc = acc - r
        elif op == "*":
            acc = acc * r
        elif op == "/":
            acc = acc / r
        else:
            acc = op(acc, r)
    return acc


def evaluate(node: Node, value, while_counts=None, lengths=None) -> Result:
    """Depth-first evaluation of `node` on `value` (whole domain).  lengths:
    the partition lengths (outer units, global order) — used only by the
    partition-dependent NEXT-4 merging functions."""
    if isinstance(node, Leaf):
        return _leaf(node, value)
    if isinstance(node, Map):
        return evaluate(node.tree, value, lengths=lengths)
    if isinstance(node, Pipeline):
        r = Result(value)
        any_changed, execs, conv = False, 0, True
        for s in node.stages:
            r = evaluate(s, r.value)
            any_changed |= r.changed
            execs += r.executions      # while-loop executions of the whole tree (marrow.h E)
            conv &= r.converged
        r.changed = any_changed
        r.executions, r.converged = execs, conv
        return r
    if isinstance(node, MapReduce):
        m = node.map_stage
        while isinstance(m, Map):
            m = m.tree
        # a map stage that is a pipeline: its leading stages transform the
        # value, the last one (a map leaf) forms the terms
        pre = []
        if isinstance(m, Pipeline):
            pre, m = list(m.stages[:-1]), m.stages[-1]
            while isinstance(m, Map):
                m = m.tree
        if not isinstance(m, Leaf):
            raise NotImplementedError("MapReduce map stage must end with a map leaf")
        if m.kind not in ("map_identity", "map_product"):
            raise ValueError(m.kind)
        for st in pre:
            value = evaluate(st, value).value
        vals = value if isinstance(value, tuple) else (value,)

        def red(sl):
            if m.kind == "map_identity":
                return K.sum_(vals[0][sl])
            return K.dot(vals[0][sl], vals[1][sl])
        if node.op == "+":
            return Result(None, reduced=red(slice(None)))
        if isinstance(node.op, (Leaf, Pipeline)):   # device reduction stage SCT
            stages = [node.op] if isinstance(node.op, Leaf) else list(node.op.stages)
            kinds = [st.kind for st in stages]
            if kinds.count("reduce") != 1:
                raise ValueError("the reduction stage needs exactly one reduce leaf")
            r = kinds.index("reduce")
            rop = stages[r].params.get("op", "sum")
            tmaps = [st.params["map"] for st in stages[:r]]
            y = vals[1] if m.kind == "map_product" else None
            if not tmaps:
                if rop == "sum":
                    acc = red(slice(None))
                else:
                    acc = K.fold_extreme(vals[0], y, is_min=(rop == "min"))
            else:
                # the terms in fp64 (x, or x*y exact), then the term maps in order
                t = vals[0].astype(np.float64) * (y.astype(np.float64) if y is not None else 1.0)
                for tm in tmaps:
                    t = np.abs(t) if tm == "abs" else t * t
                if rop == "sum":
                    acc = K.sum_f64(t)
                else:   # maxNum / minNum: NaN terms ignored, empty -> the identity
                    t = t[~np.isnan(t)]
                    acc = (float(t.min()) if t.size else np.inf) if rop == "min" else \
                          (float(t.max()) if t.size else -np.inf)
            for st in stages[r + 1:]:    # scalar maps of the reduced value, in order
                acc = float(np.sqrt(acc)) if st.params["map"] == "sqrt" else acc * st.params["c"]
            return Result(None, reduced=acc)
        if lengths is None:
            raise ValueError("merging functions other than + need the partition lengths")
        parts, o = [], 0
        for ln in lengths:
            if ln > 0:
                parts.append(red(slice(o, o + ln)))
            o += ln
        return Result(None, reduced=_merge(node.op, parts))
    if isinstance(node, LoopFor):
        r = Result(value)
        execs, conv, changed = 0, True, False
        for _ in range(node.n):
            r = evaluate(node.body, r.value)
            execs += r.executions
            conv &= r.converged
            changed |= r.changed       # a loop body changed iff one of its executions did
        r.executions, r.converged, r.changed = execs, conv, changed
        return r
    if isinstance(node, LoopWhileChanged):
        changed, e, v = True, 0, value
        while changed and e < node.max_iters:
            r = evaluate(node.body, v)
            v, changed = r.value, r.changed
            e += 1
        return Result(v, executions=e, converged=not changed)
    if isinstance(node, LoopHost):
        e, v, stopped = 0, value, False
        while e < node.max_iters:
            if not node.cond(e):       # stage 1 on the host
                stopped = True
                break
            v = evaluate(node.body, v).value
            e += 1
        return Result(v, executions=e, converged=stopped)
    raise TypeError(node)


def leaves(node: Node):
    """Leaves in depth-first (pre-order) order."""
    if isinstance(node, Leaf):
        return [node]
    if isinstance(node, Pipeline):
        return [l for s in node.stages for l in leaves(s)]
    if isinstance(node, Map):
        return leaves(node.tree)
    if isinstance(node, MapReduce):
        return [l for c in _children(node) for l in leaves(c)]
    return leaves(node.body)


def kernel_execution_order(node: Node, while_counts: list[int]) -> list[int]:
    """Single-device kernel order: leaf occurrences numbered in
    pre-order, loop bodies repeated; LoopWhileChanged occurrences (pre-order)
    consume `while_counts`."""
    counts = list(while_counts)

    def nleaves(n):
        return 1 if isinstance(n, Leaf) else sum(nleaves(c) for c in _children(n))

    def nwhile(n):
        return int(isinstance(n, (LoopWhileChanged, LoopHost))) + sum(nwhile(c) for c in _children(n))

    if len(counts) < nwhile(node):
        raise KeyError("MissingIterationCount")

    def walk(n, lb, wb):
        if isinstance(n, Leaf):
            return [lb]
        if isinstance(n, LoopFor):
            return walk(n.body, lb, wb) * n.n
        if isinstance(n, (LoopWhileChanged, LoopHost)):
            return walk(n.body, lb, wb + 1) * counts[wb]
        out = []
        for c in _children(n):
            out += walk(c, lb, wb)
            lb += nleaves(c)
            wb += nwhile(c)
        return out

    return walk(node, 0, 0)


def _children(n):
    if isinstance(n, Leaf):
        return []
    if isinstance(n, Pipeline):
        return list(n.stages)
    if isinstance(n, Map):
        return [n.tree]
    if isinstance(n, MapReduce):   # a reduction-stage SCT runs after the map stage
        return [n.map_stage] + ([n.op] if isinstance(n.op, (Leaf, Pipeline)) else [])
    return [n.body]
