"""C-ABI host logic on CPU (no device calls): exports, tree building and
validation, ids, execution order, granule, partitioner and balancer — each
checked against the oracle (partition/balance/sct) and SPEC/paper examples."""
import random
import re

import numpy as np
import pytest

from oracle import balance as B
from oracle import partition as OP
from oracle import sct
from paper_1510_06585_b200 import marrow as M
from paper_1510_06585_b200 import trees


def test_library_exports_every_header_symbol():
    import ctypes
    hdr = open(__file__.rsplit("/tests/", 1)[0] + "/include/marrow.h").read()
    decl = set(re.findall(r"^\s*(?:mw_status|void|const char\*|int32_t)\s+(mw_\w+)\(", hdr, re.M))
    assert len(decl) >= 45
    lib = ctypes.CDLL(M._LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name
    assert decl == set(M.EXPORTS)
    assert M.lib().mw_abi_version() == 1


def test_status_strings_and_errors():
    assert M.lib().mw_status_string(M.MW_E_EPU_NU) == b"MW_E_EPU_NU"
    with pytest.raises(M.MwError) as e:
        M.mw_pipeline([M.mw_kernel_mirror()])
    assert e.value.status == M.MW_E_INVALID_SPEC and "Pipeline" in str(e.value)
    with pytest.raises(M.MwError) as e:
        M.mw_kernel_debug_traits(3, 2)
    assert e.value.status == M.MW_E_EPU_NU
    with pytest.raises(M.MwError):
        M.mw_pipeline([M.mw_kernel_mirror(), M.mw_kernel_segment(1, 2)])   # kinds do not chain
    with pytest.raises(M.MwError):
        M.mw_kernel_segment(10, 5)
    with pytest.raises(M.MwError):
        M.mw_kernel_gauss_noise(1, 300)
    for bad in (7, -1, M.MW_MERGE_USER):   # USER needs mw_map_reduce_user (a function)
        with pytest.raises(M.MwError) as e:
            M.mw_map_reduce(M.mw_kernel_map_identity(), bad)
        assert e.value.status == M.MW_E_INVALID_SPEC
    with pytest.raises(M.MwError):
        M.mw_loop_host(M.mw_kernel_mirror(), -1, lambda i: True)   # negative max_iters
    with pytest.raises(M.MwError):
        M.mw_loop_while_changed(M.mw_kernel_hysteresis_step(), 10, 0)
    for bad in (12, 17, 0):   # FFT sizes 2^13..2^16 (R23)
        with pytest.raises(M.MwError) as e:
            M.mw_kernel_fft(bad)
        assert e.value.status == M.MW_E_INVALID_SPEC
    with pytest.raises(M.MwError):
        M.mw_pipeline([M.mw_kernel_fft(16), M.mw_kernel_mirror()])   # kinds do not chain


def test_signatures():
    assert M.mw_node_signature(trees.filter_pipeline()) == (M.MW_VK_RGBA, M.MW_VK_RGBA)
    assert M.mw_node_signature(trees.hysteresis()) == (M.MW_VK_U8_2D, M.MW_VK_U8_2D)
    assert M.mw_node_signature(trees.segmentation()) == (M.MW_VK_U8, M.MW_VK_U8)
    assert M.mw_node_signature(trees.mapreduce(True)) == (M.MW_VK_VEC2, M.MW_VK_SCALAR)
    assert M.mw_node_signature(trees.nbody(3)) == (M.MW_VK_NBODY, M.MW_VK_NBODY)
    assert M.mw_node_signature(M.mw_kernel_nbody_accel(1e-4)) == (M.MW_VK_NBODY, M.MW_VK_ACCEL)
    assert M.mw_node_signature(trees.fft_pipeline()) == (M.MW_VK_CPLX, M.MW_VK_CPLX)
    assert M.mw_node_id(trees.fft_pipeline(16)) != M.mw_node_id(trees.fft_pipeline(15))
    assert M.mw_kernel_execution_order(M.mw_loop_for(trees.fft_pipeline(), 2), []) == [0, 1, 0, 1]
    # a host-condition loop takes its count like a while-loop (known after the run)
    lh = M.mw_loop_host(trees.filter_pipeline(), 10, lambda i: i < 2)
    assert M.mw_kernel_execution_order(lh, [2]) == [0, 1, 2, 0, 1, 2]
    assert M.mw_node_signature(M.mw_map_reduce(M.mw_kernel_map_product(), M.MW_MERGE_DIV)) == \
        (M.MW_VK_VEC2, M.MW_VK_SCALAR)
    assert M.mw_node_id(M.mw_map_reduce(M.mw_kernel_map_identity(), M.MW_MERGE_SUB)) != \
        M.mw_node_id(M.mw_map_reduce(M.mw_kernel_map_identity(), M.MW_MERGE_MUL))
    # device reduction stage (NEXT-4): map stage then reduction stage
    for op in (M.MW_REDUCE_SUM, M.MW_REDUCE_MAX, M.MW_REDUCE_MIN):
        t = trees.mapreduce_sct(op)
        assert M.mw_node_signature(t) == (M.MW_VK_VEC2, M.MW_VK_SCALAR)
        assert M.mw_kernel_execution_order(t, []) == [0, 1]
    ids = {M.mw_node_id(trees.mapreduce_sct(op, d)) for op in range(3) for d in (False, True)}
    assert len(ids) == 6
    assert M.mw_node_id(trees.mapreduce_sct(M.MW_REDUCE_SUM)) != M.mw_node_id(trees.mapreduce(True))
    for bad in (lambda: M.mw_kernel_reduce(3), lambda: M.mw_kernel_reduce(-1),
                lambda: M.mw_map_reduce_sct(M.mw_kernel_map_product(), M.mw_kernel_map_identity()),
                lambda: M.mw_map_reduce_sct(M.mw_kernel_mirror(), M.mw_kernel_reduce(1))):
        with pytest.raises(M.MwError) as e:
            bad()
        assert e.value.status == M.MW_E_INVALID_SPEC


def test_node_id_determinism():
    a, b = trees.filter_pipeline(), trees.filter_pipeline()
    assert M.mw_node_id(a) == M.mw_node_id(b)
    assert M.mw_node_id(a) != M.mw_node_id(trees.filter_pipeline(seed=5))
    assert M.mw_node_id(trees.hysteresis(check_every=1)) != M.mw_node_id(trees.hysteresis(check_every=4))
    assert M.mw_node_id(M.mw_kernel_saxpy(1.0)) != M.mw_node_id(M.mw_kernel_saxpy(float(np.nextafter(np.float32(1), np.float32(2)))))
    assert len(M.mw_node_id(a)) == 32


def _pair(kind_tree):
    """Build the same random tree on both sides: (oracle node, C-ABI node)."""
    return kind_tree


def test_execution_order_matches_oracle():
    # Fig. 1: pipeline(K1, loop(K2), K3) with 3 iterations -> K1, K2 x3, K3
    assert M.mw_kernel_execution_order(trees.hysteresis(), [3]) == [0, 1, 1, 1, 2]
    with pytest.raises(M.MwError) as e:
        M.mw_kernel_execution_order(trees.hysteresis(), [])
    assert e.value.status == M.MW_E_MISSING_ITERATION_COUNT
    rng = random.Random(3)
    for _ in range(200):
        o, c = _random_rgba_tree(rng, 3)
        assert M.mw_kernel_execution_order(c, []) == sct.kernel_execution_order(o, [])
    # shared leaf objects are numbered per occurrence
    m = M.mw_kernel_mirror()
    om = sct.Leaf("mirror")
    assert M.mw_kernel_execution_order(M.mw_pipeline([m, M.mw_loop_for(m, 2), m]), []) == \
        sct.kernel_execution_order(sct.Pipeline([om, sct.LoopFor(om, 2), om]), []) == [0, 1, 1, 2]
    ow = sct.LoopWhileChanged(sct.Leaf("hysteresis_step"), 9)
    cw = M.mw_loop_while_changed(M.mw_kernel_hysteresis_step(), 9)
    o = sct.Pipeline([ow, sct.LoopFor(sct.Pipeline([ow, ow]), 2)])
    c = M.mw_pipeline([cw, M.mw_loop_for(M.mw_pipeline([cw, cw]), 2)])
    assert M.mw_kernel_execution_order(c, [1, 2, 3]) == sct.kernel_execution_order(o, [1, 2, 3])


def _random_rgba_tree(rng, depth):
    if depth == 0 or rng.random() < 0.3:
        k = rng.choice(["gauss_noise", "solarize", "mirror"])
        if k == "gauss_noise":
            s, S = rng.randint(0, 99), rng.randint(0, 20)
            return sct.Leaf(k, {"seed": s, "scale": S}), M.mw_kernel_gauss_noise(s, S)
        if k == "solarize":
            t = rng.randint(0, 256)
            return sct.Leaf(k, {"threshold": t}), M.mw_kernel_solarize(t)
        return sct.Leaf(k), M.mw_kernel_mirror()
    r = rng.random()
    if r < 0.4:
        kids = [_random_rgba_tree(rng, depth - 1) for _ in range(rng.randint(2, 3))]
        return sct.Pipeline([k[0] for k in kids]), M.mw_pipeline([k[1] for k in kids])
    if r < 0.7:
        o, c = _random_rgba_tree(rng, depth - 1)
        n = rng.randint(0, 3)
        return sct.LoopFor(o, n), M.mw_loop_for(c, n)
    o, c = _random_rgba_tree(rng, depth - 1)
    return sct.Map(o), M.mw_map(c)


def test_granule():
    assert M.mw_granule(trees.filter_pipeline()) == 1
    assert M.mw_granule(trees.saxpy()) == 4
    assert M.mw_granule(trees.mapreduce()) == 1 << 16
    assert M.mw_granule(trees.nbody(1)) == 256
    assert M.mw_granule(M.mw_kernel_debug_traits(6, 2)) == 3
    assert M.mw_granule(M.mw_pipeline([M.mw_kernel_debug_traits(4, 1),
                                       M.mw_kernel_debug_traits(6, 1)])) == 12
    # S:129-131
    assert OP.granule([(4, 2), (4, 1)], align=16) == 16


def test_partition_plan_matches_oracle():
    assert M.mw_partition_plan(1024, 16, [0.75, 0.25]) == ([0, 768], [768, 256])
    assert M.mw_partition_plan(8192, 1, [1 / 3] * 3)[1] == [2731, 2731, 2730]
    with pytest.raises(M.MwError) as e:
        M.mw_partition_plan(8, 16, [0.5, 0.5], strict=True)
    assert e.value.status == M.MW_E_INFEASIBLE_PARTITION
    for bad in ([0.5, 0.6], [-0.1, 1.1], [0.0, 0.0]):
        with pytest.raises(M.MwError):
            M.mw_partition_plan(10, 1, bad)
    rng = random.Random(5)
    for _ in range(3000):
        k = rng.randint(1, 8)
        w = [rng.choice([0, 0, 1, 2, 3, 7, 1000, rng.random()]) for _ in range(k)]
        if not any(w):
            w[rng.randrange(k)] = 1
        s = sum(w)
        d = [x / s for x in w]
        g = rng.choice([1, 4, 256, 65536])
        L = rng.randint(0, 1 << rng.randint(0, 31))
        assert M.mw_partition_plan(L, g, d) == tuple(map(list, OP.partition(L, g, d)))


def test_balance_step_matches_oracle_replay():
    rng = random.Random(9)
    for mode in (B.PROPORTIONAL, B.ABS):
        k = 2 if mode == B.ABS else 5
        po = B.Params(mode=mode)
        so = B.State()
        pc = M.mw_balance_defaults(mode)
        sc = M.mw_balance_state()
        d = [1.0 / k] * k
        rate = [1.0] * k
        for run in range(400):
            if run % 37 == 0:
                rate = [rng.choice([1.0, 0.5, 0.25, 2.0]) for _ in range(k)]
            _, ln = OP.partition(1 << 20, 256, d)
            t = [float(np.float32(ln[i] / rate[i] * 1e-6 * (1 + 0.05 * rng.random()))) for i in range(k)]
            no, to = B.step(po, so, t, ln, d)
            nc, tc = M.mw_balance_step(pc, sc, t, ln, d)
            assert nc == no and to == tc and sc.lbt == so.lbt, run
            d = no
        assert so.runs == 400


def test_balance_paper_sequences():
    p, s = M.mw_balance_defaults(), M.mw_balance_state()
    lbts = []
    for _ in range(3):
        _, trig = M.mw_balance_step(p, s, [1.0, 2.0], [10, 10], [0.5, 0.5])
        lbts.append((round(s.lbt, 4), trig))
    assert lbts[:2] == [(0.6667, False), (0.8889, False)] and lbts[2][1]


def test_ctx_create_validation_without_gpu():
    with pytest.raises(M.MwError):
        M.mw_ctx_create(0, 1, 1, 1, torch_alloc=False)      # rank >= nranks
    with pytest.raises(M.MwError):
        M.mw_ctx_create(0, 0, 2, 1, torch_alloc=False)      # NCCL id missing
