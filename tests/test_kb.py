"""Knowledge Base (NEXT-2) host logic on CPU: records of profile items
(a)-(f), progressive refinement and derivation by
scope narrowing SCT -> workload -> dimensionality."""
import os

from paper_1510_06585_b200 import marrow as M
from paper_1510_06585_b200 import trees

T0 = [1, 2, 1, 8, 40, 0, 1, 1, 4, 1]
T1 = [0, 4, 1, 8, 40, 0, 0, 0, 1, 0]
T2 = [3, 2, 0, 4, 32, 1, 1, 1, 2, 1]


def test_store_lookup_exact_and_refinement(tmp_path):
    kb = M.mw_kb_open(None)
    f = trees.filter_pipeline()
    M.mw_kb_store(kb, f, [8192, 8192, 4], T0, [0.5, 0.5], 0.10)
    assert M.mw_kb_lookup(kb, f, [8192, 8192, 4], 2) == (M.MW_KB_EXACT, T0, [0.5, 0.5])
    M.mw_kb_store(kb, f, [8192, 8192, 4], T1, [0.6, 0.4], 0.20)        # worse: ignored
    assert M.mw_kb_lookup(kb, f, [8192, 8192, 4], 2)[1] == T0
    M.mw_kb_store(kb, f, [8192, 8192, 4], T1, [0.6, 0.4], 0.05)        # better: replaces
    assert M.mw_kb_lookup(kb, f, [8192, 8192, 4], 2) == (M.MW_KB_EXACT, T1, [0.6, 0.4])
    assert M.mw_kb_count(kb) == 1
    # partition count mismatch -> uniform fractions
    assert M.mw_kb_lookup(kb, f, [8192, 8192, 4], 4)[2] == [0.25] * 4


def test_scope_narrowing_order():
    kb = M.mw_kb_open(None)
    f, f2, seg = trees.filter_pipeline(), trees.filter_pipeline(seed=99), trees.segmentation()
    M.mw_kb_store(kb, f, [1024, 1024, 4], T0, [1.0], 1.0)
    M.mw_kb_store(kb, f, [4096, 4096, 4], T1, [1.0], 1.0)
    M.mw_kb_store(kb, seg, [512, 512, 4], T2, [1.0], 1.0)
    # same SCT, unseen workload: nearest neighbour among this SCT's records (log2 space)
    sc, t, _ = M.mw_kb_lookup(kb, f, [3000, 3000, 4])
    assert sc == M.MW_KB_SCT and t == T1
    sc, t, _ = M.mw_kb_lookup(kb, f, [1500, 1500, 4])
    assert sc == M.MW_KB_SCT and t == T0
    # unseen SCT, known workload: the record of that exact workload
    sc, t, _ = M.mw_kb_lookup(kb, f2, [512, 512, 4])
    assert sc == M.MW_KB_WORKLOAD and t == T2
    # unseen SCT and workload: same dimensionality, nearest
    sc, t, _ = M.mw_kb_lookup(kb, f2, [600, 600, 4])
    assert sc == M.MW_KB_DIMENSIONALITY and t == T2
    # nothing of that dimensionality
    assert M.mw_kb_lookup(kb, f2, [10, 10]) == (M.MW_KB_NONE, None, None)


def test_persistence_roundtrip(tmp_path):
    path = str(tmp_path / "kb.txt")
    kb = M.mw_kb_open(path)
    h = trees.hysteresis()
    M.mw_kb_store(kb, h, [16384, 16384], T2, [0.25, 0.25, 0.5], 0.667, M.MW_PROV_BALANCED)
    M.mw_kb_close(kb)
    assert os.path.getsize(path) > 0
    kb2 = M.mw_kb_open(path)
    assert M.mw_kb_count(kb2) == 1
    assert M.mw_kb_lookup(kb2, h, [16384, 16384], 3) == (M.MW_KB_EXACT, T2, [0.25, 0.25, 0.5])
    # a derived record is always replaced by a built one
    M.mw_kb_store(kb2, h, [2048, 2048], T0, [1.0], 0.001, M.MW_PROV_DERIVED)
    M.mw_kb_store(kb2, h, [2048, 2048], T1, [1.0], 9.0, M.MW_PROV_BUILT)
    assert M.mw_kb_lookup(kb2, h, [2048, 2048])[1] == T1
