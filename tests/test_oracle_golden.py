"""Pin the CPU oracle (oracle/rsr_oracle.py and oracle/rsr_oracle.c) to golden vectors
produced by the real reference (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import unpack_index
from oracle import c_oracle
from oracle import rsr_oracle as O


def test_worked_example_known_answers(worked):
    # conftest.py:10-26 of the reference: sigma [1,4,5,0,2,3], L [0,3,5,5], sums [12,7,0,5]
    B6, V6 = worked["B6"], worked["V6"]
    perms, segs, buckets = O.preprocess_binary(B6, 2)
    assert np.array_equal(perms[0], [1, 4, 5, 0, 2, 3])
    assert np.array_equal(segs[0][:-1], [0, 3, 5, 5])
    assert np.array_equal(perms[0], worked["block0_perm"])
    assert np.array_equal(segs[0][:-1], worked["block0_seg"])
    u = O.segment_sums(V6, perms[0], segs[0], 2)
    assert np.array_equal(u, worked["block0_sums"])
    assert np.array_equal(O.product_fold(u, 2), [5.0, 12.0])
    assert np.array_equal(O.product_dense(u, 2), [5.0, 12.0])
    out = O.multiply_half(V6, buckets, 6, 2, True)
    assert np.array_equal(out, worked["product_binary"])
    assert np.array_equal(out, [5.0, 12.0, 16.0, 18.0, 12.0, 14.0])
    (pp, ps, pb), (np_, ns, nb) = O.preprocess_ternary(B6.astype(np.int8), 2)
    assert np.array_equal(O.multiply_ternary(V6, pb, nb, 6, 2), worked["product_ternary"])
    assert np.array_equal(O.naive_multiply(V6, B6), worked["naive"])


def test_numpy_oracle_matches_reference_index_and_products(fuzz):
    for i in range(int(fuzz["count"])):
        p = f"c{i}_"
        A, k = fuzz[p + "A"], int(fuzz[p + "k"])
        (pp, ps, pb), (np_, ns, nb) = O.preprocess_ternary(A, k)
        rp, rs, rb = unpack_index(fuzz, p + "pos_")
        assert np.array_equal(pp, rp)
        assert all(np.array_equal(a, b) for a, b in zip(ps, rs))
        assert np.array_equal(pb, rb)
        rp, rs, rb = unpack_index(fuzz, p + "neg_")
        assert np.array_equal(np_, rp)
        assert all(np.array_equal(a, b) for a, b in zip(ns, rs))
        for vk in ("int", "flt"):
            v = fuzz[p + ("vi" if vk == "int" else "vf")]
            for variant, fold in (("rsr", False), ("rsrpp", True)):
                got = O.multiply_ternary(v, pb, nb, A.shape[1], k, fold)
                # same summation order as the reference => bitwise equal, floats included
                assert got.tobytes() == fuzz[p + f"{vk}_{variant}"].tobytes()
            assert O.naive_multiply(v, A).tobytes() == fuzz[p + f"{vk}_naive"].tobytes()


def test_c_oracle_matches_reference(fuzz):
    for i in range(int(fuzz["count"])):
        p = f"c{i}_"
        A, k = fuzz[p + "A"], int(fuzz[p + "k"])
        (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
        rp, rs, rb = unpack_index(fuzz, p + "pos_")
        assert np.array_equal(pp, rp)
        assert all(np.array_equal(a, b) for a, b in zip(ps, rs))
        assert np.array_equal(pb, rb)
        rp, rs, rb = unpack_index(fuzz, p + "neg_")
        assert np.array_equal(np_, rp) and np.array_equal(nb, rb)
        for vk in ("int", "flt"):
            v = fuzz[p + ("vi" if vk == "int" else "vf")]
            for variant, fold in (("rsr", False), ("rsrpp", True)):
                for workers in (1, 3):
                    got = c_oracle.multiply_parallel(v, pb, nb, A.shape[1], k, fold, workers)
                    assert got.tobytes() == fuzz[p + f"{vk}_{variant}"].tobytes()
            assert c_oracle.naive_ternary(v, A).tobytes() == fuzz[p + f"{vk}_naive"].tobytes()
        got = c_oracle.multiply_parallel(fuzz[p + "vi"], pb, None, A.shape[1], k, True, 2)
        assert got.tobytes() == fuzz[p + "int_pos_rsrpp"].tobytes()


def test_c_oracle_medium_shapes(medium):
    for i in range(4):
        p = f"m{i}_"
        rows, cols = (int(x) for x in medium[p + "shape"])
        k = int(medium[p + "k"])
        rng = np.random.default_rng([2411, rows, cols])
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        v = rng.integers(-100, 101, size=rows).astype(np.float64)
        (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
        crc = np.array([int(np.bitwise_xor.reduce(pp[b].astype(np.uint64)
                                                   * np.arange(1, rows + 1, dtype=np.uint64)))
                        for b in range(pp.shape[0])], np.uint64)
        assert np.array_equal(crc, medium[p + "pos_perm_crc"])
        assert np.array_equal([int(s[:-1].sum()) for s in ns], medium[p + "neg_seg_sum"])
        for variant, fold in (("rsrpp", True), ("rsr", False)):
            got = c_oracle.multiply_parallel(v, pb, nb, cols, k, fold, 4)
            assert got.tobytes() == medium[p + variant].tobytes()
        assert c_oracle.naive_ternary(v, A).tobytes() == medium[p + "naive"].tobytes()


def test_folds_match_reference(folds):
    for w in range(1, 11):
        for tag in ("i", "f"):
            u = folds[f"w{w}{tag}_u"]
            assert O.product_fold(u, w).tobytes() == folds[f"w{w}{tag}_rsrpp"].tobytes()
            assert O.product_dense(u, w).tobytes() == folds[f"w{w}{tag}_rsr"].tobytes()


def test_tuner_matches_reference(tuner):
    for n, kpp, kr, mk in zip(tuner["n"], tuner["k_rsrpp"], tuner["k_rsr"], tuner["max_k"]):
        assert O.optimal_k_rsrpp(int(n)) == kpp
        assert O.optimal_k_rsr(int(n)) == kr
        assert O.max_k_for_rows(int(n)) == mk


@pytest.mark.parametrize("rows,cols,k", [(1, 1, 1), (7, 13, 2), (64, 3, 3), (100, 100, 6)])
def test_c_and_numpy_oracles_agree(rows, cols, k):
    rng = np.random.default_rng([rows, cols, k])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    (pp, ps, pb), _ = O.preprocess_ternary(A, k)
    (cp, cs, cb), _ = c_oracle.preprocess_ternary(A, k)
    assert np.array_equal(pp, cp) and np.array_equal(pb, cb)
    assert all(np.array_equal(a, b) for a, b in zip(ps, cs))
