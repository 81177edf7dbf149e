"""Wide values: integer activations whose column sums exceed int32, float64 holding integers
(the reference's calling convention), high-dynamic-range floats and more than 65536 rows.

The fixtures (golden/overflow.npz) are the REAL reference's outputs (make_golden.overflow) on
inputs regenerated here from seeds (golden/overflow_inputs.py, digests checked).  The
reference computes in fp64 (core.py:110-117), so it is exact for every integer vector whose
partial sums stay below 2^53 — SPEC.md:276 promises |v| <= 2^20 at up to 2^20 rows.  There
the GPU results must be bitwise equal to it on every entry point (host multiply_ternary /
multiply_rsr, multiply_parallel, int64 device tensors).  Beyond 2^53, and for non-integer
floats, the comparison is a stated tolerance."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

sys.path.insert(0, GOLDEN)
from overflow_inputs import CASES, digest, make_inputs  # noqa: E402

EXACT = ["t_i32_2p20", "t_i64_pm2p20", "t_i64_2p36", "b_i32_pos2p20", "t_f64int_2p20", "t_i64_rows70000"]
CLASS = {"t_i32_2p20": "wide", "t_i64_pm2p20": "wide", "t_i64_2p36": "wide", "b_i32_pos2p20": "wide",
         "t_f64int_2p20": "wide", "t_i64_2p50": "wide", "t_f64_hdr": "f64", "t_f32_hdr": "f32",
         "t_f64_rows70000": "fixed", "t_i64_rows70000": "wide"}


@pytest.fixture(scope="module")
def ov():
    return load_golden("overflow.npz")


def _inputs(ov, name):
    A, v = make_inputs(name)
    assert digest(A) == str(ov[name + "_A_digest"]) and digest(v) == str(ov[name + "_v_digest"]), \
        "seeded inputs drifted from the ones the fixture was made with"
    return A, v


def _exact(A, v, domain):
    """Exact integer product in Python ints (object arithmetic)."""
    M = A.astype(np.int64) if domain == "ternary" else (A == 1).astype(np.int64)
    return (np.asarray(v).astype(object) @ M.astype(object))


# ----------------------------------------------------------------------------- CPU
@pytest.mark.parametrize("name", sorted(CASES))
def test_classifier(rsr, ov, name):
    """The NumPy restatement of the host staging classes (kernels.classify_host_vector): every
    fixture leaves the int32 kernel (its sums exceed int32), integer-valued ones take the exact
    wide multiply."""
    from paper_2411_06360_b200.kernels import classify_host_vector
    _, v = _inputs(ov, name)
    kind, arr, mx = classify_host_vector(np.asarray(v))
    assert kind == CLASS[name]
    if kind in ("wide", "fixed"):
        assert arr.dtype == np.int64 and mx == int(np.abs(arr).max())
    if kind == "fixed":  # |v_q| < 2^62 and round(v * 2^exp2)
        cls = classify_host_vector(np.asarray(v))
        assert mx < 2 ** 62 and np.array_equal(arr, np.rint(np.ldexp(np.asarray(v, np.float64), cls.exp2)).astype(np.int64))
    small = (np.asarray(v)[:100] // (2 ** 25 if kind == "wide" else 1)).astype(np.int64) % 50
    assert classify_host_vector(small)[0] == "i32"


@pytest.mark.parametrize("name", EXACT)
def test_reference_is_exact_here(ov, name):
    """Pin the fixture: in the exact regime the reference's fp64 output IS the exact integer
    product (so bitwise equality with it is the right bar)."""
    domain = CASES[name][0]
    A, v = _inputs(ov, name)
    ref = _exact(A, v, domain)
    assert all(float(x) == y for x, y in zip(ref, ov[name + "_rsrpp"]))
    assert np.array_equal(ov[name + "_rsr"], ov[name + "_rsrpp"])
    assert np.array_equal(ov[name + "_par3"], ov[name + "_rsrpp"])


def test_limb_plan():
    """csrc/wide.cu digit width s (rows * 2^(s-1) <= 2^31 - 1) and limb count, restated."""
    def bits(rows):
        s = 1
        while s < 31 and (rows << s) <= 2 ** 31 - 1:
            s += 1
        return s
    for rows, s in ((1, 31), (16384, 17), (16385, 17), (32768, 16), (65536, 15), (70000, 15), (1 << 20, 11)):
        assert bits(rows) == s
        assert rows * 2 ** (s - 1) <= 2 ** 31 - 1


# ----------------------------------------------------------------------------- GPU
def _index(rsr, A, domain, k):
    import torch
    if domain == "ternary":
        return rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k), rsr.multiply_ternary
    return rsr.preprocess(rsr.BinaryMatrix.from_dense(A.astype(np.uint8)), k), rsr.multiply_rsr


@pytest.mark.gpu
@pytest.mark.parametrize("name", EXACT)
def test_wide_integer_bitwise(rsr, cuda, ov, name):
    """Host vectors (the reference contract): bitwise equal to the reference for both
    variants and multiply_parallel; int32 / int64 / float64-integer forms of the same values
    agree; int64 device tensors give the exact integers."""
    import torch
    domain, rows, cols, k, kind, bound = CASES[name]
    A, v = _inputs(ov, name)
    idx, mult = _index(rsr, A, domain, k)
    for variant in ("rsrpp", "rsr"):
        got = mult(v, idx, variant)
        assert got.dtype == np.float64 and np.array_equal(got, ov[f"{name}_{variant}"]), variant
    assert np.array_equal(rsr.multiply_parallel(v, idx, "rsrpp", 3), ov[name + "_par3"])
    assert np.array_equal(rsr.multiply_parallel(v, idx, "rsrpp", 1), ov[name + "_par3"])
    v64 = np.asarray(v).astype(np.int64)
    for form in (v64, v64.astype(np.float64)) + ((v64.astype(np.int32),) if np.abs(v64).max() < 2 ** 31 else ()):
        assert np.array_equal(mult(form, idx), ov[name + "_rsrpp"]), form.dtype
    dev = mult(torch.from_numpy(v64).cuda(), idx)
    assert dev.dtype == torch.int64
    exact = _exact(A, v64, domain)
    assert [int(x) for x in dev.cpu().numpy()] == [int(x) for x in exact]


@pytest.mark.gpu
def test_beyond_2p53_rounds_once(rsr, cuda, ov):
    """|v| up to 2^50: partial sums pass 2^53, the reference's fp64 accumulation rounds.  Ours
    is the exact integer rounded once: equal to float(exact), and within 2^-40 of the
    reference relative to sum |v|."""
    name = "t_i64_2p50"
    domain, rows, cols, k, kind, bound = CASES[name]
    A, v = _inputs(ov, name)
    idx, mult = _index(rsr, A, domain, k)
    got = mult(v, idx)
    exact = _exact(A, v, domain)
    assert np.array_equal(got, np.array([float(x) for x in exact]))
    scale = float(np.abs(v.astype(np.float64)).sum())
    assert np.abs(got - ov[name + "_rsrpp"]).max() <= 2.0 ** -40 * scale


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["t_f64_hdr", "t_f64_rows70000"])
def test_float64_tolerance(rsr, cuda, ov, name):
    """Non-integer float64 on the fp64 gather kernel (rows beyond 65536 included): within the
    reference's float tolerance (rtol 1e-9, test_kernels.py:190-201), elementwise relative to
    the condition sum_i |v_i A_ij|."""
    domain, rows, cols, k, kind, bound = CASES[name]
    A, v = _inputs(ov, name)
    idx, mult = _index(rsr, A, domain, k)
    cond = np.abs(v) @ np.abs(A.astype(np.float64))
    for variant in ("rsrpp", "rsr"):
        got = mult(v, idx, variant)
        err = np.abs(got - ov[f"{name}_{variant}"]) / cond
        assert err.max() <= 1e-12, (variant, float(err.max()))
    assert (np.abs(rsr.multiply_parallel(v, idx, "rsrpp", 3) - ov[name + "_par3"]) / cond).max() <= 1e-12


@pytest.mark.gpu
def test_float32_high_dynamic_range(rsr, cuda, ov):
    """fp32 activations spanning ~1e-5..1e9 (outliers): the exact fixed-point path's error,
    reported elementwise relative to the condition sum_i |v_i A_ij| (the scale of any fp32
    dot product's rounding), and norm-wise against the north-star 1e-5 bound."""
    name = "t_f32_hdr"
    domain, rows, cols, k, kind, bound = CASES[name]
    A, v = _inputs(ov, name)
    idx, mult = _index(rsr, A, domain, k)
    ref = ov[name + "_rsrpp"]
    cond = np.abs(v.astype(np.float64)) @ np.abs(A.astype(np.float64))
    got = mult(v, idx)
    elem = np.abs(got - ref) / cond
    print(f"fp32 HDR: max elementwise error / condition = {elem.max():.3e}, "
          f"norm-wise = {np.abs(got - ref).max() / np.abs(ref).max():.3e}")
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    assert elem.max() <= 1e-7  # measured 1.9e-8 on the B200


@pytest.mark.gpu
@pytest.mark.parametrize("rows", [37, 1003, 16384])
def test_staging_edge_values(rsr, cuda, rows):
    """The C staging classifier (csrc/host_stage.cpp, AVX2 body + scalar tail) on the values at
    its class boundaries, through the host session: exact against integer arithmetic wherever the
    reference's fp64 result is exact; non-finite entries raise the reference's error."""
    rng = np.random.default_rng(rows)
    A = rng.integers(-1, 2, size=(rows, 29), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 5)
    exact = lambda v: [int(x) for x in (A.astype(object).T @ np.asarray(v, dtype=object))]

    def check(v):
        for form in (v, v.astype(np.float64)) + ((v.astype(np.int32),) if np.abs(v).max() < 2 ** 31 else ()):
            got = rsr.multiply_ternary(form, idx)
            assert [int(x) for x in got] == [float(int(e)) for e in exact(v)], (form.dtype, rows)

    base = rng.integers(-100, 101, size=rows).astype(np.int64)
    for pos in (0, rows - 1, rows // 2):  # the AVX2 body and the scalar tail
        for val in (-2 ** 31, 2 ** 31 - 1, 2 ** 31, -(2 ** 31) - 1, 2 ** 40):
            v = base.copy()
            v[pos] = val
            check(v)
    # max |v| * rows > 2^31 - 1 but sum |v| <= 2^31 - 1: the exact-sum branch stays on int32
    v = np.zeros(rows, np.int64)
    v[-1] = 2 ** 31 - 2
    check(v)
    v[0] = 1
    check(v)
    v[1 % rows] += 1  # sum 2^31 (rows >= 2: wide)
    check(v)
    # fractional / negative zero: fp64 gather (reference tolerance) and exact zero
    vf = base.astype(np.float64)
    vf[rows - 1] += 0.5
    got = rsr.multiply_ternary(vf, idx)
    np.testing.assert_allclose(got, A.T.astype(np.float64) @ vf, rtol=1e-9, atol=1e-9)
    assert np.array_equal(rsr.multiply_ternary(-np.zeros(rows), idx), np.zeros(29))
    for bad in (np.nan, np.inf, -np.inf):
        for pos in (0, rows - 1):
            vb = base.astype(np.float64)
            vb[pos] = bad
            with pytest.raises(ValueError, match="finite"):
                rsr.multiply_ternary(vb, idx)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k", [(1000, 333, 8), (16384, 700, 11), (4096, 4096, 10), (9000, 257, 9)])
def test_fixed_point_float64(rsr, cuda, rows, cols, k):
    """Non-integer float64 vectors with a moderate dynamic range take the fixed-point route
    (host_stage.cpp kStageFixed -> rsr_multiply_fixed): the exact product of round(v * 2^e),
    rounded once.  Within 2^-40 of the condition sum |v_i A_ij| of the exact (object-arithmetic)
    product, within the reference's float tolerance of its fp64 result, and bitwise equal
    between the session (multiply_ternary) and multiply_parallel (same classification)."""
    from oracle import c_oracle
    from paper_2411_06360_b200.kernels import classify_host_vector
    rng = np.random.default_rng([rows, cols, k, 64])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    for trial in range(3):
        v = rng.standard_normal(rows) * 10.0 ** rng.integers(-3, 4)
        fixed = classify_host_vector(v)[0] == "fixed"
        assert fixed == (rows >= 8192)  # below 8192 rows the fp64 gather kernel is the faster route
        got = rsr.multiply_ternary(v, idx)
        ref = c_oracle.naive_ternary(v, A)
        cond = np.abs(v) @ np.abs(A.astype(np.float64))
        np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)
        assert (np.abs(got - ref) / cond).max() <= 1e-12
        assert np.array_equal(rsr.multiply_parallel(v, idx, "rsrpp", 3), got)
        if fixed:  # exact integers: both variants agree bitwise
            assert np.array_equal(rsr.multiply_ternary(v, idx, "rsr"), got)
