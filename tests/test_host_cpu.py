"""Host-side logic of the product package and the C ABI, without a GPU:
library load + exported symbols, index layout math, validation errors with the
reference's messages, tuner and blocking helpers (CPU only)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_header_symbol():
    from paper_2411_06360_b200 import _native
    header = open(os.path.join(ROOT, "include", "rsr_b200.h")).read()
    declared = set(re.findall(r"\b(rsr_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    syms = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rsr_[a-z0-9_]+)", syms))
    assert declared <= exported
    L = _native.lib()  # loads without a GPU
    assert L.rsr_b200_abi_version() == _native.ABI_VERSION


def test_host_extension_links_the_library():
    """The CPython binding of the host-buffer session loads without a GPU and resolves
    rsr_host_session_multiply from the same in-tree librsr_b200.so."""
    from paper_2411_06360_b200 import _native
    ext = _native.host_ext()
    assert callable(ext.multiply)
    assert os.path.dirname(_native.EXT_PATH) == os.path.dirname(_native.LIB_PATH)
    deps = subprocess.run(["ldd", _native.EXT_PATH], capture_output=True, text=True).stdout
    assert os.path.realpath(_native.LIB_PATH) in {os.path.realpath(p) for p in re.findall(r"=> (\S+)", deps)}
    with pytest.raises(TypeError):
        ext.multiply(0)


def test_library_is_sm100a():
    from paper_2411_06360_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_layout_math_and_k_errors():
    from paper_2411_06360_b200 import _native
    desc, pb, sb, bb = _native.layout(16384, 16384, 11, 2)
    assert desc.nblocks == 1490 and desc.row_stride == 16384 and desc.seg_stride == 2049
    assert desc.perm_bytes == 2 and pb == 1490 * 16384 * 2 and sb == 1490 * 2049 * 4 and bb == pb
    desc, pb, sb, bb = _native.layout(6, 6, 2, 1)
    assert desc.nblocks == 3 and desc.row_stride == 8 and desc.seg_stride == 5
    desc, *_ = _native.layout(70000, 5, 3, 2)
    assert desc.perm_bytes == 4
    with pytest.raises(ValueError, match=r"k must be in \[1, 30\]"):
        _native.layout(6, 6, 0, 1)
    with pytest.raises(ValueError, match="exceeds max 2 for 6 rows"):
        _native.layout(6, 6, 3, 1)
    with pytest.raises(ValueError, match="device limit"):
        _native.layout(1 << 20, 8, 17, 1)


def test_value_types_and_validation(rsr):
    A = rsr.TernaryMatrix(np.array([[1.0, -1.0], [0.0, 1.0]]))
    assert A.entries.dtype == np.int8 and (A.rows, A.cols) == (2, 2)
    for bad in (2, -2, 0.5, 100):
        with pytest.raises(ValueError):
            rsr.TernaryMatrix(np.array([[1, bad], [0, 1]], np.float64))
    with pytest.raises(ValueError):
        rsr.TernaryMatrix(np.zeros((0, 3), np.int8))
    with pytest.raises(ValueError):
        A.entries[0, 0] = 1
    B = rsr.BinaryMatrix.from_dense(np.array([[1, 0, 0, 0, 0, 0, 0, 1]]))
    assert B.bits[0, 0] == 0b10000001
    with pytest.raises(ValueError):
        rsr.BinaryMatrix(1, 7, np.array([[0b10000001]], np.uint8))
    pair = rsr.decompose_ternary(rsr.TernaryMatrix(np.array([[1, -1], [0, 1]], np.int8)))
    assert np.array_equal(pair.positive.to_dense(), [[1, 0], [0, 1]])
    assert np.array_equal(pair.negative.to_dense(), [[0, 1], [0, 0]])
    assert rsr.as_vector([1, 2, 3]).dtype == np.float64
    for bad in ([], np.zeros((2, 2)), [1.0, np.nan]):
        with pytest.raises(ValueError):
            rsr.as_vector(bad)


def test_blocking_and_bits(rsr):
    assert rsr.column_blocks(6, 2) == [(0, 2), (2, 2), (4, 2)]
    assert rsr.column_blocks(5, 2) == [(0, 2), (2, 2), (4, 1)]
    assert rsr.column_blocks(4, 8) == [(0, 4)]
    B = rsr.BinaryMatrix.from_dense(np.array([[1, 0, 1, 1]]))
    assert rsr.bucket_value(B, 0, 0, 4) == 0b1011
    assert [[rsr.bin_pattern_bit(2, j, c) for c in range(2)] for j in range(4)] == [[0, 0], [0, 1], [1, 0], [1, 1]]
    with pytest.raises(ValueError):
        rsr.bin_pattern_bit(2, 4, 0)
    with pytest.raises(ValueError):
        rsr.SegmentedSums(2, np.zeros(3))


def test_tuner_matches_reference_values(rsr, tuner):
    for n, kpp, kr, mk in zip(tuner["n"], tuner["k_rsrpp"], tuner["k_rsr"], tuner["max_k"]):
        n = int(n)
        assert rsr.optimal_k_rsrpp(n) == kpp == rsr.optimal_k_rsrpp_bisect(n)
        assert rsr.optimal_k_rsr(n) == kr == rsr.optimal_k_rsr_bisect(n)
        assert rsr.max_k_for_rows(n) == mk
    assert [rsr.optimal_k_rsrpp(1 << e) for e in range(11, 17)] == [9, 9, 10, 11, 12, 13]


def test_variant_and_argument_errors_before_device_work(rsr):
    from paper_2411_06360_b200.kernels import _use_fold
    assert _use_fold("RSR++") and _use_fold("rsrpp") and not _use_fold("rsr")
    with pytest.raises(ValueError, match="variant"):
        _use_fold("fast")
    with pytest.raises(TypeError):
        rsr.preprocess(np.zeros((2, 2)), 1)
    with pytest.raises(TypeError):
        rsr.preprocess_ternary(np.zeros((2, 2)), 1)


def test_package_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2411_06360_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle-free", ""), f


def test_butterfly_schedule_roundtrip():
    """indexer.unschedule_codes inverts the device schedule format (csrc/common.cuh butterfly8,
    control bits 3c..3c+2 in bits 13-15 of code c of each 8-row group): 4096 distinct orders,
    and scheduling + unscheduling is the identity on row-order codes."""
    import numpy as np
    from paper_2411_06360_b200.indexer import _butterfly8, unschedule_codes
    ctrl = np.arange(4096, dtype=np.uint32)
    perms = _butterfly8(np.broadcast_to(np.arange(8), (4096, 8)), ctrl)
    assert len({tuple(p) for p in perms}) == 4096
    rng = np.random.default_rng(7)
    nb, rs, k = 3, 512, 11
    codes = (rng.integers(0, 1 << k, size=(nb, rs)) << 2).astype(np.uint32)   # swizzled key << 2
    g = codes.reshape(nb, rs // 8, 8)
    c = rng.integers(0, 4096, size=g.shape[:2]).astype(np.uint32)
    slots = _butterfly8(g, c)                       # slot s holds row p[s]
    for j in range(4):
        slots[..., j] |= ((c >> (3 * j)) & 7) << 13
    back = unschedule_codes(slots.reshape(nb, rs).astype(np.uint16), k)
    assert np.array_equal(back, codes.astype(np.uint16))


def test_b200_tuner_is_valid_for_every_row_count(rsr):
    """optimal_k_b200 (the device cost model) always returns a k the index accepts."""
    from paper_2411_06360_b200.indexer import max_k_for_rows
    for rows in (1, 2, 3, 6, 64, 1000, 4096, 14336, 16384, 65536, 1 << 20):
        k = rsr.optimal_k_b200(rows, 4096)
        assert 1 <= k <= max(1, max_k_for_rows(rows)) and k <= 16
    assert rsr.optimal_k_b200(16384, 16384) == rsr.optimal_k_rsrpp(16384) == 11  # headline unchanged
