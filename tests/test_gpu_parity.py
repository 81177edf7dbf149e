"""Parity of the sm_100a CUDA path against the oracle and the reference's golden vectors.

Bars: bit-exact for indices (perm / seg / keys) and for integer activations with
int32 accumulation; fp64 activations within the reference's own float test
tolerance (rtol = atol = 1e-9, test_kernels.py:269-280); fp32 activations within
||got - ref||_inf <= 1e-5 * max(||ref||_inf, 1) (north star, norm-wise).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import unpack_index
from oracle import c_oracle
from oracle import rsr_oracle as O

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


def _fp32_ok(got, ref):
    got = np.asarray(got, np.float64)
    scale = max(float(np.abs(ref).max(initial=0.0)), 1.0)
    return float(np.abs(got - ref).max(initial=0.0)) <= FP32_TOL * scale


def _dev_index_arrays(idx):
    perm, seg, bucket = idx.host_arrays()
    return perm, seg, bucket


# ----------------------------------------------------------------------------- worked example
def test_worked_example(rsr, cuda, worked):
    B = rsr.BinaryMatrix.from_dense(worked["B6"])
    idx = rsr.preprocess(B, 2)
    assert idx.block_count == 3 and (idx.rows, idx.cols, idx.k) == (6, 6, 2)
    assert np.array_equal(idx.blocks[0].permutation, [1, 4, 5, 0, 2, 3])
    assert np.array_equal(idx.blocks[0].segmentation, [0, 3, 5, 5])
    u = rsr.segmented_sum(worked["V6"], idx.blocks[0])
    assert np.array_equal(u.sums, [12.0, 7.0, 0.0, 5.0])
    assert np.array_equal(rsr.block_product_rsr(u), [5.0, 12.0])
    assert np.array_equal(rsr.block_product_rsrpp(u), [5.0, 12.0])
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(worked["B6"].astype(np.int8)), 2)
    for variant in ("rsr", "rsrpp", "rsr++"):
        assert np.array_equal(rsr.multiply_rsr(worked["V6"], idx, variant), worked["product_binary"])
        assert np.array_equal(rsr.multiply_ternary(worked["V6"], tidx, variant), worked["product_ternary"])
    for blk in tidx.negative.blocks:
        assert np.array_equal(blk.segmentation, [0, 6, 6, 6])
    assert np.array_equal(rsr.naive_multiply(worked["V6"], B), worked["naive"])
    assert rsr.reconstruct_matrix(idx) == B


# ----------------------------------------------------------------------------- golden fuzz
def test_preprocess_bitwise_vs_reference_golden(rsr, cuda, fuzz):
    for i in range(int(fuzz["count"])):
        p = f"c{i}_"
        A, k = fuzz[p + "A"], int(fuzz[p + "k"])
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        for half, pre in ((tidx.positive, "pos_"), (tidx.negative, "neg_")):
            rp, rs, rb = unpack_index(fuzz, p + pre)
            perm, seg, bucket = _dev_index_arrays(half)
            assert np.array_equal(perm, rp), (i, pre)
            assert np.array_equal(bucket, rb), (i, pre)
            for b, s in enumerate(rs):
                assert np.array_equal(seg[b, :len(s)], s), (i, pre, b)


def test_multiply_vs_reference_golden(rsr, cuda, fuzz):
    import torch
    for i in range(int(fuzz["count"])):
        p = f"c{i}_"
        A, k = fuzz[p + "A"], int(fuzz[p + "k"])
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        vi, vf = fuzz[p + "vi"], fuzz[p + "vf"]
        for variant in ("rsr", "rsrpp"):
            ref_i, ref_f = fuzz[p + f"int_{variant}"], fuzz[p + f"flt_{variant}"]
            # reference contract: NumPy fp64 in -> fp64 out (gather kernel in fp64)
            assert np.array_equal(rsr.multiply_ternary(vi, tidx, variant), ref_i)
            np.testing.assert_allclose(rsr.multiply_ternary(vf, tidx, variant), ref_f, rtol=1e-9, atol=1e-9)
            # integer NumPy input -> int32 scatter kernel, fp64 result
            assert np.array_equal(rsr.multiply_ternary(vi.astype(np.int64), tidx, variant), ref_i)
            # device tensors
            dvi = torch.from_numpy(vi.astype(np.int32)).cuda()
            got = rsr.multiply_ternary(dvi, tidx, variant)
            assert got.dtype == torch.int32 and np.array_equal(got.cpu().numpy(), ref_i)
            dvf = torch.from_numpy(vf.astype(np.float32)).cuda()
            ref32 = O.multiply_ternary(vf.astype(np.float32).astype(np.float64),
                                       unpack_index(fuzz, p + "pos_")[2], unpack_index(fuzz, p + "neg_")[2],
                                       A.shape[1], k, variant == "rsrpp")
            assert _fp32_ok(rsr.multiply_ternary(dvf, tidx, variant).cpu().numpy(), ref32)
            # deterministic int32 gather form agrees bitwise with the scatter form
            from paper_2411_06360_b200 import kernels as K, _native
            g = K._multiply_device(dvi, tidx, variant == "rsrpp", form=_native.FORM_GATHER)
            assert np.array_equal(g.cpu().numpy(), ref_i)
        assert np.array_equal(rsr.multiply_rsr(vi, tidx.positive, "rsrpp"), fuzz[p + "int_pos_rsrpp"])


def test_medium_shapes_vs_reference(rsr, cuda, medium):
    import torch
    for i in range(4):
        p = f"m{i}_"
        rows, cols = (int(x) for x in medium[p + "shape"])
        k = int(medium[p + "k"])
        rng = np.random.default_rng([2411, rows, cols])
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        v = rng.integers(-100, 101, size=rows).astype(np.float64)
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        for variant in ("rsrpp", "rsr"):
            dv = torch.from_numpy(v.astype(np.int32)).cuda()
            assert np.array_equal(rsr.multiply_ternary(dv, tidx, variant).cpu().numpy(), medium[p + variant])
            assert np.array_equal(rsr.multiply_ternary(v, tidx, variant), medium[p + variant])
        assert np.array_equal(rsr.naive_multiply(v, rsr.TernaryMatrix(A)), medium[p + "naive"])


# ----------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("rows,cols,k", [
    (1, 1, 1), (2, 1, 1), (3, 5, 1), (6, 6, 2), (9, 14, 3), (33, 65, 5), (64, 64, 6),
    (100, 7, 6), (257, 300, 8), (1000, 129, 7), (4097, 50, 12), (300, 70, 1),
])
def test_edge_shapes_all_forms(rsr, cuda, rows, cols, k):
    import torch
    from paper_2411_06360_b200 import kernels as K, _native
    rng = np.random.default_rng([rows, cols, k, 7])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    perm, seg, bucket = _dev_index_arrays(tidx.positive)
    assert np.array_equal(perm, pp) and np.array_equal(bucket, pb)
    for b, s in enumerate(ps):
        assert np.array_equal(seg[b, :len(s)], s)
    vi = rng.integers(-100, 101, size=rows)
    vf = rng.standard_normal(rows)
    for fold in (True, False):
        ref = c_oracle.multiply_parallel(vi.astype(np.float64), pb, nb, cols, k, fold, 1)
        dv = torch.from_numpy(vi.astype(np.int32)).cuda()
        for form in (_native.FORM_SCATTER, _native.FORM_GATHER):
            got = K._multiply_device(dv, tidx, fold, form=form).cpu().numpy()
            assert np.array_equal(got, ref), (form, fold)
        reff = c_oracle.multiply_parallel(vf, pb, nb, cols, k, fold, 1)
        np.testing.assert_allclose(rsr.multiply_ternary(vf, tidx, "rsrpp" if fold else "rsr"), reff,
                                   rtol=1e-9, atol=1e-9)


def test_zero_and_dense_extremes(rsr, cuda):
    import torch
    for A in (np.zeros((50, 23), np.int8), np.ones((50, 23), np.int8), -np.ones((50, 23), np.int8)):
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 4)
        v = np.arange(50, dtype=np.int32) - 25
        got = rsr.multiply_ternary(torch.from_numpy(v).cuda(), tidx).cpu().numpy()
        assert np.array_equal(got, v.astype(np.int64) @ A.astype(np.int64))
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(np.zeros((6, 3), np.int8)), 2)
    assert np.array_equal(tidx.positive.blocks[0].permutation, np.arange(6))
    assert np.array_equal(tidx.positive.blocks[0].segmentation, [0, 6, 6, 6])


def test_row_splits_and_large_k(rsr, cuda):
    """rows > 16384 exercises the multi-CTA row split (atomic output); k up to 15."""
    import torch
    for rows, cols, k in ((20000, 40, 11), (40000, 33, 15), (16385, 30, 13), (16384, 29, 14), (8192, 26, 12)):
        rng = np.random.default_rng([rows, cols])
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        v = rng.integers(-100, 101, size=rows).astype(np.int32)
        (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        perm, seg, bucket = _dev_index_arrays(tidx.negative)
        assert np.array_equal(perm, np_) and np.array_equal(bucket, nb)
        ref = v.astype(np.int64) @ A.astype(np.int64)
        for variant in ("rsrpp", "rsr"):
            got = rsr.multiply_ternary(torch.from_numpy(v).cuda(), tidx, variant).cpu().numpy()
            assert np.array_equal(got, ref), (rows, k, variant)
            got = rsr.multiply_ternary(v.astype(np.float64), tidx, variant)
            assert np.array_equal(got, ref)


def test_device_k_limit_and_errors(rsr, cuda):
    import torch
    A = rsr.TernaryMatrix(np.ones((6, 6), np.int8))
    with pytest.raises(ValueError):
        rsr.preprocess_ternary(A, 3)
    tidx = rsr.preprocess_ternary(A, 2)
    with pytest.raises(ValueError, match="does not match"):
        rsr.multiply_ternary(np.ones(5), tidx)
    with pytest.raises(ValueError):
        rsr.multiply_ternary(np.array([1.0, np.nan, 0, 0, 0, 0]), tidx)
    with pytest.raises(ValueError, match="variant"):
        rsr.multiply_ternary(np.ones(6), tidx, "fast")
    with pytest.raises(ValueError, match="worker_count"):
        rsr.multiply_parallel(np.ones(6), tidx, worker_count=0)
    with pytest.raises(ValueError, match="does not match"):
        rsr.multiply_ternary(torch.ones(5, dtype=torch.int32, device="cuda"), tidx)
    bad = torch.tensor([[1, 2], [0, 1]], dtype=torch.int8, device="cuda")
    with pytest.raises(ValueError, match="ternary entries"):
        rsr.preprocess_ternary(bad, 1)


def test_parallel_workers_bitwise_independent(rsr, cuda):
    rng = np.random.default_rng(107)
    n = 1 << 12
    for case in range(6):
        cols = int(rng.integers(512, 4097))
        A = rng.integers(-1, 2, size=(n, cols), dtype=np.int8)
        k = (8, 9, 10)[case % 3]
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        v = rng.integers(-100, 101, size=n) if case % 2 == 0 else rng.standard_normal(n)
        for variant in ("rsr", "rsrpp"):
            ref = rsr.multiply_ternary(v, tidx, variant)
            for workers in (1, 2, 4, 8, 32):
                got = rsr.multiply_parallel(v, tidx, variant, worker_count=workers)
                assert got.tobytes() == ref.tobytes()


def test_conservation_of_block_sums(rsr, cuda):
    rng = np.random.default_rng(108)
    for _ in range(10):
        rows, cols = int(rng.integers(2, 129)), int(rng.integers(1, 129))
        B = rsr.BinaryMatrix.from_dense(rng.integers(0, 2, size=(rows, cols), dtype=np.uint8))
        v = rng.integers(-100, 101, size=rows).astype(np.float64)
        for k in range(1, min(6, rsr.max_k_for_rows(rows)) + 1):
            for blk in rsr.preprocess(B, k).blocks:
                assert rsr.segmented_sum(v, blk).sums.sum() == v.sum()


def test_binary_preprocess_and_row_order(rsr, cuda):
    rng = np.random.default_rng(1)
    dense = rng.integers(0, 2, size=(64, 20), dtype=np.uint8)
    B = rsr.BinaryMatrix.from_dense(dense)
    perms, segs, buckets = O.preprocess_binary(dense, 3)
    idx = rsr.preprocess(B, 3)
    perm, seg, bucket = idx.host_arrays()
    assert np.array_equal(perm, perms) and np.array_equal(bucket, buckets)
    assert np.array_equal(rsr.binary_row_order(B, (0, 3)), perms[0])
    assert np.array_equal(rsr.full_segmentation(B, (0, 3), perms[0]), segs[0][:-1])
    with pytest.raises(ValueError):
        rsr.full_segmentation(B, (0, 3), np.arange(64))
    for k in range(1, 7):
        assert rsr.reconstruct_matrix(rsr.preprocess(B, k)) == B


def test_from_blocks_round_trip_and_validation(rsr, cuda, worked):
    B = rsr.BinaryMatrix.from_dense(worked["B6"])
    idx = rsr.preprocess(B, 2)
    blocks = [rsr.BlockIndex(b.width, b.permutation.copy(), b.segmentation.copy()) for b in idx.blocks]
    rebuilt = rsr.RsrIndex.from_blocks(6, 6, 2, blocks)
    assert rebuilt == idx
    assert np.array_equal(rsr.multiply_rsr(worked["V6"], rebuilt), worked["product_binary"])
    blocks[0].permutation[0] = blocks[0].permutation[1]
    with pytest.raises(ValueError, match="bijection"):
        rsr.RsrIndex.from_blocks(6, 6, 2, blocks)


def test_block_products_bitwise(rsr, cuda, folds):
    for w in range(1, 11):
        for tag in ("i", "f"):
            u = rsr.SegmentedSums(w, folds[f"w{w}{tag}_u"])
            assert rsr.block_product_rsrpp(u).tobytes() == folds[f"w{w}{tag}_rsrpp"].tobytes()
            assert rsr.block_product_rsr(u).tobytes() == folds[f"w{w}{tag}_rsr"].tobytes()


def test_fp32_fixed_point_scatter_deterministic(rsr, cuda):
    """fp32 activations on the scatter kernel (exact two-limb fixed-point accumulation):
    within the north-star tolerance of the fp64 oracle and bitwise reproducible."""
    import torch
    from paper_2411_06360_b200 import kernels as K, _native
    for rows, cols, k in ((300, 77, 6), (4096, 1000, 9), (16384, 400, 11), (5000, 64, 12)):
        rng = np.random.default_rng([rows, cols, 32])
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        vf = (rng.standard_normal(rows) * 3).astype(np.float32)
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        ref = vf.astype(np.float64) @ A.astype(np.float64)
        dv = torch.from_numpy(vf).cuda()
        a = K._multiply_device(dv, tidx, True, form=_native.FORM_SCATTER).cpu().numpy()
        b = K._multiply_device(dv, tidx, True, form=_native.FORM_SCATTER).cpu().numpy()
        assert a.tobytes() == b.tobytes()
        assert _fp32_ok(a, ref), float(np.abs(a - ref).max())
        g = K._multiply_device(dv, tidx, False, form=_native.FORM_GATHER).cpu().numpy()
        assert _fp32_ok(g, ref)
        auto = rsr.multiply_ternary(dv, tidx).cpu().numpy()
        assert _fp32_ok(auto, ref)


@pytest.mark.parametrize("rows,cols,k,batch", [
    (300, 77, 6, 5), (1000, 333, 2, 33), (4096, 1000, 9, 64), (2000, 130, 1, 1),
    (16384, 600, 11, 64), (5000, 257, 12, 100), (70000, 40, 8, 3),
])
def test_batched_matches_per_vector(rsr, cuda, rows, cols, k, batch):
    """multiply_batched (csrc/batched.cu, gather form over V^T) == the reference per-vector
    multiply for every row of V: bitwise for int32 (both variants, ternary and binary), within
    the fp32 bar for float32; covers short last blocks, k < 3 (warps with empty bucket
    ranges), batches across the 32/64/128-vector slice widths and u32 perms (rows > 65536)."""
    import torch
    rng = np.random.default_rng([rows, cols, k, batch])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    Vi = rng.integers(-100, 101, size=(batch, rows)).astype(np.int32)
    kp = c_oracle.keys_ternary(A, k, 1)
    kn = c_oracle.keys_ternary(A, k, -1)
    for variant in ("rsrpp", "rsr"):
        got = rsr.multiply_batched(torch.from_numpy(Vi).cuda(), tidx, variant).cpu().numpy()
        for i in range(batch):
            ref = c_oracle.multiply_parallel(Vi[i].astype(np.float64), kp, kn, cols, k, True, 1)
            assert np.array_equal(got[i].astype(np.float64), ref), (variant, i)
    Vf = (rng.standard_normal((batch, rows)) * 2).astype(np.float32)
    gotf = rsr.multiply_batched(torch.from_numpy(Vf).cuda(), tidx).cpu().numpy()
    again = rsr.multiply_batched(torch.from_numpy(Vf).cuda(), tidx).cpu().numpy()
    assert gotf.tobytes() == again.tobytes()  # deterministic
    reff = Vf.astype(np.float64) @ A.astype(np.float64)
    for i in range(batch):
        assert _fp32_ok(gotf[i], reff[i]), i
    # binary index (one half)
    B = (A == 1).astype(np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
    gotb = rsr.multiply_batched(torch.from_numpy(Vi).cuda(), bidx).cpu().numpy()
    refb = Vi.astype(np.int64) @ B.astype(np.int64)
    assert np.array_equal(gotb.astype(np.int64), refb)


def test_rsx_load_golden(rsr, cuda):
    """Reference-written .rsx files load into the device layout and multiply to the
    reference's products; invariant corruptions raise the reference's messages; our writer
    reproduces the reference's file byte for byte from a GPU-preprocessed index."""
    import json
    import os
    import torch
    rsx = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rsx")
    prods = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rsx_products.npz"))
    tidx = rsr.load_index(os.path.join(rsx, "ternary_200x77_k5.rsx"))
    bidx = rsr.load_index(os.path.join(rsx, "binary_90x33_k4.rsx"))
    assert isinstance(tidx, rsr.TernaryIndex) and isinstance(bidx, rsr.RsrIndex)
    assert np.array_equal(rsr.multiply_ternary(prods["ternary_v"], tidx), prods["ternary_y"])
    assert np.array_equal(rsr.multiply_rsr(prods["binary_v"], bidx), prods["binary_y"])
    # device int32 path too (scheduled keys rebuilt on the device)
    got = rsr.multiply_ternary(torch.from_numpy(prods["ternary_v"].astype(np.int32)).cuda(), tidx)
    assert np.array_equal(got.cpu().numpy().astype(np.float64), prods["ternary_y"])
    verdicts = json.load(open(os.path.join(rsx, "verdicts.json")))
    for name in ("perm_duplicate", "perm_range", "seg_start", "seg_order", "t_pos5_neg2", "t_neg3"):
        with pytest.raises(rsr.FormatError) as exc:
            rsr.load_index(os.path.join(rsx, f"corrupt_{name}.rsx"))
        assert str(exc.value) == verdicts[name], name
    # same matrices as tests/golden/make_golden.py rsx_files(): our preprocess + save == reference file
    rng = np.random.default_rng(2024)
    A = rng.integers(-1, 2, size=(200, 77), dtype=np.int8)
    B = rng.integers(0, 2, size=(90, 33)).astype(np.uint8)
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        rsr.save_index(rsr.preprocess_ternary(rsr.TernaryMatrix(A), 5), os.path.join(tmp, "t.rsx"))
        rsr.save_index(rsr.preprocess(rsr.BinaryMatrix.from_dense(B), 4), os.path.join(tmp, "b.rsx"))
        assert open(os.path.join(tmp, "t.rsx"), "rb").read() == open(os.path.join(rsx, "ternary_200x77_k5.rsx"), "rb").read()
        assert open(os.path.join(tmp, "b.rsx"), "rb").read() == open(os.path.join(rsx, "binary_90x33_k4.rsx"), "rb").read()
        # round trip at a size with u16 perms, scheduled keys and a short last block
        A2 = np.random.default_rng(5).integers(-1, 2, size=(4096, 1000), dtype=np.int8)
        i2 = rsr.preprocess_ternary(torch.from_numpy(A2).cuda(), 9)
        rsr.save_index(i2, os.path.join(tmp, "r.rsx"))
        back = rsr.load_index(os.path.join(tmp, "r.rsx"))
        v2 = torch.from_numpy(np.random.default_rng(6).integers(-100, 101, 4096).astype(np.int32)).cuda()
        assert torch.equal(rsr.multiply_ternary(v2, back), rsr.multiply_ternary(v2, i2))
        assert all(np.array_equal(a, b) for a, b in zip(back.positive.host_arrays(), i2.positive.host_arrays()))


def test_bitlinear_decode_chain_graph(rsr, cuda):
    """BitLinear layers on the Llama-3-8B MLP shapes (up 4096->14336, down 14336->4096) chained
    on the device and captured in one CUDA graph: fp32 within the north-star tolerance of a
    dense fp64 reference, int32 bit-exact; graph replay reproduces eager results."""
    import torch
    rng = np.random.default_rng(11)
    Wu = rng.integers(-1, 2, size=(4096, 14336), dtype=np.int8)
    Wd = rng.integers(-1, 2, size=(14336, 4096), dtype=np.int8)
    up = rsr.BitLinear(torch.from_numpy(Wu).cuda())
    down = rsr.BitLinear(torch.from_numpy(Wd).cuda())
    assert (up.k, down.k) == (rsr.optimal_k_b200(4096, 14336), rsr.optimal_k_b200(14336, 4096))
    x = torch.from_numpy(rng.standard_normal(4096).astype(np.float32)).cuda()
    y = down(up(x) * 0.01)
    h = (x.cpu().double().numpy() @ Wu.astype(np.float64)).astype(np.float32).astype(np.float64) * 0.01
    ref = h.astype(np.float32).astype(np.float64) @ Wd.astype(np.float64)
    assert _fp32_ok(y.cpu().numpy(), ref), float(np.abs(y.cpu().numpy() - ref).max())
    xi = torch.from_numpy(rng.integers(-8, 9, 4096).astype(np.int32)).cuda()
    yi = down(up(xi) // 64)
    hi = (xi.cpu().numpy().astype(np.int64) @ Wu.astype(np.int64)) // 64
    assert np.array_equal(yi.cpu().numpy().astype(np.int64), hi @ Wd.astype(np.int64))
    # capture the chain in one graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        yg = down(up(x) * 0.01)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, y)


@pytest.mark.parametrize("rows,cols", [(1, 1), (33, 7), (1000, 333), (4096, 4096), (2500, 1030)])
def test_dense_standard_gemv(rsr, cuda, rows, cols):
    """The dense 2-bit GPU GEMV (the paper's standard multiply, csrc/dense.cu) equals the
    reference's naive_multiply (C port, core.py:135-143): int32 bitwise, fp32 within the bar."""
    import torch
    rng = np.random.default_rng([rows, cols, 77])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    D = rsr.DenseTernary(A)
    vi = rng.integers(-100, 101, rows).astype(np.int32)
    ref = c_oracle.naive_ternary(vi.astype(np.float64), A)
    got = D.multiply(torch.from_numpy(vi).cuda()).cpu().numpy()
    assert np.array_equal(got.astype(np.float64), ref)
    vf = rng.standard_normal(rows).astype(np.float32)
    reff = vf.astype(np.float64) @ A.astype(np.float64)
    assert _fp32_ok(D.multiply(torch.from_numpy(vf).cuda()).cpu().numpy(), reff)
    with pytest.raises(ValueError):
        rsr.DenseTernary(np.full((4, 4), 2, np.int8))


def test_counted_twins_vs_reference(rsr, cuda):
    """Instrumented twins (reference kernels.py:240-320): products bitwise equal to the
    reference's counted twin and the same accumulate counts (n + 2*2^w - 2 per block for
    RSR++, n + w*2^w for RSR)."""
    import os
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "counted.npz"))
    for i in range(3):
        B, k, v = d[f"c{i}_B"], int(d[f"c{i}_k"]), d[f"c{i}_v"]
        idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
        for variant in ("rsr", "rsrpp"):
            y, total = rsr.multiply_counted(v, idx, variant)
            assert y.tobytes() == d[f"c{i}_{variant}_y"].tobytes(), (i, variant)
            assert total == int(d[f"c{i}_{variant}_total"])
        sums, adds = rsr.segmented_sum_counted(v, idx.blocks[0])
        assert sums.sums.tobytes() == d[f"c{i}_seg0_sums"].tobytes() and adds == int(d[f"c{i}_seg0_adds"])
        for name, fn in (("rsr", rsr.block_product_rsr_counted), ("rsrpp", rsr.block_product_rsrpp_counted)):
            prod, adds = fn(sums)
            assert prod.tobytes() == d[f"c{i}_bp0_{name}"].tobytes() and adds == int(d[f"c{i}_bp0_{name}_adds"])


# ----------------------------------------------------------------------------- host-buffer sessions
@pytest.mark.parametrize("rows,cols,k", [(1, 1, 1), (37, 29, 3), (1000, 777, 8), (16384, 1001, 11),
                                         (20000, 515, 12), (2048, 8193, 10), (512, 12001, 9)])
def test_host_session_all_types(rsr, cuda, rows, cols, k):
    """NumPy in -> fresh fp64 NumPy out through the host session (rows <= 16384: one launch that
    pulls v from mapped memory and streams seq-tagged results back; rows > 16384 and fp64 /
    wide kinds: H2D, multiply, D2H): int32 / int64 bit-exact, fp32 within the north-star bound,
    fp64 within the reference's float tolerance; repeated calls reuse the session."""
    rng = np.random.default_rng([rows, cols, k])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    for trial in range(3):
        vi = rng.integers(-100, 101, size=rows)
        ref = c_oracle.naive_ternary(vi.astype(np.float64), A)
        for v in (vi.astype(np.int32), vi.astype(np.int64)):
            got = rsr.multiply_ternary(v, idx)
            assert got.dtype == np.float64 and got.shape == (cols,)
            assert np.array_equal(got, ref)
        vf = rng.standard_normal(rows)
        reff = c_oracle.naive_ternary(vf.astype(np.float32).astype(np.float64), A)
        assert _fp32_ok(rsr.multiply_ternary(vf.astype(np.float32), idx), reff)
        ref64 = c_oracle.naive_ternary(vf, A)
        np.testing.assert_allclose(rsr.multiply_ternary(vf, idx), ref64, rtol=1e-9, atol=1e-9)
        a = rsr.multiply_ternary(vi.astype(np.int32), idx, "rsr")
        assert np.array_equal(a, ref)
        assert a is not rsr.multiply_ternary(vi.astype(np.int32), idx)  # fresh arrays


def test_host_session_threads_and_errors(rsr, cuda):
    """One session per thread: concurrent host-buffer multiplies give the single-thread
    results; bad lengths raise the reference's ValueError."""
    import threading
    rng = np.random.default_rng(7)
    A = rng.integers(-1, 2, size=(4096, 4096), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 9)
    vs = [rng.integers(-100, 101, size=4096).astype(np.int32) for _ in range(4)]
    refs = [c_oracle.naive_ternary(v.astype(np.float64), A) for v in vs]
    errors = []

    def work(i):
        try:
            for _ in range(50):
                if not np.array_equal(rsr.multiply_ternary(vs[i], idx), refs[i]):
                    errors.append(i)
                    return
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    with pytest.raises(ValueError, match="does not match"):
        rsr.multiply_ternary(vs[0][:100], idx)


def test_host_session_concurrent_streams(rsr, cuda):
    """Sessions on four non-blocking streams at once, each launch a full 148-CTA grid that pulls
    its vector from mapped memory (csrc/multiply.cu pull_payload): kernels that cannot all be
    resident together must neither deadlock nor mix payloads (a CTA whose peers are not running
    copies the payload itself); int32 and fp32 launches interleave on every session."""
    import threading
    import torch
    rng = np.random.default_rng(11)
    rows, cols = 16384, 2048
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 11)
    vs = [rng.integers(-100, 101, size=rows).astype(np.int32) for _ in range(4)]
    refs = [c_oracle.naive_ternary(v.astype(np.float64), A) for v in vs]
    vf = [rng.standard_normal(rows).astype(np.float32) for _ in range(4)]
    reff = [c_oracle.naive_ternary(v.astype(np.float64), A) for v in vf]
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for it in range(40):
                    if it % 3 == 2:
                        if not _fp32_ok(rsr.multiply_ternary(vf[i], idx), reff[i]):
                            errors.append(("fp32", i, it))
                            return
                    elif not np.array_equal(rsr.multiply_ternary(vs[i], idx), refs[i]):
                        errors.append(("int32", i, it))
                        return
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors


@pytest.mark.parametrize("rows,cols,k,batch,vmax", [
    (64, 5, 5, 2, 511),        # one full bin: 64 * 511 = 32704, at the int16 edge (packed)
    (64, 5, 5, 3, 512),        # 64 * 512 = 32768: the guard refuses, per-vector path
    (1003, 37, 6, 5, 100),     # ragged rows / last block, odd batch (one unpaired vector)
    (16384, 600, 11, 8, 100),  # the headline block width, full CTAs
    (4096, 333, 10, 6, 2**31 - 1),
])
def test_batched_packed_pairs(rsr, cuda, rows, cols, k, batch, vmax):
    """The int32 batched loop runs two vectors per scatter launch (v + v' * 2^16 per
    reduction) when max bucket load * max |v| <= 32767 (csrc/capi.cu, multiply.cu PACK):
    results must equal the reference per vector on both sides of that guard."""
    import torch
    rng = np.random.default_rng([rows, cols, k, batch, vmax])
    if rows == 64:
        A = np.ones((rows, cols), dtype=np.int8)  # every row in logical bin 2^k - 1
        Vi = np.full((batch, rows), vmax, dtype=np.int32)
        Vi[1::2] = -vmax
    else:
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        Vi = rng.integers(-vmax, vmax, size=(batch, rows), endpoint=True, dtype=np.int64).astype(np.int32)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    for variant in ("rsrpp", "rsr"):
        got = rsr.multiply_batched(torch.from_numpy(Vi).cuda(), tidx, variant).cpu().numpy()
        for i in range(batch):
            one = rsr.multiply_ternary(torch.from_numpy(Vi[i].copy()).cuda(), tidx, variant).cpu().numpy()
            assert np.array_equal(got[i], one), (variant, i)
        if vmax <= 512:
            ref = (Vi.astype(np.int64) @ A.astype(np.int64))
            assert np.array_equal(got.astype(np.int64), ref), variant
    B = (A == 1).astype(np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
    gotb = rsr.multiply_batched(torch.from_numpy(Vi).cuda(), bidx).cpu().numpy()
    refb = (Vi.astype(np.int64) @ B.astype(np.int64))
    assert np.array_equal(gotb.astype(np.int64), (refb + 2**31) % 2**32 - 2**31)


def test_batched_under_graph_capture(rsr, cuda):
    """Inside CUDA graph capture the int32 batched call must not synchronise (the packed-pair
    guard needs a host read): it falls back to per-vector launches, with the same results."""
    import torch
    rng = np.random.default_rng(7)
    A = rng.integers(-1, 2, size=(2048, 300), dtype=np.int8)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 10)
    V = torch.from_numpy(rng.integers(-100, 101, size=(6, 2048)).astype(np.int32)).cuda()
    eager = rsr.multiply_batched(V, tidx)  # packed pairs (guard passes), also warms the workspace
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        captured = rsr.multiply_batched(V, tidx)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(captured, eager)
    ref = V.cpu().numpy().astype(np.int64) @ A.astype(np.int64)
    assert np.array_equal(eager.cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("rows,cols,k,batch,vmax", [
    (300, 77, 5, 3, 100),        # one plan block pass, odd batch
    (1003, 37, 6, 70, 100),      # two 64-vector slices, ragged rows and last plan block
    (16384, 600, 11, 64, 100),   # the headline split (16384 rows), split slots in every unit
    (16384, 601, 11, 64, 300),   # |v| > 127: the int32-lane form (32 vectors per pass)
    (20000, 515, 12, 7, 100),    # two row splits (atomic output)
    (4096, 333, 10, 130, 2**31 - 1),  # int32-range values: wraps like every int32 path
    (1000, 3096, 9, 64, 100),    # 172 passes on 148 CTAs: remainder passes split 6 ways by rows
])
def test_batch_plan_kernel(rsr, cuda, rows, cols, k, batch, vmax):
    """The batch-native kernel (csrc/batch_lanes.cu: lanes span 64 vectors, re-cut 9-wide plan
    blocks with split slots) against exact int64 products (mod 2^32) and against the
    per-vector path, for both variants and binary indexes; the plan is built once and kept."""
    import torch
    from paper_2411_06360_b200 import kernels as K
    rng = np.random.default_rng([rows, cols, k, batch, vmax % 1000])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    V = rng.integers(-vmax, vmax, size=(batch, rows), endpoint=True, dtype=np.int64).astype(np.int32)
    idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
    wrap = lambda x: ((x + 2**31) % 2**32) - 2**31  # noqa: E731
    ref = wrap(V.astype(np.int64) @ A.astype(np.int64))
    dV = torch.from_numpy(V).cuda()
    for variant in ("rsrpp", "rsr"):
        got = rsr.multiply_batched(dV, idx, variant).cpu().numpy()
        assert idx._bplan, "the batch plan applies here"
        assert np.array_equal(got.astype(np.int64), ref), variant
    K._PLAN_OFF = True
    try:
        old = rsr.multiply_batched(dV, idx).cpu().numpy()
    finally:
        K._PLAN_OFF = False
    assert np.array_equal(old, rsr.multiply_batched(dV, idx).cpu().numpy())
    B = (A == 1).astype(np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
    gotb = rsr.multiply_batched(dV, bidx).cpu().numpy()
    assert np.array_equal(gotb.astype(np.int64), wrap(V.astype(np.int64) @ B.astype(np.int64)))


@pytest.mark.parametrize("rows,cols", [(1, 1), (17, 5), (300, 77), (1000, 513), (4096, 4100)])
def test_dense_i8_comparator(rsr, cuda, rows, cols):
    """The IDP4A dense comparator (csrc/dense.cu dense_gemv_i8_kernel, 2-bit fields shifted to
    the top of their byte) is exact for int8 activations, ragged shapes included."""
    import torch
    rng = np.random.default_rng([rows, cols, 8])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    v = rng.integers(-128, 128, size=rows).astype(np.int8)
    d = rsr.DenseTernary(torch.from_numpy(A).cuda())
    got = d.multiply_i8(torch.from_numpy(v).cuda()).cpu().numpy()
    assert np.array_equal(got.astype(np.int64), v.astype(np.int64) @ A.astype(np.int64))


def test_seeded_fuzz_every_entry_point(rsr, cuda):
    """40 seeded random shapes (rows 1..2500, cols 1..1500, every admissible k up to the device
    limit, ternary and binary) through every public entry point — host int32 / int64 / fp64-integer
    vectors (session: int32 kernel or wide multiply), device int32 / int64 tensors, block-range
    multiply_parallel, the batch kernel — each bitwise against the C oracle's exact products."""
    import torch
    rng = np.random.default_rng(20241106)
    for case in range(40):
        rows = int(rng.integers(1, 2501))
        cols = int(rng.integers(1, 1501))
        k = int(rng.integers(1, min(16, rsr.max_k_for_rows(rows)) + 1))
        ternary = bool(case % 4 != 3)
        A = rng.integers(-1 if ternary else 0, 2, size=(rows, cols), dtype=np.int8)
        big = case % 5 == 0  # sums beyond int32: the exact wide multiply
        v = rng.integers(-(2 ** 30) if big else -100, (2 ** 30) if big else 101, size=rows, dtype=np.int64)
        M = A.astype(object) if big else A.astype(np.int64)
        exact = np.array([int(x) for x in (v.astype(object) @ M)] if big else v @ M, dtype=object if big else np.int64)
        ref = np.array([float(x) for x in exact])
        if ternary:
            idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
            mult = rsr.multiply_ternary
        else:
            idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(A.astype(np.uint8)), k)
            mult = rsr.multiply_rsr
        forms = [v, v.astype(np.float64)] + ([] if big else [v.astype(np.int32)])
        for form in forms:
            assert np.array_equal(mult(form, idx), ref), (case, rows, cols, k, form.dtype)
        assert np.array_equal(rsr.multiply_parallel(v, idx, "rsrpp", int(rng.integers(1, 6))), ref), case
        dev64 = mult(torch.from_numpy(v).cuda(), idx).cpu().numpy()
        assert [int(x) for x in dev64] == [int(x) for x in exact], case
        if not big:
            dev32 = mult(torch.from_numpy(v.astype(np.int32)).cuda(), idx, "rsr").cpu().numpy()
            assert np.array_equal(dev32.astype(np.int64), exact), case
            B = int(rng.integers(2, 70))
            V = rng.integers(-100, 101, size=(B, rows)).astype(np.int32)
            got = rsr.multiply_batched(torch.from_numpy(V).cuda(), idx).cpu().numpy()
            assert np.array_equal(got.astype(np.int64), V.astype(np.int64) @ A.astype(np.int64)), case


def test_fused_bitlinear_matches_separate_layers(rsr, cuda):
    """FusedBitLinear (one index over [W_gate | W_up], blocks straddling the two layers) gives each
    layer's output bitwise equal to the separate BitLinear, single vectors and batches."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(11)
    Wg = (torch.randint(0, 3, (1024, 1500), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
    Wu = (torch.randint(0, 3, (1024, 1333), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
    fused = rsr.FusedBitLinear([Wg, Wu])
    sep = [rsr.BitLinear(Wg), rsr.BitLinear(Wu)]
    x = torch.randint(-100, 101, (1024,), device="cuda", generator=g).to(torch.int32)
    X = torch.randint(-100, 101, (9, 1024), device="cuda", generator=g).to(torch.int32)
    for inp in (x, X):
        for a, b in zip(fused(inp), (s(inp) for s in sep)):
            assert torch.equal(a, b)
    with pytest.raises(ValueError):
        rsr.FusedBitLinear([Wg, Wu[:1000]])


def test_host_session_pull_steal_path(cuda):
    """The pull's fallback (csrc/multiply.cu pull_payload): with the chunk wait forced to 0 ns
    every CTA copies the whole payload itself instead of waiting for its peers' chunks — results
    must be identical (run in a fresh process: the knob is read once)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, "REPO")
import paper_2411_06360_b200 as rsr
from oracle import c_oracle
rng = np.random.default_rng(5)
for rows, cols, k in ((16384, 1500, 11), (4096, 4096, 10), (3000, 77, 6)):
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    for it in range(4):
        v = rng.integers(-100, 101, size=rows)
        ref = c_oracle.naive_ternary(v.astype(np.float64), A)
        assert np.array_equal(rsr.multiply_ternary(v.astype(np.float64), idx), ref), (rows, it)
        vf = rng.standard_normal(rows).astype(np.float32)
        reff = c_oracle.naive_ternary(vf.astype(np.float64), A)
        got = rsr.multiply_ternary(vf, idx)
        assert np.abs(got - reff).max() <= 1e-5 * max(1.0, np.abs(reff).max()), (rows, it)
print("steal ok")
'''.replace("REPO", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, RSR_B200_PULL_STEAL_NS="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "steal ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("rows,cols,k", [(16384, 3000, 11), (4096, 4096, 10), (3000, 77, 6), (20000, 500, 9)])
def test_independent_launches_keep_stream_order(rsr, cuda, rows, cols, k):
    """RSR_MULTIPLY_INDEPENDENT (rsr_multiply_ex): a launch starts reducing before the previous
    one has finished, but its writes to out still wait for it.  Long streams of independent
    launches — alternating indexes and vectors, several writing the SAME output buffer right
    after a dependent launch into it, ternary and binary, int32 and fp32 — must give exactly the
    dependent results, eagerly and replayed from a CUDA graph."""
    import torch
    from paper_2411_06360_b200 import kernels as K
    rng = np.random.default_rng([rows, cols, k, 77])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idxs = [rsr.preprocess_ternary(rsr.TernaryMatrix(A), k),
            rsr.preprocess_ternary(rsr.TernaryMatrix(A[:, ::-1].copy()), k)]
    Ab = rng.integers(0, 2, size=(rows, cols), dtype=np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(Ab), k)
    vs = [rng.integers(-100, 101, size=rows).astype(np.int32) for _ in range(3)]
    dvs = [torch.from_numpy(v).cuda() for v in vs]
    refs = {(i, j): c_oracle.naive_ternary(vs[j].astype(np.float64), A if i == 0 else A[:, ::-1].copy())
            for i in range(2) for j in range(3)}
    shared = torch.empty(cols, dtype=torch.int32, device="cuda")
    outs = [torch.empty(cols, dtype=torch.int32, device="cuda") for _ in range(4)]

    def stream_of_launches():
        K._multiply_device(dvs[0], idxs[0], True, None, shared)  # dependent, then independents into it
        for t in range(24):
            i, j = t % 2, t % 3
            K._multiply_device(dvs[j], idxs[i], t % 4 != 3, None, outs[t % 4], independent=True)
            if t % 5 == 4:
                K._multiply_device(dvs[j], idxs[i], True, None, shared, independent=True)
        t_sh = max(t for t in range(24) if t % 5 == 4)  # the last launch into `shared`
        return [(t % 2, t % 3) for t in range(20, 24)], (t_sh % 2, t_sh % 3)

    last, sh = stream_of_launches()
    torch.cuda.synchronize()
    for t, (i, j) in zip(range(20, 24), last):
        assert np.array_equal(outs[t % 4].cpu().numpy().astype(np.float64), refs[(i, j)]), ("eager", t)
    assert np.array_equal(shared.cpu().numpy().astype(np.float64), refs[sh])
    # the same stream captured once and replayed
    for o in outs + [shared]:
        o.fill_(-7)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        stream_of_launches()
    torch.cuda.current_stream().wait_stream(cap)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for t, (i, j) in zip(range(20, 24), last):
        assert np.array_equal(outs[t % 4].cpu().numpy().astype(np.float64), refs[(i, j)]), ("graph", t)
    # binary and fp32 forms
    refb = vs[1].astype(np.float64) @ Ab.astype(np.float64)
    vf = rng.standard_normal(rows).astype(np.float32)
    reff = vf.astype(np.float64) @ A.astype(np.float64)
    dvf = torch.from_numpy(vf).cuda()
    ob = [K._multiply_device(dvs[1], bidx, t % 2 == 0, independent=True) for t in range(6)]
    of = [K._multiply_device(dvf, idxs[0], True, independent=True) for t in range(6)]
    torch.cuda.synchronize()
    for x in ob:
        assert np.array_equal(x.cpu().numpy().astype(np.float64), refb)
    if rows <= 16384:
        for x in of:
            assert _fp32_ok(x.cpu().numpy(), reff)


def test_multiply_ex_flags(rsr, cuda):
    """rsr_multiply_ex rejects unknown flags with RSR_ERR_INVALID (and leaves out untouched)."""
    import ctypes
    import torch
    from paper_2411_06360_b200 import _native
    A = np.random.default_rng(3).integers(-1, 2, size=(64, 20), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 4)
    dv = torch.ones(64, dtype=torch.int32, device="cuda")
    out = torch.full((20,), 5, dtype=torch.int32, device="cuda")
    L = _native.lib()
    st = L.rsr_multiply_ex(ctypes.byref(idx.desc), dv.data_ptr(), _native.I32, out.data_ptr(), _native.I32,
                           _native.VARIANT_RSRPP, _native.FORM_AUTO, 0, idx.desc.nblocks, 6,
                           _native.current_stream_ptr())
    assert st != 0 and b"flags" in L.rsr_b200_last_error()
    st = L.rsr_multiply_ex(ctypes.byref(idx.desc), dv.data_ptr(), _native.I32, out.data_ptr(), _native.I32,
                           _native.VARIANT_RSRPP, _native.FORM_AUTO, 0, idx.desc.nblocks,
                           _native.MULTIPLY_INDEPENDENT, _native.current_stream_ptr())
    assert st == 0
    assert np.array_equal(out.cpu().numpy().astype(np.float64), np.ones(64) @ A.astype(np.float64))
