"""INTEGRATION.md's reference-side binding (integration/rsr_b200_binding.py), driven end to end:
the ctypes stub a reference maintainer would add, against an index the C ABI built, with
results checked against the C oracle (the reference's algorithm)."""

from __future__ import annotations

import ctypes
import importlib.util
import os

import numpy as np
import pytest

from conftest import ROOT


def _stub():
    spec = importlib.util.spec_from_file_location("rsr_b200_binding",
                                                  os.path.join(ROOT, "integration", "rsr_b200_binding.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_stub_loads_and_declares_the_header_signatures():
    """CPU: the stub binds the library without a GPU and its structs match the header's."""
    from paper_2411_06360_b200 import _native
    stub = _stub()
    assert ctypes.sizeof(stub._Desc) == ctypes.sizeof(_native.IndexDesc)
    assert [f[0] for f in stub._Desc._fields_] == [f[0] for f in _native.IndexDesc._fields_]


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k", [(300, 77, 5), (4096, 1000, 9), (16384, 515, 11)])
def test_stub_end_to_end(rsr, cuda, rows, cols, k):
    import torch
    from oracle import c_oracle
    stub = _stub()
    rng = np.random.default_rng([rows, cols, k, 9])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    tidx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)  # rsr_preprocess_ternary underneath

    class Idx:  # what the reference's index object would carry
        pass
    idx = Idx()
    idx.rows, idx.cols = rows, cols
    idx._device_desc = stub._Desc.from_buffer_copy(tidx.desc)
    d_v = torch.empty(rows, dtype=torch.float64, device="cuda")
    d_out = torch.empty(cols, dtype=torch.float64, device="cuda")
    idx._d_v, idx._d_out = d_v.data_ptr(), d_out.data_ptr()
    (pp, ps, pb), (np_, ns, nb) = c_oracle.preprocess_ternary(A, k)
    torch.cuda.synchronize()
    for fold in (True, False):
        vi = rng.integers(-100, 101, size=rows).astype(np.float64)
        ref = c_oracle.multiply_parallel(vi, pb, nb, cols, k, fold, 1)
        one = stub.multiply_ternary_oneshot(vi, idx, fold)
        np.testing.assert_allclose(one, ref, rtol=1e-12, atol=1e-9)
        s = stub.Session(idx)
        for v in (vi, vi.astype(np.int32), vi.astype(np.int64), vi * 2 ** 22):
            want = c_oracle.multiply_parallel(np.asarray(v, np.float64), pb, nb, cols, k, fold, 1)
            assert np.array_equal(s.multiply(v, fold), want), v.dtype
        vf = rng.standard_normal(rows)
        np.testing.assert_allclose(s.multiply(vf, fold), c_oracle.multiply_parallel(vf, pb, nb, cols, k, fold, 1),
                                   rtol=1e-9, atol=1e-9 * np.abs(vf).sum())
        with pytest.raises(ValueError, match="finite"):
            bad = vf.copy()
            bad[rows // 2] = np.nan
            s.multiply(bad, fold)
        s.close()


def _build_c_example(tmp_path):
    """integration/c_example.c: a plain-C consumer of include/rsr_b200.h (what a C / cgo / JNI
    binding calls), compiled and linked against the library like INTEGRATION.md says."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:  # pragma: no cover
        pytest.skip("gcc unavailable")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe = str(tmp_path / "c_example")
    lib = os.path.join(ROOT, "paper_2411_06360_b200", "lib")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
           os.path.join(ROOT, "integration", "c_example.c"), "-L", lib, "-lrsr_b200", "-L", f"{cuda}/lib64", "-lcudart",
           f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{cuda}/lib64", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    """CPU: the header is valid C11 and the library resolves every symbol the C example uses."""
    assert os.path.exists(_build_c_example(tmp_path))


@pytest.mark.gpu
def test_c_consumer_runs(cuda, tmp_path):
    """GPU: the C example preprocesses, multiplies through a host session and checks every
    column against its own naive product (bit-exact)."""
    import subprocess
    exe = _build_c_example(tmp_path)
    for args in ([], ["16384", "1001", "11"]):
        r = subprocess.run([exe] + args, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "c_example ok" in r.stdout, r.stdout + r.stderr
