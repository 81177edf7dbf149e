"""The binding a maintainer of the REFERENCE package would add to `rsr/kernels.py` to run its
hot path on the B200 library (INTEGRATION.md §2 quotes this file).  Plain ctypes against
include/rsr_b200.h — no torch, no import of the drop-in package.  The reference keeps its own
validation (`_use_fold` kernels.py:17-21, `as_vector` core.py:110-117); the index object only
needs `rows`, `cols` and `_device_desc` (an rsr_index_desc filled once by
rsr_preprocess_ternary or rsr_index_import) plus `_d_v` / `_d_out` device scratch of
rows / cols doubles for the one-shot entry point.

tests/test_integration_stub.py drives every function here on the GPU.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB = os.environ.get("RSR_B200_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2411_06360_b200", "lib", "librsr_b200.so")
_lib = ctypes.CDLL(LIB)


class _Half(ctypes.Structure):
    _fields_ = [("perm", ctypes.c_void_p), ("seg", ctypes.c_void_p), ("bucket", ctypes.c_void_p)]


class _Desc(ctypes.Structure):  # rsr_index_desc
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("k", ctypes.c_int32),
                ("nblocks", ctypes.c_int32), ("perm_bytes", ctypes.c_int32), ("halves", ctypes.c_int32),
                ("row_stride", ctypes.c_int64), ("seg_stride", ctypes.c_int64), ("half", _Half * 2)]


RSR_I32, RSR_F32, RSR_F64, RSR_I64 = 0, 1, 2, 3
_CODES = {np.dtype(np.int32): RSR_I32, np.dtype(np.int64): RSR_I64, np.dtype(np.float32): RSR_F32,
          np.dtype(np.float64): RSR_F64}
P, SZ = ctypes.c_void_p, ctypes.c_size_t
_lib.rsr_b200_last_error.restype = ctypes.c_char_p
_lib.rsr_multiply_host.argtypes = [ctypes.POINTER(_Desc), P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, P, P]
_lib.rsr_host_session_create.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(P)]
_lib.rsr_host_session_multiply.argtypes = [P, P, ctypes.c_int, SZ, P, ctypes.c_int, SZ, ctypes.c_int, P]
_lib.rsr_host_session_destroy.argtypes = [P]


def _raise(st):
    if st:
        raise ValueError(_lib.rsr_b200_last_error().decode())


def multiply_ternary_oneshot(v, idx, use_fold: bool) -> np.ndarray:
    """In place of `_run_index` x 2 + `pos - neg` (kernels.py:196-206): one C call does H2D,
    the fused multiply and D2H (rsr_multiply_host).  v is the reference's validated fp64
    vector; the fp64 gather kernel computes it."""
    out = np.empty(idx.cols, np.float64)
    _raise(_lib.rsr_multiply_host(ctypes.byref(idx._device_desc), v.ctypes.data, RSR_F64, out.ctypes.data,
                                  RSR_F64, int(use_fold), idx._d_v, idx._d_out, None))
    return out


class Session:
    """The inference-loop binding: one host-buffer session per index (mapped staging the
    kernel pulls v from, device scratch, mapped tagged results), reused every call.  It classifies v while staging it, so integer-
    valued vectors (int32 / int64 / fp64 holding integers) are exact (int32 kernel when
    sum |v| fits, the wide multiply otherwise)."""

    def __init__(self, idx):
        self.cols = idx.cols
        self.h = P()
        _raise(_lib.rsr_host_session_create(ctypes.byref(idx._device_desc), ctypes.byref(self.h)))

    def multiply(self, v: np.ndarray, use_fold: bool) -> np.ndarray:
        v = np.ascontiguousarray(v)
        out = np.empty(self.cols, np.float64)  # fresh fp64 result, like the reference
        _raise(_lib.rsr_host_session_multiply(self.h, v.ctypes.data, _CODES[v.dtype], v.nbytes, out.ctypes.data,
                                              RSR_F64, out.nbytes, int(use_fold), None))
        return out

    def close(self):
        if self.h:
            _lib.rsr_host_session_destroy(self.h)
            self.h = P()
