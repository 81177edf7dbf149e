"""ctypes binding of the C ABI in include/rsr_b200.h (librsr_b200.so).

The library is the product: every multiply / preprocess call goes through it.
There is no CPU fallback — if the library (or a CUDA device) is missing, the
call raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSR_B200_LIB") or os.path.join(_HERE, "lib", "librsr_b200.so")  # override: A/B builds

RSR_OK, RSR_ERR_INVALID, RSR_ERR_UNSUPPORTED, RSR_ERR_CUDA = 0, 1, 2, 3
I32, F32, F64, I64 = 0, 1, 2, 3
VARIANT_RSR, VARIANT_RSRPP = 0, 1
FORM_AUTO, FORM_SCATTER, FORM_GATHER = 0, 1, 2

ABI_VERSION = 3
MULTIPLY_INDEPENDENT = 1  # rsr_multiply_ex flag (include/rsr_b200.h)

# Every symbol include/rsr_b200.h declares (tests check the .so exports them all).
EXPORTS = (
    "rsr_b200_abi_version", "rsr_b200_last_error", "rsr_index_layout",
    "rsr_preprocess_workspace_bytes", "rsr_preprocess_ternary", "rsr_preprocess_binary",
    "rsr_index_import_workspace_bytes", "rsr_index_import",
    "rsr_multiply", "rsr_multiply_ex", "rsr_multiply_wide_workspace_bytes", "rsr_multiply_wide", "rsr_multiply_batched_workspace_bytes", "rsr_multiply_batched", "rsr_multiply_host",
    "rsr_host_session_create", "rsr_host_session_destroy", "rsr_host_session_multiply", "rsr_segmented_sum",
    "rsr_block_product", "rsr_naive_multiply_ternary",
    "rsr_dense_plane_words", "rsr_dense_pack_ternary", "rsr_dense_multiply",
    "rsr_dense_i8_words", "rsr_dense_pack_ternary_i8", "rsr_dense_multiply_i8",
    "rsr_batch_plan_layout", "rsr_batch_plan_build", "rsr_multiply_batched_plan_workspace_bytes",
    "rsr_multiply_batched_plan", "rsr_multiply_allgather", "rsr_allgather_wait", "rsr_multiply_fixed",
)


class HalfIndex(ctypes.Structure):
    _fields_ = [("perm", ctypes.c_void_p), ("seg", ctypes.c_void_p), ("bucket", ctypes.c_void_p)]


class IndexDesc(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("k", ctypes.c_int32), ("nblocks", ctypes.c_int32),
        ("perm_bytes", ctypes.c_int32), ("halves", ctypes.c_int32),
        ("row_stride", ctypes.c_int64), ("seg_stride", ctypes.c_int64),
        ("half", HalfIndex * 2),
    ]


class BatchPlan(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("kb", ctypes.c_int32), ("nblocks", ctypes.c_int32), ("halves", ctypes.c_int32),
        ("split_rows", ctypes.c_int32), ("nsplits", ctypes.c_int32), ("extra_cap", ctypes.c_int32),
        ("extra", ctypes.c_int32), ("vmax", ctypes.c_int32), ("row_stride", ctypes.c_int64),
        ("codes", ctypes.c_void_p), ("slot_bins", ctypes.c_void_p),
    ]


class NativeError(RuntimeError):
    """A CUDA-side failure inside librsr_b200.so."""


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"librsr_b200.so not found at {LIB_PATH}; build it with `make` "
            "(or __graft_entry__.build()). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32_, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    st = ctypes.c_int
    L.rsr_b200_abi_version.restype = ctypes.c_int
    L.rsr_b200_last_error.restype = ctypes.c_char_p
    L.rsr_index_layout.argtypes = [I64, I64, I32_, I32_, ctypes.POINTER(IndexDesc),
                                   ctypes.POINTER(SZ), ctypes.POINTER(SZ), ctypes.POINTER(SZ)]
    L.rsr_index_layout.restype = st
    L.rsr_preprocess_workspace_bytes.argtypes = [ctypes.POINTER(IndexDesc)]
    L.rsr_preprocess_workspace_bytes.restype = SZ
    L.rsr_preprocess_ternary.argtypes = [P, I64, ctypes.POINTER(IndexDesc), P, P, SZ, P]
    L.rsr_preprocess_ternary.restype = st
    L.rsr_preprocess_binary.argtypes = [P, I64, ctypes.POINTER(IndexDesc), P, SZ, P]
    L.rsr_preprocess_binary.restype = st
    L.rsr_multiply.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_int, P, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, I32_, I32_, P]
    L.rsr_multiply.restype = st
    if hasattr(L, "rsr_multiply_ex") or not os.environ.get("RSR_B200_LIB"):  # (A/B builds may predate it)
        L.rsr_multiply_ex.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_int, P, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, I32_, I32_, ctypes.c_uint32, P]
        L.rsr_multiply_ex.restype = st
    if hasattr(L, "rsr_multiply_fixed") or not os.environ.get("RSR_B200_LIB"):  # (A/B builds may predate it)
        L.rsr_multiply_fixed.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_uint64, ctypes.c_int32, P,
                                         ctypes.c_int, I32_, I32_, P, SZ, P]
        L.rsr_multiply_fixed.restype = st
    if hasattr(L, "rsr_multiply_allgather") or not os.environ.get("RSR_B200_LIB"):  # (A/B builds may predate it)
        L.rsr_multiply_allgather.argtypes = [ctypes.POINTER(IndexDesc), P, P, ctypes.c_int, P, P, ctypes.c_int32,
                                             ctypes.c_int64, P, P]
        L.rsr_multiply_allgather.restype = st
        L.rsr_allgather_wait.argtypes = [P, ctypes.c_uint64, P]
        L.rsr_allgather_wait.restype = st
    L.rsr_multiply_wide_workspace_bytes.argtypes = [ctypes.POINTER(IndexDesc), ctypes.c_uint64]
    L.rsr_multiply_wide_workspace_bytes.restype = SZ
    L.rsr_multiply_wide.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_uint64, P, ctypes.c_int, ctypes.c_int,
                                    I32_, I32_, P, SZ, P]
    L.rsr_multiply_wide.restype = st
    L.rsr_index_import_workspace_bytes.argtypes = [ctypes.POINTER(IndexDesc)]
    L.rsr_index_import_workspace_bytes.restype = SZ
    L.rsr_index_import.argtypes = [ctypes.POINTER(IndexDesc), P, P, P, P, I64, P, SZ, P, P]
    L.rsr_index_import.restype = st
    L.rsr_multiply_batched_workspace_bytes.argtypes = [ctypes.POINTER(IndexDesc), I64, ctypes.c_int]
    L.rsr_multiply_batched_workspace_bytes.restype = SZ
    L.rsr_multiply_batched.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_int, I64, P,
                                       ctypes.c_int, ctypes.c_int, P, SZ, P]
    L.rsr_multiply_batched.restype = st
    L.rsr_multiply_host.argtypes = [ctypes.POINTER(IndexDesc), P, ctypes.c_int, P, ctypes.c_int,
                                    ctypes.c_int, P, P, P]
    L.rsr_multiply_host.restype = st
    L.rsr_host_session_create.argtypes = [ctypes.POINTER(IndexDesc), ctypes.POINTER(P)]
    L.rsr_host_session_create.restype = st
    L.rsr_host_session_destroy.argtypes = [P]
    L.rsr_host_session_destroy.restype = None
    L.rsr_host_session_multiply.argtypes = [P, P, ctypes.c_int, SZ, P, ctypes.c_int, SZ, ctypes.c_int, P]
    L.rsr_host_session_multiply.restype = st
    L.rsr_segmented_sum.argtypes = [ctypes.POINTER(IndexDesc), I32_, I32_, P, ctypes.c_int, P, P]
    L.rsr_segmented_sum.restype = st
    L.rsr_block_product.argtypes = [P, I32_, ctypes.c_int, P, P, P]
    L.rsr_block_product.restype = st
    L.rsr_dense_plane_words.argtypes = [I64, I64]
    L.rsr_dense_plane_words.restype = SZ
    L.rsr_dense_pack_ternary.argtypes = [P, I64, I64, I64, P, P, P, P]
    L.rsr_dense_pack_ternary.restype = st
    L.rsr_dense_multiply.argtypes = [P, P, I64, I64, P, ctypes.c_int, P, P]
    L.rsr_dense_multiply.restype = st
    L.rsr_dense_i8_words.argtypes = [I64, I64]
    L.rsr_dense_i8_words.restype = SZ
    L.rsr_dense_pack_ternary_i8.argtypes = [P, I64, I64, I64, P, P, P]
    L.rsr_dense_pack_ternary_i8.restype = st
    L.rsr_dense_multiply_i8.argtypes = [P, I64, I64, P, P, P]
    L.rsr_dense_multiply_i8.restype = st
    L.rsr_naive_multiply_ternary.argtypes = [P, I64, I64, I64, P, ctypes.c_int, P, P]
    L.rsr_naive_multiply_ternary.restype = st
    L.rsr_batch_plan_layout.argtypes = [ctypes.POINTER(IndexDesc), ctypes.POINTER(BatchPlan), ctypes.POINTER(SZ),
                                        ctypes.POINTER(SZ), ctypes.POINTER(SZ)]
    L.rsr_batch_plan_layout.restype = st
    L.rsr_batch_plan_build.argtypes = [ctypes.POINTER(IndexDesc), ctypes.POINTER(BatchPlan), P, SZ, P]
    L.rsr_batch_plan_build.restype = st
    L.rsr_multiply_batched_plan_workspace_bytes.argtypes = [ctypes.POINTER(BatchPlan), I64]
    L.rsr_multiply_batched_plan_workspace_bytes.restype = SZ
    L.rsr_multiply_batched_plan.argtypes = [ctypes.POINTER(IndexDesc), ctypes.POINTER(BatchPlan), P, I64, P,
                                            ctypes.c_int, P, SZ, P]
    L.rsr_multiply_batched_plan.restype = st
    if L.rsr_b200_abi_version() != ABI_VERSION:
        raise ImportError("librsr_b200.so ABI version mismatch; rebuild with `make`")
    _lib = L
    return _lib


_ext = None
EXT_PATH = None


def host_ext():
    """The CPython binding of rsr_host_session_multiply (csrc/pyhost.c -> lib/_rsrhost*.so):
    buffer-protocol arguments and the GIL released while the call waits on the GPU."""
    global _ext, EXT_PATH
    if _ext is not None:
        return _ext
    import importlib.machinery
    import importlib.util
    lib()  # the extension links librsr_b200.so; load (and version-check) it first
    for suffix in importlib.machinery.EXTENSION_SUFFIXES:
        path = os.path.join(_HERE, "lib", "_rsrhost" + suffix)
        if os.path.exists(path):
            spec = importlib.util.spec_from_file_location("_rsrhost", path)
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            _ext, EXT_PATH = mod, path
            return _ext
    raise ImportError(f"_rsrhost extension not found under {os.path.join(_HERE, 'lib')}; build it with `make`")


def check(status: int) -> None:
    """Map an rsr_status to the reference's exception types."""
    if status == RSR_OK:
        return
    msg = (lib().rsr_b200_last_error() or b"").decode()
    if status in (RSR_ERR_INVALID, RSR_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise NativeError(msg)


def layout(rows: int, cols: int, k: int, halves: int):
    desc = IndexDesc()
    pb, sb, bb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    check(lib().rsr_index_layout(rows, cols, k, halves, ctypes.byref(desc),
                                 ctypes.byref(pb), ctypes.byref(sb), ctypes.byref(bb)))
    return desc, pb.value, sb.value, bb.value


def current_stream_ptr() -> int:
    """cudaStream_t of torch's current stream on the current device (kernels are enqueued
    there, like a torch op).  Uses the raw query (sub-microsecond) when available."""
    import torch
    try:
        return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
    except AttributeError:  # pragma: no cover
        return torch.cuda.current_stream().cuda_stream
