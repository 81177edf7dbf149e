"""Inference: segmented sums, block products and the fused multiply, on the GPU.

Mirrors the reference `rsr.kernels` (kernels.py:1-239): same names, argument
meanings, validation order and error messages.  Every multiply runs the sm_100a
kernels in librsr_b200.so (see csrc/multiply.cu):

* NumPy / list input keeps the reference contract (any real vector in, fresh fp64
  out).  One host-buffer session call per multiply (rsr_host_session_multiply,
  csrc/host.cu) stages v into pinned memory and classifies it in the same pass
  (csrc/host_stage.cpp): integer-valued vectors (int32 / int64 / float64 holding
  integers) run on the int32 scatter kernel when sum |v| <= 2^31 - 1 — bit-exact —
  and on the exact wide multiply otherwise (csrc/wide.cu, limbs + int128
  recombination), so the result equals the reference's fp64 result wherever that
  one is exact; float32 vectors run in fp32 (exact fixed point);
  non-integer float64 vectors run as an exact int64 fixed-point product rounded
  once (>= 8192 rows, dynamic range <= 2^21) or on the fp64 gather kernel.
* torch CUDA tensors stay on the device: int32 -> int32 (scatter kernel, int32
  arithmetic modulo 2^32), int64 -> int64 (wide multiply, exact modulo 2^64),
  float32 -> float32, float64 -> float64 (gather kernel).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import as_vector
from .indexer import BlockIndex, RsrIndex, TernaryIndex, column_blocks

_VARIANTS = {"rsr": False, "rsrpp": True, "rsr++": True}


def _use_fold(variant: str) -> bool:
    """kernels.py:17-21."""
    try:
        return _VARIANTS[str(variant).lower()]
    except KeyError:
        raise ValueError(f"variant must be rsr or rsrpp, got {variant!r}") from None


@dataclass(eq=False)
class SegmentedSums:
    """Per-bucket sums u of one block; length is exactly 2^width (kernels.py:24-34)."""

    width: int
    sums: np.ndarray

    def __post_init__(self):
        self.sums = np.ascontiguousarray(self.sums, np.float64)
        if self.width < 1 or self.sums.shape != (1 << self.width,):
            raise ValueError(f"sums length must be 2^{self.width}")


def bin_pattern_bit(width: int, row: int, col: int) -> int:
    """Bit col (0 = most significant) of row's width-bit binary expansion (kernels.py:37-43)."""
    if not 0 <= row < (1 << width):
        raise ValueError(f"row {row} out of range for width {width}")
    if not 0 <= col < width:
        raise ValueError(f"col {col} out of range for width {width}")
    return (row >> (width - 1 - col)) & 1


# ---------------------------------------------------------------------------
# per-block operations
# ---------------------------------------------------------------------------

def segmented_sum(v, block: BlockIndex) -> SegmentedSums:
    """Per-bucket sums: sums[j] = sum of v[perm[p]] over segment j, ascending p
    (kernels.py:94-101), computed on the GPU (rsr_segmented_sum)."""
    import torch
    v = as_vector(v)
    if v.shape[0] != block.permutation.shape[0]:
        raise ValueError(f"vector length {v.shape[0]} does not match {block.permutation.shape[0]} rows")
    if block._src is not None:
        idx, b = block._src
    else:  # a free-standing block: upload it as a one-block index
        idx = RsrIndex.from_blocks(block.permutation.shape[0], block.width, block.width, [block])
        b = 0
    dv = torch.from_numpy(v).cuda()
    u = torch.empty(1 << block.width, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().rsr_segmented_sum(
        ctypes.byref(idx.desc), 0, b, dv.data_ptr(), _native.F64, u.data_ptr(), _native.current_stream_ptr()))
    return SegmentedSums(block.width, u.cpu().numpy())


def _block_product(u: SegmentedSums, fold: bool) -> np.ndarray:
    import torch
    du = torch.from_numpy(u.sums).cuda()
    buf = torch.empty(max(1, (1 << u.width) >> 1), dtype=torch.float64, device="cuda")
    out = torch.empty(u.width, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().rsr_block_product(
        du.data_ptr(), u.width, _native.VARIANT_RSRPP if fold else _native.VARIANT_RSR,
        buf.data_ptr(), out.data_ptr(), _native.current_stream_ptr()))
    return out.cpu().numpy()


def block_product_rsr(u: SegmentedSums) -> np.ndarray:
    """Product of u against the implicit Bin pattern, one column at a time (kernels.py:104-108)."""
    return _block_product(u, False)


def block_product_rsrpp(u: SegmentedSums) -> np.ndarray:
    """Same value via the odd-sum / pairwise-compaction fold (kernels.py:111-116)."""
    return _block_product(u, True)


# ---------------------------------------------------------------------------
# instrumented twins (kernels.py:240-320): the same per-block device ops, plus the number of
# accumulate steps the reference's loops perform — an audit of the work bound
# n + 2*2^w - 2 per block (RSR++) / n + w*2^w (RSR)
# ---------------------------------------------------------------------------

def segmented_sum_counted(v, block: BlockIndex):
    """(segmented_sum, adds): one accumulate per sorted position (kernels.py:244-262)."""
    sums = segmented_sum(v, block)
    return sums, int(block.permutation.shape[0])


def block_product_rsr_counted(u: SegmentedSums):
    """(block_product_rsr, width * 2^width) (kernels.py:265-277)."""
    return block_product_rsr(u), u.width * (1 << u.width)


def block_product_rsrpp_counted(u: SegmentedSums):
    """(block_product_rsrpp, 2 * 2^width - 2) (kernels.py:280-302)."""
    return block_product_rsrpp(u), 2 * (1 << u.width) - 2


def multiply_counted(v, idx: RsrIndex, variant: str = "rsrpp"):
    """Multiply via the per-block ops, returning (product, total accumulate count)
    (kernels.py:305-320); bitwise equal to the reference's counted twin."""
    use_fold = _use_fold(variant)
    out = np.empty(idx.cols, np.float64)
    total = 0
    for (start, _), blk in zip(column_blocks(idx.cols, idx.k), idx.blocks):
        sums, adds = segmented_sum_counted(v, blk)
        total += adds
        product, adds = block_product_rsrpp_counted(sums) if use_fold else block_product_rsr_counted(sums)
        total += adds
        out[start:start + blk.width] = product
    return out, total


# ---------------------------------------------------------------------------
# fused multiply
# ---------------------------------------------------------------------------

_DTYPES = {}


def _torch_dtype_code(t) -> int:
    import torch
    if not _DTYPES:
        _DTYPES.update({torch.int32: _native.I32, torch.float32: _native.F32, torch.float64: _native.F64,
                        torch.int64: _native.I64})
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ValueError("device vectors must be int32, int64, float32 or float64") from None


class _HostStaging(threading.local):
    """Per-thread device scratch and host-buffer sessions.  Thread-local: concurrent multiplies
    from several threads never share buffers."""

    def __init__(self):
        self.bufs = {}
        self.plans = {}  # id(index) -> (weakref to the index, _HostPlan); no strong refs


_staging = _HostStaging()
_HOST_CODES = {np.dtype(np.int32): _native.I32, np.dtype(np.int64): _native.I64,
               np.dtype(np.float32): _native.F32, np.dtype(np.float64): _native.F64}
_I32_MAX = 2 ** 31 - 1


class _HostPlan:
    """One host-buffer session (rsr_host_session_*: mapped staging the kernel pulls v from,
    device scratch, mapped seq-tagged result words) for one index and thread, created on first
    use and destroyed with the index or the thread."""
    __slots__ = ("session", "cols", "call", "stream", "__weakref__")

    def __init__(self, idx):
        import torch
        L = _native.lib()
        h = ctypes.c_void_p()
        _native.check(L.rsr_host_session_create(ctypes.byref(idx.desc), ctypes.byref(h)))
        self.session = h.value
        self.cols = idx.cols
        self.call = _native.host_ext().multiply
        # torch's current stream on the session's device, queried per call (sub-microsecond)
        dev = torch.cuda.current_device()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        self.stream = (lambda: raw(dev)) if raw is not None else _native.current_stream_ptr
        weakref.finalize(self, L.rsr_host_session_destroy, h.value)


def _host_plan(idx) -> _HostPlan:
    plans = _staging.plans
    ent = plans.get(id(idx))
    if ent is None or ent[0]() is not idx:
        key = id(idx)
        ent = plans[key] = (weakref.ref(idx, lambda _r, k=key, d=plans: d.pop(k, None)), _HostPlan(idx))
    return ent[1]


def _host_vector(v_in) -> np.ndarray:
    """The vector as a C-contiguous 1-D int32 / int64 / float32 / float64 array with the
    reference's value (`as_vector`, core.py:110-117, casts everything to float64: narrower
    integer types widen losslessly; anything else takes that cast)."""
    raw = v_in if type(v_in) is np.ndarray else np.asarray(v_in)
    dt = raw.dtype
    if dt in _HOST_CODES:
        arr = raw
    elif dt.kind == "b" or (dt.kind in "iu" and dt.itemsize < 4):  # bool, (u)int8, (u)int16
        arr = raw.astype(np.int32)
    elif dt == np.uint32 or (dt == np.uint64 and raw.size and int(raw.max()) < 2 ** 63):
        arr = raw.astype(np.int64)
    else:
        arr = as_vector(raw)  # the reference's own cast and checks (float16, uint64 >= 2^63, ...)
    if arr.ndim != 1 or arr.shape[0] < 1:
        raise ValueError("vector must be 1-D with at least one entry")
    return arr if arr.flags.c_contiguous else np.ascontiguousarray(arr)


def _check_finite(arr: np.ndarray) -> None:
    if arr.dtype.kind == "f" and not np.isfinite(arr).all():
        raise ValueError("vector entries must be finite")


def _check_length(arr: np.ndarray, rows: int) -> None:
    if arr.shape[0] != rows:
        _check_finite(arr)  # as_vector validates before the length check (kernels.py:188-190)
        raise ValueError(f"vector length {arr.shape[0]} does not match {rows} rows")


class _Class(tuple):
    """(kind, array, max_abs), plus .exp2 for the fixed-point class."""
    exp2 = 0


def _cls(kind, arr, mx, exp2=0):
    c = _Class((kind, arr, mx))
    c.exp2 = exp2
    return c


_FIXED_RANGE = 2.0 ** 21  # max / min nonzero |v| for the fixed-point class (host_stage.cpp)
_FIXED_MIN_ROWS = 8192   # below it the fp64 gather kernel is faster (host_stage.cpp kFixedMinRows)


def classify_host_vector(arr: np.ndarray):
    """(kind, array, max_abs): the computation csrc/host_stage.cpp picks for a host vector,
    restated in NumPy for the paths that do not use a session (multiply_parallel).
    kind "i32": integer-valued with sum |v| <= 2^31 - 1 (int32 kernel, bit-exact);
    "wide": other integer-valued vectors with |v| < 2^63 (exact wide multiply);
    "fixed": non-integer float64 with >= 8192 rows and max / min nonzero |v| <= 2^21, as the int64 fixed point
    round(v * 2^exp2) with |v_q| < 2^62 (`.exp2`; exact integer product, rounded once);
    "f32": float32; "f64": other float64 (the fp64 gather kernel)."""
    if arr.dtype == np.float32:
        _check_finite(arr)
        return _cls("f32", arr, 0)
    if arr.dtype.kind == "f":
        _check_finite(arr)
        if not ((np.abs(arr) < 2.0 ** 63).all() and (arr == np.trunc(arr)).all()):
            a = np.abs(arr)
            amax = float(a.max())
            nz = a[a > 0]
            if arr.size >= _FIXED_MIN_ROWS and amax > 0 and amax <= float(nz.min()) * _FIXED_RANGE:
                e = 61 - (int(np.frexp(amax)[1]) - 1)  # amax * 2^e < 2^62 (ilogb(amax) = frexp exponent - 1)
                q = np.rint(np.ldexp(arr.astype(np.float64), e)).astype(np.int64)
                return _cls("fixed", q, int(np.abs(q).max()), e)
            return _cls("f64", arr, 0)
        arr = arr.astype(np.int64)
    mx = max(abs(int(arr.min())), abs(int(arr.max())))
    total = float(np.abs(arr.astype(np.float64)).sum())  # exact for sums below 2^53
    if total <= _I32_MAX:
        return _cls("i32", arr.astype(np.int32), mx)
    return _cls("wide", arr.astype(np.int64), mx)


def _run_host(idx, arr: np.ndarray, use_fold: bool) -> np.ndarray:
    """One session call: host vector (int32 / int64 / float32 / float64) -> fresh fp64 result
    (the reference's result type)."""
    plan = _host_plan(idx)
    out = np.empty(plan.cols, np.float64)
    st = plan.call(plan.session, arr, _HOST_CODES[arr.dtype], out, _native.F64,
                   _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR, plan.stream())
    if st:
        _native.check(st)
    return out


def _wide_workspace(idx, max_abs: int, device):
    import torch
    nbytes = _native.lib().rsr_multiply_wide_workspace_bytes(ctypes.byref(idx.desc), max_abs)
    return torch.empty(max(1, (nbytes + 7) // 8), dtype=torch.int64, device=device), nbytes


def _multiply_device(v, idx, use_fold: bool, block_range=None, out=None, form=_native.FORM_AUTO, max_abs: int = 0,
                     exp2: int = 0, independent: bool = False):
    """Device-tensor path: v CUDA tensor [rows] -> CUDA tensor [cols].  exp2 != 0: v is the int64
    fixed point round(v * 2^exp2) of a float64 vector (classify_host_vector), result fp64.
    independent: the caller guarantees no kernel still in flight on the stream writes v, so the
    launch starts reducing on the SMs the previous launch has freed (rsr_multiply_ex flag
    RSR_MULTIPLY_INDEPENDENT; out still waits for the previous launch)."""
    import torch
    code = _torch_dtype_code(v)
    if v.dim() != 1 or v.shape[0] < 1:
        raise ValueError("vector must be 1-D with at least one entry")
    if v.shape[0] != idx.rows:
        raise ValueError(f"vector length {v.shape[0]} does not match {idx.rows} rows")
    v = v.contiguous()
    if out is None:
        out = torch.empty(idx.cols, dtype=v.dtype, device=v.device)
    b0, b1 = block_range if block_range is not None else (0, idx.desc.nblocks)
    variant = _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR
    if code == _native.I64 and exp2:  # fixed-point fp64: exact integer product, rounded once, scaled
        ws, nbytes = _wide_workspace(idx, max_abs, v.device)
        _native.check(_native.lib().rsr_multiply_fixed(
            ctypes.byref(idx.desc), v.data_ptr(), max_abs, exp2, out.data_ptr(), variant, b0, b1,
            ws.data_ptr(), nbytes, _native.current_stream_ptr()))
        return out
    if code == _native.I64:  # exact wide multiply (limbs through the int32 kernel)
        ws, nbytes = _wide_workspace(idx, max_abs, v.device)
        _native.check(_native.lib().rsr_multiply_wide(
            ctypes.byref(idx.desc), v.data_ptr(), max_abs, out.data_ptr(), _torch_dtype_code(out), variant, b0, b1,
            ws.data_ptr(), nbytes, _native.current_stream_ptr()))
        return out
    if independent:
        _native.check(_native.lib().rsr_multiply_ex(
            ctypes.byref(idx.desc), v.data_ptr(), code, out.data_ptr(), _torch_dtype_code(out),
            variant, form, b0, b1, _native.MULTIPLY_INDEPENDENT, _native.current_stream_ptr()))
        return out
    _native.check(_native.lib().rsr_multiply(
        ctypes.byref(idx.desc), v.data_ptr(), code, out.data_ptr(), _torch_dtype_code(out),
        variant, form, b0, b1, _native.current_stream_ptr()))
    return out


def _multiply_host(v_in, idx, use_fold: bool, compute: str | None) -> np.ndarray:
    """Host-buffer path (reference contract): NumPy in, fresh fp64 NumPy out, via one
    host-buffer session call (stage + classify, one pulling / publishing launch or H2D +
    multiply + D2H, result)."""
    arr = _host_vector(v_in)
    _check_length(arr, idx.rows)
    if compute is None:
        return _run_host(idx, arr, use_fold)
    if compute == "float32":
        _check_finite(arr)
        return _run_host(idx, arr.astype(np.float32), use_fold)
    if compute == "int32":
        kind, vv, _ = classify_host_vector(arr)
        if kind != "i32":
            raise ValueError("compute='int32' needs integer-valued activations with sum |v| <= 2^31 - 1")
        return _run_host(idx, vv, use_fold)
    if compute == "float64":  # the fp64 gather kernel, no integer routing
        import torch
        _check_finite(arr)
        dv = torch.from_numpy(np.ascontiguousarray(arr, np.float64)).cuda()
        return _multiply_device(dv, idx, use_fold).cpu().numpy()
    raise ValueError("compute must be int32, float32 or float64 for host vectors")


def _is_device_tensor(v) -> bool:
    if type(v) is np.ndarray:  # the common host case, without touching torch
        return False
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor) and v.is_cuda


def multiply_rsr(v, idx: RsrIndex, variant: str = "rsrpp", *, compute: str | None = None):
    """v times the indexed binary matrix; block results concatenated in order (kernels.py:185-193)."""
    use_fold = _use_fold(variant)
    if _is_device_tensor(v):
        return _multiply_device(v, idx, use_fold)
    return _multiply_host(v, idx, use_fold, compute)


def multiply_ternary(v, idx: TernaryIndex, variant: str = "rsrpp", *, compute: str | None = None):
    """v times the indexed ternary matrix: positive-half product minus negative-half
    (kernels.py:196-206), fused into one launch."""
    use_fold = _use_fold(variant)
    if _is_device_tensor(v):
        return _multiply_device(v, idx, use_fold)
    return _multiply_host(v, idx, use_fold, compute)


def multiply_parallel(v, idx, variant: str = "rsrpp", worker_count: int = 1, *, compute: str | None = None):
    """Blocks partitioned across workers, each writing a disjoint output slice
    (kernels.py:209-239).  Each worker's block range [i*nb//W, (i+1)*nb//W) is one
    block-range launch on the current stream (the same partition the multi-GPU
    path shards across ranks); the result is bitwise independent of W.  Host vectors
    take the same exact routing as multiply_ternary (classify_host_vector)."""
    import torch
    use_fold = _use_fold(variant)
    if worker_count < 1:
        raise ValueError("worker_count must be at least 1")
    nb = idx.desc.nblocks
    bounds = [i * nb // worker_count for i in range(worker_count + 1)]
    ranges = [(lo, hi) for lo, hi in zip(bounds, bounds[1:]) if lo < hi]
    if _is_device_tensor(v):
        if v.shape[0] != idx.rows:
            raise ValueError(f"vector length {v.shape[0]} does not match {idx.rows} rows")
        out = torch.empty(idx.cols, dtype=v.dtype, device=v.device)
        for r in ranges:
            _multiply_device(v, idx, use_fold, r, out)
        return out
    arr = _host_vector(v)
    _check_length(arr, idx.rows)
    if compute == "float32":
        kind, vv, mx = "f32", arr.astype(np.float32), 0
    elif compute == "float64":
        _check_finite(arr)
        kind, vv, mx = "f64", arr.astype(np.float64), 0
    elif compute in (None, "int32"):
        cls = classify_host_vector(arr)
        kind, vv, mx = cls
        if compute == "int32" and kind != "i32":
            raise ValueError("compute='int32' needs integer-valued activations with sum |v| <= 2^31 - 1")
    else:
        raise ValueError("compute must be int32, float32 or float64 for host vectors")
    dv = torch.from_numpy(vv).cuda()
    if kind == "f32":
        out = torch.empty(idx.cols, dtype=torch.float32, device=dv.device)
    else:  # int32 / wide / fp64 kernels write fp64 directly
        out = torch.empty(idx.cols, dtype=torch.float64, device=dv.device)
    exp2 = cls.exp2 if compute in (None, "int32") else 0
    for r in ranges:
        _multiply_device(dv, idx, use_fold, r, out, max_abs=mx, exp2=exp2)
    return out.double().cpu().numpy()


def batch_plan(idx):
    """The index re-cut for the batch-native kernel (rsr_batch_plan_*, csrc/batch_lanes.cu):
    built on the device on first use (one host synchronisation, never while the stream is
    being captured) and kept with the index.  None when the batch kernel does not apply."""
    import torch
    bp = idx._bplan
    if bp is None:
        if torch.cuda.is_current_stream_capturing():
            return None
        L = _native.lib()
        pl = _native.BatchPlan()
        cb, mb, wb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        st = L.rsr_batch_plan_layout(ctypes.byref(idx.desc), ctypes.byref(pl), ctypes.byref(cb), ctypes.byref(mb),
                                     ctypes.byref(wb))
        if st == _native.RSR_ERR_UNSUPPORTED:
            idx._bplan = False
            return None
        _native.check(st)
        codes = torch.empty(max(1, cb.value // 2), dtype=torch.int16, device="cuda")
        maps = torch.empty(max(1, mb.value // 2), dtype=torch.int16, device="cuda")
        ws = torch.empty(max(1, wb.value), dtype=torch.uint8, device="cuda")
        pl.codes, pl.slot_bins = codes.data_ptr(), maps.data_ptr()
        st = L.rsr_batch_plan_build(ctypes.byref(idx.desc), ctypes.byref(pl), ws.data_ptr(), wb.value,
                                    _native.current_stream_ptr())
        if st == _native.RSR_ERR_UNSUPPORTED:
            idx._bplan = False
            return None
        _native.check(st)
        bp = idx._bplan = (pl, codes, maps)
    return bp or None


_PLAN_OFF = __import__("os").environ.get("RSR_B200_BATCH_PLAN", "1") == "0"  # diagnostics: old batch forms


def multiply_batched(V, idx, variant: str = "rsrpp"):
    """V [batch, rows] CUDA tensor -> [batch, cols] of the same dtype.  int32 batches run the
    batch-native kernel (batch_plan; csrc/batch_lanes.cu: lanes span 64 vectors, conflict-free
    reductions, no host synchronisation, CUDA-graph capturable once the plan exists).  Otherwise
    (fp32, fp64, or no plan): index beyond L2: the
    batched gather kernel (csrc/batched.cu: each index byte read once per slice of up to 128
    vectors).  Index L2-resident: scatter launches, int32 two vectors per launch when the
    device guard proves the packing exact (one host sync per call; include/rsr_b200.h).  fp64
    runs one multiply per vector.  The reference has no batch API: this equals
    `multiply_ternary` / `multiply_rsr` applied to every row of V (kernels.py:185-206)."""
    import torch
    use_fold = _use_fold(variant)
    if not _is_device_tensor(V) or V.dim() != 2 or V.shape[1] != idx.rows:
        raise ValueError("V must be a CUDA tensor of shape [batch, rows]")
    V = V.contiguous()
    code = _torch_dtype_code(V)
    if code == _native.I64:
        raise ValueError("batched vectors must be int32, float32 or float64")
    out = torch.empty((V.shape[0], idx.cols), dtype=V.dtype, device=V.device)
    bp = batch_plan(idx) if (code == _native.I32 and not _PLAN_OFF and V.shape[0] > 1) else None
    if bp is not None:  # int32: the batch-native kernel (lanes span the vectors; no host sync)
        pl = bp[0]
        L = _native.lib()
        nbytes = L.rsr_multiply_batched_plan_workspace_bytes(ctypes.byref(pl), V.shape[0])
        ws = torch.empty(max(1, nbytes), dtype=torch.uint8, device=V.device)
        _native.check(L.rsr_multiply_batched_plan(
            ctypes.byref(idx.desc), ctypes.byref(pl), V.data_ptr(), V.shape[0], out.data_ptr(),
            _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR, ws.data_ptr(), nbytes,
            _native.current_stream_ptr()))
        return out
    nbytes = _native.lib().rsr_multiply_batched_workspace_bytes(ctypes.byref(idx.desc), V.shape[0], code)
    # int64 elements: at least nbytes (allocations are 256-byte aligned)
    # per-call workspace from torch's stream-ordered caching allocator (never shared across streams)
    ws = torch.empty(max(1, (nbytes + 7) // 8), dtype=torch.int64, device=V.device) if nbytes else None
    _native.check(_native.lib().rsr_multiply_batched(
        ctypes.byref(idx.desc), V.data_ptr(), code, V.shape[0], out.data_ptr(), code,
        _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR,
        ws.data_ptr() if ws is not None else None, ws.numel() * 8 if ws is not None else 0,
        _native.current_stream_ptr()))
    return out
