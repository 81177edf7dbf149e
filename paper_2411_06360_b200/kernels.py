"""Inference: segmented sums, block products and the fused multiply, on the GPU.

Mirrors the reference `rsr.kernels` (kernels.py:1-239): same names, argument
meanings, validation order and error messages.  Every multiply is one launch
of the sm_100a kernels in librsr_b200.so (see csrc/multiply.cu):

* NumPy / list input keeps the reference contract (fp64 in, fp64 out).  The
  call copies v to a pinned buffer, and one C-ABI call (`rsr_multiply_host`)
  does H2D, the multiply and D2H.  fp64 vectors use the deterministic gather
  kernel in fp64; integer-typed NumPy vectors use the int32 scatter kernel
  (exact) and still return fp64.
* torch CUDA tensors stay on the device: int32 -> int32 (scatter kernel, bit-
  exact), float32 -> float32 and float64 -> float64 (gather kernel).
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
        _DTYPES.update({torch.int32: _native.I32, torch.float32: _native.F32, torch.float64: _native.F64})
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ValueError("device vectors must be int32, float32 or float64") from None


class _HostStaging(threading.local):
    """Per-thread device scratch and host-buffer sessions.  Thread-local: concurrent multiplies
    from several threads never share buffers."""

    def __init__(self):
        self.bufs = {}
        self.plans = {}  # id(index) -> (weakref to the index, {kind: _HostPlan}); no strong refs

    def get(self, key, shape, dtype, pinned):
        """(tensor, numpy view or None, data pointer) of a cached buffer of `shape` elements."""
        import torch
        dev = -1 if pinned else torch.cuda.current_device()
        ent = self.bufs.get((key, shape, dev))
        if ent is None or ent[0].dtype != dtype:
            t = (torch.empty(shape, dtype=dtype, pin_memory=True) if pinned
                 else torch.empty(shape, dtype=dtype, device="cuda"))
            ent = (t, t.numpy() if pinned else None, t.data_ptr())
            self.bufs[(key, shape, dev)] = ent
        return ent


_staging = _HostStaging()
_KIND_CODE = {"i32": _native.I32, "f32": _native.F32, "f64": _native.F64}


class _HostPlan:
    """One host-buffer session (rsr_host_session_*: pinned staging, device scratch, mapped
    result + completion flag) for one index, vector type and thread, created on first use and
    destroyed with the index or the thread."""
    __slots__ = ("session", "cols", "call", "stream", "__weakref__")

    def __init__(self, idx, kind):
        import torch
        L = _native.lib()
        h = ctypes.c_void_p()
        _native.check(L.rsr_host_session_create(ctypes.byref(idx.desc), _KIND_CODE[kind], ctypes.byref(h)))
        self.session = h.value
        self.cols = idx.cols
        self.call = _native.host_ext().multiply
        # torch's current stream on the session's device, queried per call (sub-microsecond)
        dev = torch.cuda.current_device()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        self.stream = (lambda: raw(dev)) if raw is not None else _native.current_stream_ptr
        weakref.finalize(self, L.rsr_host_session_destroy, h.value)


def _host_plan(idx, kind) -> _HostPlan:
    plans = _staging.plans
    ent = plans.get(id(idx))
    if ent is None or ent[0]() is not idx:
        key = id(idx)
        ent = plans[key] = (weakref.ref(idx, lambda _r, k=key, d=plans: d.pop(k, None)), {})
    per = ent[1]
    plan = per.get(kind)
    if plan is None:
        plan = per[kind] = _HostPlan(idx, kind)
    return plan


def _run_host(idx, kind, v: np.ndarray, use_fold: bool) -> np.ndarray:
    """One session call: v (C-contiguous, the session's type) -> fresh fp64 result (the
    reference's result type)."""
    plan = _host_plan(idx, kind)
    out = np.empty(plan.cols, np.float64)
    st = plan.call(plan.session, v, out, _native.F64, _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR,
                   plan.stream())
    if st:
        _native.check(st)
    return out


def _multiply_device(v, idx, use_fold: bool, block_range=None, out=None, form=_native.FORM_AUTO):
    """Device-tensor path: v CUDA tensor [rows] -> CUDA tensor [cols]."""
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
    _native.check(_native.lib().rsr_multiply(
        ctypes.byref(idx.desc), v.data_ptr(), code, out.data_ptr(), _torch_dtype_code(out),
        _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR, form, b0, b1,
        _native.current_stream_ptr()))
    return out


def _multiply_host(v_in, idx, use_fold: bool, compute: str | None) -> np.ndarray:
    """Host-buffer path (reference contract): NumPy in, fresh fp64 NumPy out, via one
    rsr_multiply_host call (H2D + multiply + D2H + sync)."""
    raw = np.asarray(v_in)
    if raw.dtype.kind in "iub" and compute in (None, "int32"):
        # integer activations (always finite): no float64 round trip, range check only
        # for dtypes wider than int32
        if raw.ndim != 1 or raw.shape[0] < 1:
            raise ValueError("vector must be 1-D with at least one entry")
        if raw.shape[0] != idx.rows:
            raise ValueError(f"vector length {raw.shape[0]} does not match {idx.rows} rows")
        if raw.dtype == np.int32:
            return _run_host(idx, "i32", raw if raw.flags.c_contiguous else np.ascontiguousarray(raw), use_fold)
        if raw.dtype.itemsize < 4 or (raw.min() >= -2 ** 31 and raw.max() < 2 ** 31):
            return _run_host(idx, "i32", np.ascontiguousarray(raw, np.int32), use_fold)
        if compute == "int32":
            raise ValueError("integer activations exceed the int32 range")
    if raw.dtype == np.float32 and compute in (None, "float32"):
        # fp32 activations are computed in fp32 (north star: within 1e-5 relative of the
        # fp64 reference); results come back as fresh fp64 arrays like the reference's
        if raw.ndim != 1 or raw.shape[0] < 1:
            raise ValueError("vector must be 1-D with at least one entry")
        if not np.isfinite(raw).all():
            raise ValueError("vector entries must be finite")
        if raw.shape[0] != idx.rows:
            raise ValueError(f"vector length {raw.shape[0]} does not match {idx.rows} rows")
        return _run_host(idx, "f32", np.ascontiguousarray(raw), use_fold)
    v = as_vector(v_in)
    if v.shape[0] != idx.rows:
        raise ValueError(f"vector length {v.shape[0]} does not match {idx.rows} rows")
    if compute == "float32":
        return _run_host(idx, "f32", v.astype(np.float32), use_fold)
    if compute == "int32":
        if np.any(v != np.round(v)) or np.abs(v).max(initial=0) >= 2 ** 31:
            raise ValueError("compute='int32' needs integer-valued activations in the int32 range")
        return _run_host(idx, "i32", v.astype(np.int32), use_fold)
    if compute in (None, "float64"):
        return _run_host(idx, "f64", np.ascontiguousarray(v), use_fold)
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
    path shards across ranks); the result is bitwise independent of W."""
    import torch
    use_fold = _use_fold(variant)
    if worker_count < 1:
        raise ValueError("worker_count must be at least 1")
    device_in = _is_device_tensor(v)
    if device_in:
        dv = v
    else:
        vv = as_vector(v)
        if vv.shape[0] != idx.rows:
            raise ValueError(f"vector length {vv.shape[0]} does not match {idx.rows} rows")
        raw = np.asarray(v)
        if compute == "int32" or (compute is None and raw.dtype.kind in "iub"):
            dv = torch.from_numpy(vv.astype(np.int32)).cuda()
        else:
            dv = torch.from_numpy(vv).cuda()
    if dv.shape[0] != idx.rows:
        raise ValueError(f"vector length {dv.shape[0]} does not match {idx.rows} rows")
    out_dtype = torch.float64 if (not device_in) else dv.dtype
    out = torch.empty(idx.cols, dtype=out_dtype, device=dv.device)
    nb = idx.desc.nblocks
    bounds = [i * nb // worker_count for i in range(worker_count + 1)]
    for lo, hi in zip(bounds, bounds[1:]):
        if lo < hi:
            _multiply_device(dv, idx, use_fold, (lo, hi), out)
    return out if device_in else out.cpu().numpy()


def multiply_batched(V, idx, variant: str = "rsrpp"):
    """V [batch, rows] CUDA tensor -> [batch, cols] of the same dtype.  Index beyond L2: the
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
    out = torch.empty((V.shape[0], idx.cols), dtype=V.dtype, device=V.device)
    nbytes = _native.lib().rsr_multiply_batched_workspace_bytes(ctypes.byref(idx.desc), V.shape[0], code)
    # int64 elements: at least nbytes (allocations are 256-byte aligned)
    ws = _staging.get("batch_ws", max(1, (nbytes + 7) // 8), torch.int64, False)[0] if nbytes else None
    _native.check(_native.lib().rsr_multiply_batched(
        ctypes.byref(idx.desc), V.data_ptr(), code, V.shape[0], out.data_ptr(), code,
        _native.VARIANT_RSRPP if use_fold else _native.VARIANT_RSR,
        ws.data_ptr() if ws is not None else None, ws.numel() * 8 if ws is not None else 0,
        _native.current_stream_ptr()))
    return out
