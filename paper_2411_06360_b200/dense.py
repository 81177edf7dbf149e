"""Dense ternary multiply on the GPU — the paper's "standard" multiply (reference
core.py:135-169 `naive_multiply`) kept as the honest comparator of the RSR++
path.  See csrc/dense.cu.

* `multiply` — 2-bit planes, any int32 / fp32 vector (exact int32).
* `multiply_i8` — int8-range activations (the reference's own benchmark vectors are integers in
  [-100, 100]) with IDP4A on a 2-bit layout: streams the 2-bit matrix at HBM speed.
* `multiply_batched_i8` — B vectors at once: int8 x int8 -> int32 GEMM on the tensor cores
  (cuBLASLt through torch._int_mm, the library GEMM) against an int8 copy of the matrix."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .core import TernaryMatrix


class DenseTernary:
    """A ternary matrix packed as two device bit-planes (2 bits per entry)."""

    def __init__(self, matrix, keep_int8: bool = False):
        import torch
        entries = matrix.entries if isinstance(matrix, TernaryMatrix) else matrix
        if not isinstance(entries, torch.Tensor):
            entries = torch.from_numpy(np.ascontiguousarray(np.asarray(entries, np.int8)))
        entries = entries.to(device="cuda", dtype=torch.int8).contiguous()
        if entries.dim() != 2:
            raise ValueError("matrix must be 2-D")
        self.rows, self.cols = (int(x) for x in entries.shape)
        words = _native.lib().rsr_dense_plane_words(self.rows, self.cols)
        self.pos = torch.empty(words, dtype=torch.int32, device="cuda")
        self.neg = torch.empty(words, dtype=torch.int32, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        _native.check(_native.lib().rsr_dense_pack_ternary(
            entries.data_ptr(), self.cols, self.rows, self.cols, self.pos.data_ptr(), self.neg.data_ptr(),
            bad.data_ptr(), _native.current_stream_ptr()))
        words8 = _native.lib().rsr_dense_i8_words(self.rows, self.cols)
        self.q = torch.empty(words8, dtype=torch.int32, device="cuda")
        _native.check(_native.lib().rsr_dense_pack_ternary_i8(
            entries.data_ptr(), self.cols, self.rows, self.cols, self.q.data_ptr(), bad.data_ptr(),
            _native.current_stream_ptr()))
        if int(bad.item()):
            raise ValueError("ternary entries must be in {-1, 0, 1}")
        self._entries = entries if keep_int8 else None

    @property
    def nbytes(self) -> int:
        return 2 * self.pos.numel() * 4

    @property
    def nbytes_i8(self) -> int:
        """Bytes of the 2-bit IDP4A layout (what multiply_i8 streams)."""
        return self.q.numel() * 4

    def multiply_i8(self, v, out=None):
        """v int8 CUDA tensor [rows] -> int32 [cols], exact (IDP4A, csrc/dense.cu)."""
        import torch
        if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dim() == 1 and v.dtype == torch.int8):
            raise ValueError("v must be a 1-D int8 CUDA tensor")
        if v.shape[0] != self.rows:
            raise ValueError(f"vector length {v.shape[0]} does not match {self.rows} rows")
        v = v.contiguous()
        if out is None:
            out = torch.empty(self.cols, dtype=torch.int32, device=v.device)
        _native.check(_native.lib().rsr_dense_multiply_i8(
            self.q.data_ptr(), self.rows, self.cols, v.data_ptr(), out.data_ptr(), _native.current_stream_ptr()))
        return out

    def multiply_batched_i8(self, V):
        """V int8 CUDA tensor [B, rows] (B > 16, sizes multiples of 8) -> int32 [B, cols]: the
        library int8 GEMM (cuBLASLt via torch._int_mm) on the int8 matrix (keep_int8=True)."""
        import torch
        if self._entries is None:
            raise ValueError("construct with keep_int8=True for the batched dense comparator")
        return torch._int_mm(V, self._entries)

    def multiply(self, v, out=None):
        """v CUDA tensor [rows] (int32 exact / float32) -> [cols] of the same dtype."""
        import torch
        if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dim() == 1):
            raise ValueError("v must be a 1-D CUDA tensor")
        if v.shape[0] != self.rows:
            raise ValueError(f"vector length {v.shape[0]} does not match {self.rows} rows")
        code = {torch.int32: _native.I32, torch.float32: _native.F32}.get(v.dtype)
        if code is None:
            raise ValueError("dense multiply takes int32 or float32 vectors")
        v = v.contiguous()
        if out is None:
            out = torch.empty(self.cols, dtype=v.dtype, device=v.device)
        _native.check(_native.lib().rsr_dense_multiply(
            self.pos.data_ptr(), self.neg.data_ptr(), self.rows, self.cols, v.data_ptr(), code,
            out.data_ptr(), _native.current_stream_ptr()))
        return out
