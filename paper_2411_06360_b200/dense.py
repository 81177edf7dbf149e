"""Dense 2-bit ternary GEMV on the GPU — the paper's "standard" multiply (reference
core.py:135-169 `naive_multiply`) kept as the honest comparator of the RSR++
path.  See csrc/dense.cu."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .core import TernaryMatrix


class DenseTernary:
    """A ternary matrix packed as two device bit-planes (2 bits per entry)."""

    def __init__(self, matrix):
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
        if int(bad.item()):
            raise ValueError("ternary entries must be in {-1, 0, 1}")

    @property
    def nbytes(self) -> int:
        return 2 * self.pos.numel() * 4

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
