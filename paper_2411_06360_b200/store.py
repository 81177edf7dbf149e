"""Bit-exact `.rsx` index files (reference store.py:1-101).

Same format as the reference: a 29-byte little-endian header ``<4sHBQQHI`` (magic ``RSX1``,
version 1, kind 1 binary / 2 ternary, rows, cols, k, block count), then per half (ternary:
positive then negative) and per column block: u16 width, u32 permutation [rows], u32
segment starts [2^width] (no sentinel).  Same checks, same ``FormatError`` messages.

Loading ships the stored arrays to HBM once and rebuilds the device layout there
(`rsr_index_import`: u16 perm, u32 seg + sentinel, key codes rebuilt from the segments, key
schedule) — no host-side `_buckets_from_segments` (indexer.py:176-186).  The invariants the
reference re-validates through `RsrIndex.from_blocks` (indexer.py:89-129) are checked on the
device; the first failing block is re-checked on the host only to word the error exactly
like the reference.
"""

from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np

from . import _native
from .core import FormatError
from .indexer import RsrIndex, TernaryIndex, _check_k, _DeviceArrays, column_blocks

_MAGIC = b"RSX1"
_VERSION = 1
_KIND_BINARY = 1
_KIND_TERNARY = 2
_HEADER = struct.Struct("<4sHBQQHI")  # magic, version, kind, rows, cols, k, block_count
HEADER_BYTES = _HEADER.size


# ----------------------------------------------------------------------------- writing
def _halves(idx):
    if isinstance(idx, TernaryIndex):
        return _KIND_TERNARY, (idx.positive, idx.negative)
    if isinstance(idx, RsrIndex):
        return _KIND_BINARY, (idx,)
    raise TypeError("expected RsrIndex or TernaryIndex")


def save_index(idx, path) -> None:
    """Write an index (store.py:31-45); ternary files store the positive half then the negative."""
    kind, halves = _halves(idx)
    parts = [_HEADER.pack(_MAGIC, _VERSION, kind, idx.rows, idx.cols, idx.k, halves[0].block_count)]
    for half in halves:
        perm, seg, _ = half.host_arrays()
        for b, (_, width) in enumerate(column_blocks(half.cols, half.k)):
            parts.append(struct.pack("<H", width))
            parts.append(perm[b, :half.rows].astype("<u4").tobytes())
            parts.append(seg[b, :1 << width].astype("<u4").tobytes())
    Path(path).write_bytes(b"".join(parts))


# ----------------------------------------------------------------------------- reading
def _read_half(raw: bytes, offset: int, rows: int, cols: int, k: int, block_count: int):
    """Structure checks of store.py:48-66 in the reference's order; returns (per-block perm
    views, per-block seg views, offset).  No array is allocated before its bytes are known to
    exist (a corrupt k cannot ask for 2^k entries)."""
    expected = column_blocks(cols, k)  # ValueError for k < 1, as the reference
    if block_count != len(expected):
        raise FormatError(f"block_count {block_count} does not match ceil(cols/k)")
    perms, segs = [], []
    for _, width in expected:
        if offset + 2 > len(raw):
            raise FormatError("truncated block header")
        (stored_width,) = struct.unpack_from("<H", raw, offset)
        offset += 2
        if stored_width != width:
            raise FormatError(f"block width {stored_width} does not partition {cols} columns")
        nbytes = 4 * rows + 4 * (1 << width)
        if offset + nbytes > len(raw):
            raise FormatError("truncated payload")
        perms.append(np.frombuffer(raw, "<u4", count=rows, offset=offset))
        segs.append(np.frombuffer(raw, "<u4", count=1 << width, offset=offset + 4 * rows))
        offset += nbytes
    return perms, segs, offset


def _block_error(perm: np.ndarray, seg: np.ndarray, rows: int, b: int):
    """The reference's message for block b, or None (indexer.py:110-122, same order)."""
    p = perm.astype(np.int64)
    counts = np.bincount(np.minimum(p, rows), minlength=rows + 1)[:rows]
    if p.size and (p.max() >= rows or (counts != 1).any()):
        return f"block {b}: permutation is not a bijection"
    s = seg.astype(np.int64)
    if s[0] != 0:
        return f"block {b}: segmentation must start at 0"
    if (np.diff(s) < 0).any() or s[-1] > rows:
        return f"block {b}: segmentation must be non-decreasing and <= rows"
    return None


def _half_violation(perms, segs, rows: int):
    """First failing block of one half in the reference's order (RsrIndex.from_blocks), or None.
    Host NumPy, used only on error paths: the device import validates the good case."""
    for b, (p, s) in enumerate(zip(perms, segs)):
        msg = _block_error(p, s, rows, b)
        if msg:
            return msg
    return None


def load_index(path, device=None):
    """Read and re-validate an index file (store.py:80-101); returns an RsrIndex or a
    TernaryIndex resident in HBM.  Errors come in the reference's order: the header, then for
    each half its structure and then its invariants (k, then block by block), then trailing
    bytes."""
    import torch
    raw = Path(path).read_bytes()
    if len(raw) < HEADER_BYTES:
        raise FormatError("truncated header")
    magic, version, kind, rows, cols, k, block_count = _HEADER.unpack_from(raw)
    if magic != _MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != _VERSION:
        raise FormatError(f"unsupported version {version}")
    if kind not in (_KIND_BINARY, _KIND_TERNARY):
        raise FormatError(f"unknown index kind {kind}")
    if rows < 1 or cols < 1:
        raise FormatError("index dimensions must be at least 1x1")
    offset = HEADER_BYTES
    halves = []
    for h in range(2 if kind == _KIND_TERNARY else 1):
        try:
            perms, segs, offset = _read_half(raw, offset, rows, cols, k, block_count)
        except FormatError:
            # the reference validated the previous half before reading this one
            if halves:
                msg = _half_violation(*halves[-1], rows)
                if msg:
                    raise FormatError(f"invariant violation: {msg}") from None
            raise
        try:  # RsrIndex.from_blocks checks k first (indexer.py:96)
            _check_k(k, rows)
        except ValueError as exc:
            raise FormatError(f"invariant violation: {exc}") from None
        halves.append((perms, segs))
    if offset != len(raw):
        for hp in halves:
            msg = _half_violation(*hp, rows)
            if msg:
                raise FormatError(f"invariant violation: {msg}")
        raise FormatError("trailing bytes")
    widths = [w for _, w in column_blocks(cols, k)]
    stacked = []
    for perms, segs in halves:
        perm = np.stack(perms).astype(np.uint32)
        seg = np.zeros((len(widths), 1 << k), np.uint32)
        for b, (sg, w) in enumerate(zip(segs, widths)):
            seg[b, :1 << w] = sg
        stacked.append((perm, seg))
    halves = stacked

    arrays = _DeviceArrays(rows, cols, k, len(halves), device)
    dev = arrays.device
    d_in = [(torch.from_numpy(p.view(np.int32)).to(dev), torch.from_numpy(s.view(np.int32)).to(dev))
            for p, s in halves]
    L = _native.lib()
    nbytes = L.rsr_index_import_workspace_bytes(ctypes.byref(arrays.desc))
    ws = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.int32, device=dev)
    err = torch.tensor([0, 2 ** 31 - 1], dtype=torch.int32, device=dev)
    p1, s1 = d_in[1] if len(d_in) == 2 else (None, None)
    _native.check(L.rsr_index_import(
        ctypes.byref(arrays.desc), d_in[0][0].data_ptr(), d_in[0][1].data_ptr(),
        p1.data_ptr() if p1 is not None else None, s1.data_ptr() if s1 is not None else None,
        1 << k, ws.data_ptr(), ws.numel() * 4, err.data_ptr(), _native.current_stream_ptr()))
    flags, _ = (int(x) for x in err.cpu())
    if flags:  # word the error as the reference would: half 0 block by block, then half 1
        for perm, seg in halves:
            msg = _half_violation(list(perm), [seg[b, :1 << w] for b, w in enumerate(widths)], rows)
            if msg:
                raise FormatError(f"invariant violation: {msg}")
        raise FormatError("invariant violation: index arrays failed validation")
    if kind == _KIND_BINARY:
        return RsrIndex(arrays, 0)
    return TernaryIndex(RsrIndex(arrays, 0), RsrIndex(arrays, 1))
