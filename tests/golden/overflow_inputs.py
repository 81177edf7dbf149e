"""Seeded inputs of the overflow / wide-value fixtures (overflow.npz).

Shared by tests/golden/make_golden.py (which runs the REAL reference on them) and the tests
(which regenerate the same inputs from the seeds, checked against the recorded digests), so
the committed fixture holds only reference outputs.  Pure NumPy.
"""

from __future__ import annotations

import hashlib

import numpy as np

# name: (domain, rows, cols, k, vector kind, bound)
CASES = {
    # int32 activations |v| <= 2^20 at 16384 rows: column sums up to 2^34
    "t_i32_2p20": ("ternary", 16384, 40, 8, "int32", 2 ** 20),
    # every entry +-2^20: the largest sums of that contract
    "t_i64_pm2p20": ("ternary", 16384, 40, 8, "int64_pm", 2 ** 20),
    # int64 activations beyond int32 (|v| <= 2^36): sums up to 2^50, still exact in fp64
    "t_i64_2p36": ("ternary", 16384, 40, 8, "int64", 2 ** 36),
    # binary, all +2^20: column sums up to 2^34
    "b_i32_pos2p20": ("binary", 16384, 40, 8, "int32_pos", 2 ** 20),
    # the reference's own calling convention: float64 holding integers
    "t_f64int_2p20": ("ternary", 16384, 40, 8, "f64int", 2 ** 20),
    # beyond 2^53 partial sums: the reference's fp64 sums round (tolerance, not bitwise)
    "t_i64_2p50": ("ternary", 4096, 40, 8, "int64", 2 ** 50),
    # non-integer float64 / float32 with a high dynamic range (outliers)
    "t_f64_hdr": ("ternary", 16384, 40, 8, "f64hdr", 0),
    "t_f32_hdr": ("ternary", 16384, 40, 8, "f32hdr", 0),
    # more rows than the u16 permutation range (ADVICE: the fp64 gather kernel's old limit)
    "t_f64_rows70000": ("ternary", 70000, 24, 8, "f64", 0),
    "t_i64_rows70000": ("ternary", 70000, 24, 8, "int64", 2 ** 33),
}


def make_inputs(name: str):
    """(A int8 [rows, cols] (ternary entries, or 0/1 for binary), v) of one case."""
    domain, rows, cols, k, kind, bound = CASES[name]
    seed = int.from_bytes(hashlib.sha256(name.encode()).digest()[:4], "little")
    rng = np.random.default_rng([seed, rows, cols])
    lo = -1 if domain == "ternary" else 0
    A = rng.integers(lo, 2, size=(rows, cols), dtype=np.int8)
    if kind == "int32":
        v = rng.integers(-bound, bound, size=rows, endpoint=True).astype(np.int32)
    elif kind == "int32_pos":
        v = np.full(rows, bound, np.int32)
    elif kind == "int64_pm":
        v = np.where(rng.integers(0, 2, size=rows) == 1, bound, -bound).astype(np.int64)
    elif kind == "int64":
        v = rng.integers(-bound, bound, size=rows, endpoint=True, dtype=np.int64)
    elif kind == "f64int":
        v = rng.integers(-bound, bound, size=rows, endpoint=True).astype(np.float64)
    elif kind in ("f64hdr", "f32hdr"):
        v = rng.standard_normal(rows) * np.exp(rng.uniform(-12, 12, size=rows))  # ~1e-5 .. 1e5
        v[rng.integers(0, rows, size=8)] *= 1e4                                     # outliers ~1e9
        if kind == "f32hdr":
            v = v.astype(np.float32)
    elif kind == "f64":
        v = rng.standard_normal(rows)
    else:
        raise ValueError(kind)
    return A, v


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
