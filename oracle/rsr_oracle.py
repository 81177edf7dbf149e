"""CPU oracle for the RSR / RSR++ hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-NumPy restatement of the reference `rsr` package's
algorithm (arxiv 2411.06360 reference, `/root/reference/pkg/src/rsr`).  It is
the checker the parity tests, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` leg compare the CUDA path against.  Nothing in the product
package (`paper_2411_06360_b200`) imports it; the product fails loudly when its
CUDA library is missing instead of falling back here.

Parity is PINNED: `tests/test_oracle_golden.py` checks every function below
against golden vectors produced by importing the real reference
(`tests/golden/make_golden.py`), including the reference's own known-answer
tests (the 6x6 worked example, conftest.py:10-26).

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import numpy as np

MAX_K = 30  # indexer.py:11


def max_k_for_rows(rows: int) -> int:
    """indexer.py:14-16 — min(30, max(1, floor(log2 rows)))."""
    return min(MAX_K, max(1, int(rows).bit_length() - 1))


def column_blocks(cols: int, k: int) -> list[tuple[int, int]]:
    """indexer.py:193-199 — contiguous (start, width) blocks; last may be short."""
    return [(s, min(k, cols - s)) for s in range(0, cols, k)]


def block_keys(dense01: np.ndarray, start: int, width: int) -> np.ndarray:
    """indexer.py:215-219 — MSB-first integer of each row's bits in the block."""
    weights = (1 << np.arange(width - 1, -1, -1)).astype(np.int64)
    return dense01[:, start:start + width].astype(np.int64) @ weights


def decompose_ternary(A: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """core.py:124-128 — positive half marks +1 entries, negative half marks -1."""
    A = np.asarray(A)
    return (A == 1).astype(np.uint8), (A == -1).astype(np.uint8)


def preprocess_binary(dense01: np.ndarray, k: int):
    """indexer.py:251-278 — per block: stable row order (perm), cumulative
    segmentation with trailing sentinel (seg, length 2^w + 1) and row keys.

    Returns (perms u32 [NB, n], segs list of int64 [2^w+1], buckets int64 [NB, n]).
    """
    dense01 = np.asarray(dense01)
    n, m = dense01.shape
    perms, segs, buckets = [], [], []
    for start, width in column_blocks(m, k):
        keys = block_keys(dense01, start, width)
        perms.append(np.argsort(keys, kind="stable").astype(np.uint32))   # indexer.py:269
        counts = np.bincount(keys, minlength=1 << width)                    # indexer.py:274
        segs.append(np.concatenate(([0], np.cumsum(counts))).astype(np.int64))  # :275-276
        buckets.append(keys)
    return np.stack(perms), segs, np.stack(buckets)


def preprocess_ternary(A: np.ndarray, k: int):
    """indexer.py:281-286 — index both binary halves with the same k."""
    pos, neg = decompose_ternary(A)
    return preprocess_binary(pos, k), preprocess_binary(neg, k)


def segment_sums(v: np.ndarray, perm: np.ndarray, seg: np.ndarray, width: int) -> np.ndarray:
    """kernels.py:50-60 — gather form (paper Eq. 4): u[j] = sum_{p in [L_j, L_{j+1})} v[perm[p]],
    accumulated in ascending p."""
    v = np.asarray(v, np.float64)
    out = np.empty(1 << width, np.float64)
    for j in range(1 << width):
        acc = 0.0
        for p in range(int(seg[j]), int(seg[j + 1])):
            acc += v[perm[p]]
        out[j] = acc
    return out


def product_dense(u: np.ndarray, width: int) -> np.ndarray:
    """kernels.py:63-71 — RSR block product r[c] = sum_j u[j] * bit_{w-1-c}(j)."""
    out = np.empty(width, np.float64)
    for c in range(width):
        shift = width - 1 - c
        acc = 0.0
        for j in range(1 << width):
            acc += u[j] * ((j >> shift) & 1)
        out[c] = acc
    return out


def product_fold(u: np.ndarray, width: int) -> np.ndarray:
    """kernels.py:74-91 — RSR++ fold (paper Alg. 3): odd-position sum gives the
    last column, pairwise compaction halves the vector, repeat."""
    out = np.empty(width, np.float64)
    half = (1 << width) >> 1
    buf = np.empty(max(1, half), np.float64)
    acc = 0.0
    for t in range(half):
        acc += u[2 * t + 1]
        buf[t] = u[2 * t] + u[2 * t + 1]
    out[width - 1] = acc
    size = half
    for c in range(width - 2, -1, -1):
        half = size >> 1
        acc = 0.0
        for t in range(half):
            acc += buf[2 * t + 1]
            buf[t] = buf[2 * t] + buf[2 * t + 1]
        out[c] = acc
        size = half
    return out


def multiply_half(v: np.ndarray, buckets: np.ndarray, cols: int, k: int, use_fold: bool,
                  block_range: tuple[int, int] | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """kernels.py:127-177 (`_run_blocks`) — scatter form: u[bucket[r]] += v[r] over
    ascending r, then the block product into out[col_start : col_start + w].
    Vectorised with np.add.at, which accumulates in index order (ascending r), so
    every bucket sum has the reference's summation order."""
    v = np.asarray(v, np.float64)
    blocks = column_blocks(cols, k)
    b0, b1 = block_range if block_range is not None else (0, len(blocks))
    if out is None:
        out = np.zeros(cols, np.float64)
    for b in range(b0, b1):
        start, width = blocks[b]
        u = np.zeros(1 << width, np.float64)
        np.add.at(u, buckets[b], v)
        out[start:start + width] = product_fold(u, width) if use_fold else product_dense(u, width)
    return out


def multiply_ternary(v, pos_buckets, neg_buckets, cols, k, use_fold=True) -> np.ndarray:
    """kernels.py:196-206 — positive-half product minus negative-half product."""
    return (multiply_half(v, pos_buckets, cols, k, use_fold)
            - multiply_half(v, neg_buckets, cols, k, use_fold))


def naive_multiply(v: np.ndarray, dense: np.ndarray) -> np.ndarray:
    """core.py:135-154 — out[j] = sum_i v[i] * A[i, j], ascending i, fp64."""
    v = np.asarray(v, np.float64)
    dense = np.asarray(dense)
    out = np.zeros(dense.shape[1], np.float64)
    for i in range(dense.shape[0]):
        out += v[i] * dense[i].astype(np.float64)
    return out


def _scan_optimal(n: int, term) -> int:
    """indexer.py:316-326 — argmin_k (n/k) * term(n, k), exact cross-multiplied
    comparison, ties to the smaller k."""
    if n < 1:
        raise ValueError("n must be at least 1")
    best_k, best_t = 1, term(n, 1)
    for k in range(2, max_k_for_rows(n) + 1):
        t = term(n, k)
        if t * best_k < best_t * k:
            best_k, best_t = k, t
    return best_k


def optimal_k_rsr(n: int) -> int:
    """indexer.py:343-345 — cost model n + k*2^k."""
    return _scan_optimal(n, lambda n, k: n + k * (1 << k))


def optimal_k_rsrpp(n: int) -> int:
    """indexer.py:348-350 — cost model n + 2^k."""
    return _scan_optimal(n, lambda n, k: n + (1 << k))
