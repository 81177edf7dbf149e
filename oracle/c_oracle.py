"""ctypes binding of oracle/rsr_oracle.c — TEST INFRASTRUCTURE ONLY (checker and
CPU baseline; never imported by the product package)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "librsr_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64, I = ctypes.c_int64, ctypes.c_int
        L.rsr_oracle_keys_ternary.argtypes = [P, I64, I64, I, I, P]
        L.rsr_oracle_sort_block.argtypes = [P, I64, I, P, P]
        L.rsr_oracle_run_blocks.argtypes = [P, P, I64, I64, I, I64, I64, I, P]
        L.rsr_oracle_multiply_parallel.argtypes = [P, P, P, I64, I64, I, I, I, P, P]
        L.rsr_oracle_naive_ternary.argtypes = [P, P, I64, I64, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def keys_ternary(A: np.ndarray, k: int, sign: int) -> np.ndarray:
    A = np.ascontiguousarray(A, np.int8)
    n, m = A.shape
    nb = (m + k - 1) // k
    keys = np.empty((nb, n), np.uint16)
    lib().rsr_oracle_keys_ternary(_p(A), n, m, k, sign, _p(keys))
    return keys


def sort_block(keys: np.ndarray, width: int):
    keys = np.ascontiguousarray(keys, np.uint16)
    n = keys.shape[0]
    perm = np.empty(n, np.uint32)
    seg = np.empty((1 << width) + 1, np.int64)
    lib().rsr_oracle_sort_block(_p(keys), n, width, _p(perm), _p(seg))
    return perm, seg


def preprocess_ternary(A: np.ndarray, k: int):
    """Returns ((perms, segs, keys) positive, (perms, segs, keys) negative)."""
    A = np.ascontiguousarray(A, np.int8)
    n, m = A.shape
    halves = []
    for sign in (1, -1):
        keys = keys_ternary(A, k, sign)
        perms, segs = [], []
        for b in range(keys.shape[0]):
            w = min(k, m - b * k)
            p, s = sort_block(keys[b], w)
            perms.append(p)
            segs.append(s)
        halves.append((np.stack(perms), segs, keys))
    return tuple(halves)


def multiply_parallel(v, keys_pos, keys_neg, m: int, k: int, use_fold: bool = True,
                      workers: int = 1) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    kp = np.ascontiguousarray(keys_pos, np.uint16)
    kn = None if keys_neg is None else np.ascontiguousarray(keys_neg, np.uint16)
    out = np.empty(m, np.float64)
    scratch = np.empty(m, np.float64)
    lib().rsr_oracle_multiply_parallel(_p(v), _p(kp), None if kn is None else _p(kn),
                                       v.shape[0], m, k, int(use_fold), int(workers),
                                       _p(out), _p(scratch))
    return out


def naive_ternary(v, A) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    A = np.ascontiguousarray(A, np.int8)
    out = np.empty(A.shape[1], np.float64)
    lib().rsr_oracle_naive_ternary(_p(v), _p(A), A.shape[0], A.shape[1], _p(out))
    return out
