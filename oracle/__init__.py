"""oracle — TEST INFRASTRUCTURE ONLY (never imported by the product package).

Plain CPU definitions of what the SparseDNN hot path computes, written from the paper:
  * spmm(...)            → liboracle.so `oracle_spmm` (C, fp64 accumulation; PAPER.md P:62, P:135,
                           P:139).  Returns (Y fp32, S fp64 error scale).
  * spmm_omp(...)        → the OpenMP-over-rows timing variant (bitwise identical).
  * alg1(...)            → liboracle.so `oracle_alg1` (Algorithm 1, bitset brute force).
  * alg1_bruteforce(...) → the same algorithm in pure Python over sets, for tiny inputs.
  * conv.conv2d(...)     → sparse k×k convolution by its definition (numpy, fp64),
                           pinned by tests/test_conv_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may use
this package.  It shares no code with paper_2101_07948_b200/ (the CUDA path) and imports nothing
from it.  Every function is pinned by tests/test_oracle.py against the paper's worked examples,
closed forms, brute force and library routines (numpy / scipy); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spmm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        lib.oracle_spmm.argtypes = [i32p, i32p, f32p, ctypes.c_int32, ctypes.c_int32, f32p, ctypes.c_int64,
                                    f32p, ctypes.c_int32, f32p, f64p]
        lib.oracle_spmm.restype = ctypes.c_int
        lib.oracle_spmm_omp.argtypes = lib.oracle_spmm.argtypes + [ctypes.c_int32]
        lib.oracle_spmm_omp.restype = ctypes.c_int
        lib.oracle_alg1.argtypes = [i32p, i32p, ctypes.c_int32, ctypes.c_int32, i32p]
        lib.oracle_alg1.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def _args(row_ptr, col_idx, vals, M, K, X, bias):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim != 2 or X.shape[0] != K:
        raise ValueError(f"X must be K×N with K={K}, got {X.shape}")
    if row_ptr.shape != (M + 1,):
        raise ValueError("row_ptr must have M+1 entries")
    bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    return row_ptr, col_idx, vals, X, bias


def spmm(row_ptr, col_idx, vals, M: int, K: int, X, bias=None, act: int = 1, want_scale: bool = True):
    """Y = act(W·X + b) with fp64 accumulation; returns (Y float32 M×N, S float64 M×N or None)."""
    row_ptr, col_idx, vals, X, bias = _args(row_ptr, col_idx, vals, M, K, X, bias)
    N = X.shape[1]
    Y = np.empty((M, N), dtype=np.float32)
    S = np.empty((M, N), dtype=np.float64) if want_scale else None
    rc = _load().oracle_spmm(_p(row_ptr, ctypes.c_int32), _p(col_idx, ctypes.c_int32), _p(vals, ctypes.c_float),
                             M, K, _p(X, ctypes.c_float), N, _p(bias, ctypes.c_float), act,
                             _p(Y, ctypes.c_float), _p(S, ctypes.c_double))
    if rc != 0:
        raise RuntimeError(f"oracle_spmm failed rc={rc}")
    return Y, S


def spmm_omp(row_ptr, col_idx, vals, M: int, K: int, X, bias=None, act: int = 1, threads: int = 0,
             want_scale: bool = False):
    """Timing variant; returns (Y, S or None, threads_used)."""
    row_ptr, col_idx, vals, X, bias = _args(row_ptr, col_idx, vals, M, K, X, bias)
    N = X.shape[1]
    Y = np.empty((M, N), dtype=np.float32)
    S = np.empty((M, N), dtype=np.float64) if want_scale else None
    used = _load().oracle_spmm_omp(_p(row_ptr, ctypes.c_int32), _p(col_idx, ctypes.c_int32),
                                   _p(vals, ctypes.c_float), M, K, _p(X, ctypes.c_float), N,
                                   _p(bias, ctypes.c_float), act, _p(Y, ctypes.c_float),
                                   _p(S, ctypes.c_double), threads)
    if used < 0:
        raise RuntimeError(f"oracle_spmm_omp failed rc={used}")
    return Y, S, used


def alg1(row_ptr, col_idx, M: int, K: int) -> np.ndarray:
    """Algorithm 1 in C: order[i] = source row placed at position i."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    order = np.empty(M, dtype=np.int32)
    rc = _load().oracle_alg1(_p(row_ptr, ctypes.c_int32), _p(col_idx, ctypes.c_int32), M, K,
                             _p(order, ctypes.c_int32))
    if rc != 0:
        raise RuntimeError("oracle_alg1 failed")
    return order


def alg1_bruteforce(row_sets: list[set[int]]) -> list[int]:
    """Algorithm 1 over Python sets, in the paper's notation.

    rem = {0 ... m-1}                                   (line 3, reading C1)
    row = argmax_{x in rem} |nnz(A[x])|                 (line 4)
    B[0] = A[row]; rem.remove(row)                      (lines 5-6)
    for i in 1 ... m-1:                                 (line 7, reading C1)
        row = argmax_{x in rem} |nnz(B[i-1]) ∩ nnz(A[x])|   (line 8, reading C4)
        B[i] = A[row]; rem.remove(row)                  (lines 9-10)
    argmax ties → lowest original index (readings C2, C3).
    """
    m = len(row_sets)
    if m == 0:
        return []
    rem = list(range(m))
    row = min(rem, key=lambda x: (-len(row_sets[x]), x))
    order = [row]
    rem.remove(row)
    for _ in range(1, m):
        prev = row_sets[order[-1]]
        row = min(rem, key=lambda x: (-len(prev & row_sets[x]), x))
        order.append(row)
        rem.remove(row)
    return order
