"""CPU oracle for the MaxK-GNN hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package. The product path (``paper_2312_08656_b200``) never imports
it and shares no code with it.

Every function is the plain definition from the paper, in fp64 (oracle.c has the citations):
  topk_cbsr   Eq. 1, PAPER.md:228-234 (§3.1) + CBSR layout PAPER.md:326 (§3.2)
  densify     the dense matrix a CBSR block stands for
  spgemm_fwd  X_l = A · h(X_{l-1})  (Eq. 3 left; row-wise form PAPER.md:326)
  sspmm_bwd   dL/dh = (A^T · dL/dX_l) sampled at sp_index (Eq. 3 right PAPER.md:320, Eq. 4
              PAPER.md:341-343, "known output sparse pattern" PAPER.md:440)
Pins: tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, OpenMP). Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        lib.oracle_topk_cbsr.argtypes = [vp, i64, i32, i64, i32, vp, vp]
        lib.oracle_topk_cbsr.restype = ctypes.c_int
        lib.oracle_densify.argtypes = [i64, i32, i32, vp, vp, vp]
        lib.oracle_densify.restype = None
        lib.oracle_spmm_rows.argtypes = [vp, vp, vp, vp, i64, vp, i32, vp]
        lib.oracle_spmm_rows.restype = None
        lib.oracle_transpose.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp]
        lib.oracle_transpose.restype = ctypes.c_int
        lib.oracle_sspmm_rows.argtypes = [vp, vp, vp, vp, i64, i32, vp, i32, vp, i64, vp]
        lib.oracle_sspmm_rows.restype = None
        lib.oracle_num_threads.argtypes = []
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        lib.oracle_set_num_threads.restype = None
        _lib = lib
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray):
    return a.ctypes.data if a.size else None


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def topk_cbsr(x: np.ndarray, k: int):
    """Exact per-row top-k (value desc, column asc) -> (data float32 [n,k], idx int32 [n,k] ascending)."""
    x = _c(x, np.float32)
    n, h = x.shape
    data = np.empty((n, k), dtype=np.float32)
    idx = np.empty((n, k), dtype=np.int32)
    rc = _load().oracle_topk_cbsr(_p(x), n, h, h, k, _p(data), _p(idx))
    if rc == -1:
        raise ValueError(f"invalid top-k arguments (n={n}, h={h}, k={k})")
    if rc == -2:
        raise ValueError("NaN in top-k input (precondition violation)")
    return data, idx


def densify(data: np.ndarray, idx: np.ndarray, h: int) -> np.ndarray:
    data = _c(data, np.float32)
    idx = _c(idx, np.int32)
    n, k = data.shape
    out = np.empty((n, h), dtype=np.float64)
    _load().oracle_densify(n, h, k, _p(data), _p(idx), _p(out))
    return out


def spmm(row_ptr, col_idx, val, dense: np.ndarray, rows=None) -> np.ndarray:
    """Y = A · dense (fp64) for all rows, or for the row subset ``rows``."""
    row_ptr = _c(row_ptr, np.int64)
    col_idx = _c(col_idx, np.int32)
    val = _c(val, np.float32)
    dense = _c(dense, np.float64)
    h = dense.shape[1]
    if rows is None:
        n_sel, rp = row_ptr.shape[0] - 1, None
    else:
        rp = _c(rows, np.int64)
        n_sel = rp.shape[0]
    y = np.empty((n_sel, h), dtype=np.float64)
    _load().oracle_spmm_rows(_p(row_ptr), _p(col_idx), _p(val), _p(rp) if rp is not None else None,
                             n_sel, _p(dense), h, _p(y))
    return y


def spgemm_fwd(row_ptr, col_idx, val, data, idx, h: int, rows=None) -> np.ndarray:
    """Y = A · densify(CBSR) in fp64 (Eq. 3 left / row-wise product PAPER.md:326)."""
    return spmm(row_ptr, col_idx, val, densify(data, idx, h), rows=rows)


def transpose(row_ptr, col_idx, val, n_cols: int):
    """(t_ptr, t_row, t_val): CSR of A^T by stable counting sort."""
    row_ptr = _c(row_ptr, np.int64)
    col_idx = _c(col_idx, np.int32)
    val = _c(val, np.float32)
    n_rows = row_ptr.shape[0] - 1
    nnz = int(row_ptr[-1] - row_ptr[0])
    t_ptr = np.empty(n_cols + 1, dtype=np.int64)
    t_row = np.empty(nnz, dtype=np.int32)
    t_val = np.empty(nnz, dtype=np.float32)
    rc = _load().oracle_transpose(_p(row_ptr), _p(col_idx), _p(val), n_rows, n_cols, _p(t_ptr),
                                  _p(t_row), _p(t_val))
    if rc != 0:
        raise ValueError("col_idx out of range")
    return t_ptr, t_row, t_val


def sspmm_bwd(row_ptr, col_idx, val, dy: np.ndarray, idx: np.ndarray, rows=None, transposed=None):
    """dXs = (A^T · dY) sampled at idx, fp64, for all CBSR rows or the subset ``rows``.

    ``idx`` is the [n_cols, k] forward pattern. ``transposed`` may pass a cached transpose().
    """
    dy = _c(dy, np.float32)
    idx = _c(idx, np.int32)
    n_cols, k = idx.shape
    h = dy.shape[1]
    t_ptr, t_row, t_val = transposed if transposed is not None else transpose(row_ptr, col_idx, val, n_cols)
    if rows is None:
        n_sel, rp = n_cols, None
    else:
        rp = _c(rows, np.int64)
        n_sel = rp.shape[0]
    out = np.empty((n_sel, k), dtype=np.float64)
    _load().oracle_sspmm_rows(_p(t_ptr), _p(t_row), _p(t_val), _p(dy), h, h, _p(idx), k,
                              _p(rp) if rp is not None else None, n_sel, _p(out))
    return out


def linear(x: np.ndarray, w_t: np.ndarray, bias=None) -> np.ndarray:
    """z = X·W + b in fp64 (the argument of max-k in Eq. 1); w_t is W transposed ([h, f]).

    The product is a library matmul (numpy) on exactly converted inputs — a plain definition.
    """
    z = np.asarray(x, np.float64) @ np.asarray(w_t, np.float64).T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)[None, :]
    return z
