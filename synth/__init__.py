"""Seeded synthetic inputs shared by the CUDA path (tests, bench) and the CPU oracle.

This module holds none of the method's arithmetic (no top-k, aggregation or gradient). It draws
graphs shaped like the paper's datasets (Table 1) and N(0,1) feature matrices
(§5.3). The recipe is stated in DESIGN.md §3 and in synth.c's header.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None

GRAPH_SEED_BASE = 0x4D61784B  # graph seed = base + config index
X_SEED = 1
DY_SEED = 2


def build(force: bool = False) -> str:
    """Compile synth.c into libsynth.so (gcc, OpenMP). Returns the library path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, u64, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.synth_degrees.argtypes = [i64, i64, dbl, i64, u64, vp, vp, vp]
        lib.synth_degrees.restype = ctypes.c_int
        lib.synth_columns.argtypes = [i64, vp, vp, u64, vp]
        lib.synth_columns.restype = ctypes.c_int
        lib.synth_mean_values.argtypes = [i64, vp, vp]
        lib.synth_mean_values.restype = None
        lib.synth_normal_f32.argtypes = [u64, i64, i64, vp]
        lib.synth_normal_f32.restype = None
        lib.synth_num_threads.argtypes = []
        lib.synth_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


@dataclass
class Csr:
    """CSR adjacency: row_ptr int64 [n+1], col_idx int32 [nnz], val float32 [nnz]."""

    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray
    n_cols: int

    @property
    def n_rows(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1] - self.row_ptr[0])


def power_law_degrees(n: int, nnz: int, seed: int, gamma: float = 2.1, d_max: int = 0):
    """Degree sequence (int64 [n]) and column weights (float64 [n]) of the Chung–Lu graph."""
    lib = _load()
    deg = np.empty(n, dtype=np.int64)
    w = np.empty(n, dtype=np.float64)
    rc = lib.synth_degrees(n, nnz, gamma, d_max, seed & 0xFFFFFFFFFFFFFFFF, _ptr(deg), _ptr(w), None)
    if rc != 0:
        raise ValueError(f"synth_degrees failed ({rc})")
    return deg, w


def power_law_graph(n: int, nnz: int, seed: int, gamma: float = 2.1, d_max: int = 0,
                    rows: tuple[int, int] | None = None) -> Csr:
    """Directed Chung–Lu power-law CSR with sorted unique columns and val = 1/deg.

    ``rows=(r0, r1)`` generates only that row block (row_ptr rebased to 0), bit-identical to the
    same rows of the full graph — used by multi-GPU ranks.
    """
    lib = _load()
    deg, w = power_law_degrees(n, nnz, seed, gamma, d_max)
    r0, r1 = (0, n) if rows is None else rows
    deg_blk = np.ascontiguousarray(deg[r0:r1])
    row_ptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
    np.cumsum(deg_blk, out=row_ptr[1:])
    nnz_blk = int(row_ptr[-1])
    col = np.empty(nnz_blk, dtype=np.int32)
    val = np.empty(nnz_blk, dtype=np.float32)
    # synth_columns is keyed by the node id, so generate with a shifted view: node v = r0 + local
    if r1 > r0:
        full_ptr = np.zeros(n + 1, dtype=np.int64)
        # only rows in [r0, r1) have nonzero length in this pass
        lens = np.zeros(n, dtype=np.int64)
        lens[r0:r1] = deg_blk
        np.cumsum(lens, out=full_ptr[1:])
        rc = lib.synth_columns(n, _ptr(full_ptr), _ptr(w), seed & 0xFFFFFFFFFFFFFFFF, _ptr(col))
        if rc != 0:
            raise RuntimeError(f"synth_columns failed ({rc})")
        lib.synth_mean_values(r1 - r0, _ptr(row_ptr), _ptr(val))
    return Csr(row_ptr, col, val, n)


def normal_f32(shape, seed: int, row_offset: int = 0) -> np.ndarray:
    """iid N(0,1) float32 array of the given shape (counter-based Box–Muller).

    ``row_offset`` r returns rows [r, r + shape[0]) of the same matrix generated from row 0.
    """
    lib = _load()
    out = np.empty(shape, dtype=np.float32)
    start = int(row_offset) * (int(np.prod(shape[1:])) if len(shape) > 1 else 1)
    lib.synth_normal_f32(seed & 0xFFFFFFFFFFFFFFFF, start, out.size, _ptr(out))
    return out


def num_threads() -> int:
    return int(_load().synth_num_threads())


# --------------------------------------------------------------------------------------------
# Configs of BASELINE.json (N and nnz from the config strings; Table 1).
# --------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class GraphConfig:
    name: str
    n: int
    nnz: int
    h: int
    ks: tuple
    index: int  # position in BASELINE.json configs -> graph seed
    gamma: float = 2.1  # power-law exponent (2.1 default, 2.5 the sensitivity point)

    @property
    def seed(self) -> int:
        return GRAPH_SEED_BASE + self.index

    def d_max(self) -> int:
        return int(min(self.n - 1, math.ceil(2.0 * math.sqrt(self.nnz))))


CONFIGS = {
    "tiny": GraphConfig("tiny", 1_000, 10_000, 64, (8,), 0),
    "flickr": GraphConfig("flickr", 89_250, 900_000, 256, (16, 32, 64), 1),
    "proteins": GraphConfig("proteins", 132_534, 39_600_000, 256, (32,), 2),
    "reddit": GraphConfig("reddit", 232_965, 114_615_891, 256, (8, 16, 32, 64), 3),
    "products": GraphConfig("products", 2_449_029, 61_900_000, 256, (32,), 4),
    # SURVEY §8(f) f3 secondary points (not BASELINE.json configs; graph seeds continue the index):
    # Yelp-shaped at the paper's hidden dimension 384 (Table 3) and k = 96,
    # so CBSR indices are uint16; N and nnz from Table 1.
    "yelp": GraphConfig("yelp", 716_847, 13_954_819, 384, (96,), 5),
    # proteins / products at Table 1's directed edge counts (R13)
    "proteins_directed": GraphConfig("proteins_directed", 132_534, 79_122_504, 256, (32,), 6),
    "products_directed": GraphConfig("products_directed", 2_449_029, 123_718_280, 256, (32,), 7),
    # SURVEY §8(d) d.2 sensitivity point: the Reddit-shaped graph with a flatter degree tail (gamma = 2.5)
    "reddit_g25": GraphConfig("reddit_g25", 232_965, 114_615_891, 256, (32,), 8, 2.5),
}


def config_graph(name: str, rows: tuple[int, int] | None = None) -> Csr:
    c = CONFIGS[name]
    return power_law_graph(c.n, c.nnz, c.seed, gamma=c.gamma, rows=rows)


# --------------------------------------------------------------------------------------------
# Adversarial feature generators for the top-k parity suite.
# --------------------------------------------------------------------------------------------
def quantized_f32(shape, seed: int) -> np.ndarray:
    """Values in {-2,...,2} * 0.5 — heavy ties at the k-boundary."""
    g = np.random.default_rng(seed)
    return (g.integers(-4, 5, size=shape).astype(np.float32) * np.float32(0.25))


def special_f32(shape, seed: int) -> np.ndarray:
    """Mix of +-0.0, +-Inf, subnormals, huge values and exact duplicates (NaN-free)."""
    g = np.random.default_rng(seed)
    pool = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 1e-40, -1e-40, 3.4e38, -3.4e38,
                     1.0, -1.0, 0.5, 2.0, -2.0], dtype=np.float32)
    x = g.standard_normal(size=shape).astype(np.float32)
    mask = g.random(size=shape) < 0.5
    x[mask] = pool[g.integers(0, pool.size, size=int(mask.sum()))]
    return x


def random_csr(n_rows: int, n_cols: int, avg_deg: float, seed: int, duplicates: bool = False,
               empty_rows: float = 0.1, weights: str = "normal") -> Csr:
    """Small uniform random CSR for parity tests (ragged degrees, empty rows, optional duplicates)."""
    g = np.random.default_rng(seed)
    deg = g.poisson(avg_deg, size=n_rows).astype(np.int64)
    deg[g.random(n_rows) < empty_rows] = 0
    if not duplicates:
        deg = np.minimum(deg, n_cols)
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    cols = []
    for d in deg:
        if duplicates:
            c = np.sort(g.integers(0, n_cols, size=int(d)))
        else:
            c = np.sort(g.choice(n_cols, size=int(d), replace=False))
        cols.append(c)
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    if weights == "normal":
        val = g.standard_normal(size=col.size).astype(np.float32)
    elif weights == "mean":
        val = np.repeat(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0), deg).astype(np.float32)
    else:
        val = np.ones(col.size, dtype=np.float32)
    return Csr(row_ptr, col, val, n_cols)
