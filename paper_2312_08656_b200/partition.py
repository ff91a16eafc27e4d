"""nnz-balanced row partitioner and slot remap for the multi-GPU path.

The paper is single-GPU; its partitioning remark is the only hook. We
shard A by contiguous row blocks [r_g, r_{g+1}) with row_ptr[r_g] ~= g * nnz / G, so every GPU owns the
same number of edges (the unit of work of both kernels). The CBSR rows are exchanged through one
equal-count NCCL all-gather, so each rank's CBSR rows live in a padded "slot" block of R_max rows:
    slot(j) = g(j) * R_max + (j - r_{g(j)}),   Nc = G * R_max.
col_idx is remapped to slots once, at partition time, so the kernels see an ordinary n_rows x Nc CSR
block and are identical for 1 and G GPUs. Host logic only (numpy), no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RowPartition:
    bounds: np.ndarray  # int64 [G+1], bounds[0] = 0, bounds[G] = n
    r_max: int          # rows per slot block

    @property
    def world(self) -> int:
        return int(self.bounds.shape[0] - 1)

    @property
    def n_slots(self) -> int:
        return self.world * self.r_max

    def rows(self, g: int) -> tuple[int, int]:
        return int(self.bounds[g]), int(self.bounds[g + 1])

    def slot_of(self, j: np.ndarray) -> np.ndarray:
        j = np.asarray(j, dtype=np.int64)
        g = np.searchsorted(self.bounds, j, side="right") - 1
        return g * self.r_max + (j - self.bounds[g])

    def node_of_slot(self, s: np.ndarray) -> np.ndarray:
        s = np.asarray(s, dtype=np.int64)
        g, off = s // self.r_max, s % self.r_max
        return self.bounds[g] + off


def partition_rows_by_nnz(row_ptr: np.ndarray, world: int) -> RowPartition:
    """Contiguous row blocks with ~equal nnz: r_g = first row whose row_ptr >= g*nnz/G (binary search).

    A row is never split across GPUs; each block is non-empty when n >= world.
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = row_ptr.shape[0] - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    nnz = int(row_ptr[-1] - row_ptr[0])
    targets = row_ptr[0] + (np.arange(1, world, dtype=np.float64) * nnz / world)
    cuts = np.searchsorted(row_ptr, targets, side="left").astype(np.int64)
    bounds = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
    # keep blocks non-empty where possible (tiny graphs, extreme hubs)
    for g in range(1, world):
        lo = bounds[g - 1] + (1 if n >= world else 0)
        hi = n - (world - g if n >= world else 0)
        bounds[g] = min(max(bounds[g], lo), hi)
    r_max = int(max(1, (bounds[1:] - bounds[:-1]).max())) if n > 0 else 1
    return RowPartition(bounds, r_max)


def remap_columns(col_idx: np.ndarray, part: RowPartition) -> np.ndarray:
    """col_idx (node ids) -> slots, int32. Nc must fit int32 (maxk.h n_cols <= INT32_MAX)."""
    if part.n_slots > np.iinfo(np.int32).max:
        raise ValueError("slot space exceeds int32")
    return part.slot_of(col_idx).astype(np.int32)


def nnz_balance(row_ptr: np.ndarray, part: RowPartition) -> np.ndarray:
    """Edges owned by each rank."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    return row_ptr[part.bounds[1:]] - row_ptr[part.bounds[:-1]]


def split_local_remote(row_ptr: np.ndarray, col_slots: np.ndarray, val: np.ndarray, part: RowPartition, rank: int):
    """Split a rank's CSR block (columns already in slot space) into the edges whose column is one of the rank's
    own slots and the rest, keeping each row's edge order (the local edges need only this
    rank's CBSR rows, so they run while the all-gather is in flight, and their backward reductions target only
    this rank's block, so they run while the reduce-scatter is in flight).

    Returns (local, remote), each (row_ptr int64, col int32, val float32) over the same rows:
      local  columns shifted to [0, R_max) — pair with the rank's slot block of the CBSR (n_cols = R_max);
      remote columns in the full slot space [0, Nc) (n_cols = Nc), none in the rank's own block.
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col_slots, dtype=np.int64)
    val = np.asarray(val, dtype=np.float32)
    n = row_ptr.shape[0] - 1
    base = int(row_ptr[0])
    col = col[base:int(row_ptr[-1])] if col.shape[0] != int(row_ptr[-1] - row_ptr[0]) else col
    val = val[base:int(row_ptr[-1])] if val.shape[0] != int(row_ptr[-1] - row_ptr[0]) else val
    R = part.r_max
    is_local = (col // R) == rank
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    out = []
    for mask, shift in ((is_local, rank * R), (~is_local, 0)):
        cnt = np.bincount(rows[mask], minlength=n).astype(np.int64)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(cnt, out=rp[1:])
        out.append((rp, (col[mask] - shift).astype(np.int32), val[mask]))
    return out[0], out[1]

