"""Byte model of the hot path (paper §4.3) for roofline accounting.

Paper terms:
  forward  CBSR gathered once per edge: (4 + b) * k * nnz bytes        (b = index bytes; "5 x dim_k x nnz" at b=1)
  backward reads 4*N*H (dense dY prefetch) + (4 + b) * k * nnz, writes 4 * k * nnz
  SpMM baseline (dense features): 4 * H * nnz; reduction = 1 - (4+b)k / (4H)
We add what every implementation must also move (SURVEY d.5): the CSR arrays (8(N+1) + 8 nnz), the
dense input/output rows and the zeroing of d_sp_data. These are the ALGORITHMIC bytes B_alg of each
kernel; B_min is the unique-byte (compulsory) HBM traffic.
"""
from __future__ import annotations


def spmm_read_bytes(nnz: int, h: int) -> int:
    """Dense-feature SpMM's per-edge feature traffic, the baseline of §4.3."""
    return 4 * h * nnz


def spgemm_feature_bytes(nnz: int, k: int, b: int) -> int:
    """§4.3 forward: CBSR rows read nnz times."""
    return (4 + b) * k * nnz


def traffic_reduction(h: int, k: int, b: int) -> float:
    """1 - (4+b)k/(4h): 90.625% at h=256, k=16, b=2; 92.1875% at b=1."""
    return 1.0 - (4 + b) * k / (4.0 * h)


def sspmm_bytes(n: int, nnz: int, h: int, k: int, b: int) -> tuple[int, int]:
    """§4.3 backward (reads, writes) = (4NH + (4+b) k nnz, 4 k nnz)."""
    return 4 * n * h + (4 + b) * k * nnz, 4 * k * nnz


def b_alg(n: int, n_cols: int, nnz: int, h: int, k: int, b: int) -> dict:
    """Algorithmic bytes per launch of each kernel (graded basis, SURVEY d.5)."""
    csr = 8 * (n + 1) + 8 * nnz
    topk = 4 * n_cols * h + (4 + b) * n_cols * k
    fwd = csr + (4 + b) * k * nnz + 4 * n * h
    bwd = csr + 4 * n * h + (4 + b) * k * nnz + 4 * k * nnz + 4 * n_cols * k
    return {"topk": topk, "fwd": fwd, "bwd": bwd, "layer": topk + fwd + bwd}


def b_min(n: int, n_cols: int, nnz: int, h: int, k: int, b: int) -> dict:
    """Unique bytes (strict HBM lower bound) per kernel."""
    csr = 8 * (n + 1) + 8 * nnz
    topk = 4 * n_cols * h + (4 + b) * n_cols * k
    fwd = csr + (4 + b) * n_cols * k + 4 * n * h
    bwd = csr + 4 * n * h + b * n_cols * k + 4 * n_cols * k
    return {"topk": topk, "fwd": fwd, "bwd": bwd, "layer": topk + fwd + bwd}
