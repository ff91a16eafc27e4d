"""Graph-resident MaxK aggregation: one object per (graph, h, k), buffers preallocated in HBM.

A "layer pass" (one step of the hot path) is
    sp_data, sp_idx = maxk_topk_cbsr(X)                 (Eq. 1; + the pair / bank-balanced copy where it exists)
    Y               = maxk_spgemm_fwd(A, sp_data, sp_idx) (Eq. 3 left)
    dXs             = maxk_sspmm_bwd(A, dY, sp_idx)       (Eq. 3 right)
all on one CUDA stream through the C-ABI. Nothing is allocated per pass.
"""
from __future__ import annotations

import torch

from . import maxk


class MaxkAggregation:
    def __init__(self, row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, h: int, k: int,
                 use_plan: bool = True, stream=None):
        if not row_ptr.is_cuda:
            raise ValueError("graph arrays must be CUDA tensors")
        self.row_ptr, self.col_idx, self.val = row_ptr, col_idx, val
        self.n_rows = row_ptr.shape[0] - 1
        self.n_cols = n_cols
        self.h, self.k = h, k
        rp = row_ptr[[0, -1]].tolist()
        self.nnz = int(rp[1] - rp[0])
        self.stream = stream
        self.plan = maxk.maxk_plan_create(row_ptr, h, k, stream=stream) if use_plan else None
        dev = row_ptr.device
        self.sp_data = torch.empty((n_cols, k), dtype=torch.float32, device=dev)
        self.sp_idx = torch.empty((n_cols, k), dtype=maxk.idx_dtype(h), device=dev)
        self.y = torch.empty((self.n_rows, h), dtype=torch.float32, device=dev)
        self.d_sp_data = torch.empty((n_cols, k), dtype=torch.float32, device=dev)
        # the forward gathers the CBSR pair layout where it exists (k in {8, 16}: one 128-byte line per row)
        self.sp_pairs = (torch.empty((n_cols, k, 2), dtype=torch.int32, device=dev)
                         if maxk.pairs_default(h, k) else None)
        self._pairs_stale = False  # a top-k call could not write the pair layout: the forward reads the two blocks
        # k in {32, 64, 128}: the forward gathers the bank-balanced copy of the CBSR (its replicated row buffers then
        # conflict only on unbalanced pairs); the backward keeps the column-ordered sp_idx
        banked = maxk.banked_default(h, k, self.n_rows, self.nnz)
        self._pairs_banked = banked and self.sp_pairs is not None  # k = 16: the balanced pair order instead
        banked = banked and k != 16  # the two-block copy: k in {32, 64, 128}
        self.sp_bdata = torch.empty((n_cols, k), dtype=torch.float32, device=dev) if banked else None
        self.sp_bidx = torch.empty((n_cols, k), dtype=maxk.idx_dtype(h), device=dev) if banked else None
        self._banked_stale = False

    @staticmethod
    def _float4_rows(x: torch.Tensor) -> bool:
        """x rows are 16-byte aligned (what the pair-writing top-k kernel loads)."""
        return x.data_ptr() % 16 == 0 and (x.shape[0] <= 1 or x.stride(0) % 4 == 0) and x.stride(-1) == 1

    def topk(self, x: torch.Tensor, row_offset: int = 0):
        """CBSR of x written into rows [row_offset, row_offset + x.shape[0]) of the resident CBSR buffers."""
        n = x.shape[0]
        rows = slice(row_offset, row_offset + n)
        with maxk.nvtx_range("maxk/topk"):
            if self.sp_pairs is not None and self._float4_rows(x):
                maxk.maxk_topk_cbsr_pairs(x, self.k, self.sp_data[rows], self.sp_idx[rows], self.sp_pairs[rows],
                                          stream=self.stream, banked=self._pairs_banked)
                if row_offset == 0 and n == self.n_cols:
                    self._pairs_stale = False  # every row refreshed
            elif self.sp_bdata is not None and self._float4_rows(x):
                maxk.maxk_topk_cbsr_banked(x, self.k, self.sp_data[rows], self.sp_idx[rows], self.sp_bdata[rows],
                                           self.sp_bidx[rows], stream=self.stream)
                if row_offset == 0 and n == self.n_cols:
                    self._banked_stale = False
            else:
                maxk.maxk_topk_cbsr(x, self.k, self.sp_data[rows], self.sp_idx[rows], stream=self.stream)
                self._pairs_stale = self.sp_pairs is not None
                self._banked_stale = self.sp_bdata is not None
        return self.sp_data, self.sp_idx

    def forward(self):
        with maxk.nvtx_range("maxk/spgemm_fwd"):
            if self.sp_pairs is not None and not self._pairs_stale:
                return maxk.maxk_spgemm_fwd_pairs(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz,
                                                  self.sp_pairs, self.h, y=self.y, plan=self.plan, stream=self.stream)
            data, idx = ((self.sp_bdata, self.sp_bidx) if self.sp_bdata is not None and not self._banked_stale
                         else (self.sp_data, self.sp_idx))
            return maxk.maxk_spgemm_fwd(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz, data, idx,
                                        self.h, y=self.y, plan=self.plan, stream=self.stream)

    def backward(self, dy: torch.Tensor):
        with maxk.nvtx_range("maxk/sspmm_bwd"):
            return maxk.maxk_sspmm_bwd(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz, dy, self.sp_idx,
                                       d_sp_data=self.d_sp_data, plan=self.plan, stream=self.stream)

    def step(self, x: torch.Tensor, dy: torch.Tensor):
        """One pass of the whole hot path on a single GPU (n_cols == n_rows)."""
        with maxk.nvtx_range("maxk/layer_step"):
            self.topk(x)
            self.forward()
            self.backward(dy)
        return self.y, self.d_sp_data

    def capture_step(self, x: torch.Tensor, dy: torch.Tensor) -> "torch.cuda.CUDAGraph":
        """Capture one layer pass (top-k -> forward -> backward, all on the C-ABI kernels) into a CUDA graph.

        graph.replay() re-runs it on the same device buffers: copy each step's inputs into x and dy, read y and
        d_sp_data afterwards. Safe to replay because the kernels' scheduling counters are reset on the device by
        the last warp of every launch. Removes the per-launch host overhead of launch-bound (small) graphs."""
        s = torch.cuda.Stream(device=x.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up outside the capture (first-call CUDA attribute setup)
            self.step(x, dy)
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self.step(x, dy)
        return graph

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None
