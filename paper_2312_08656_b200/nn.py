"""MaxK-GNN layer as a torch.autograd.Function over the C-ABI kernels (full-layer timing).

One layer of the paper's dataflow (Fig. 5; Eq. 1; Eq. 3):
    forward   Z = X W + b                                   (GEMM: cuBLAS, or fused with the top-k below)
              (sp_data, sp_idx) = max-k(Z)                  (maxk_topk_cbsr / maxk_linear_topk_cbsr)
              Y = A · CBSR                                  (maxk_spgemm_fwd)
    backward  dXs = (A^T dY) at sp_idx                      (maxk_sspmm_bwd)
              dZ  = scatter(dXs, sp_idx)                    (maxk_cbsr_scatter; MaxK Def. ii)
              dW = X^T dZ, dX = dZ W^T, db = sum(dZ)        (GEMMs: cuBLAS)
The aggregation operator A is the graph's CSR with its values (1/deg for the SAGE mean aggregator,
PAPER.md:315). Everything between the two GEMMs runs in libmaxk.so; no CPU fallback.
"""
from __future__ import annotations

import torch

from . import maxk


class Graph:
    """A CSR graph resident on the GPU with its work plan (built once, reused by every layer and step)."""

    def __init__(self, row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, h: int, k: int):
        self.row_ptr, self.col_idx, self.val = row_ptr, col_idx, val
        self.n_rows = row_ptr.shape[0] - 1
        self.n_cols = n_cols
        rp = row_ptr[[0, -1]].tolist()
        self.nnz = int(rp[1] - rp[0])
        self.plan = maxk.maxk_plan_create(row_ptr, h, k)


class MaxKAggregate(torch.autograd.Function):
    """Y = A · max-k(Z) with the backward of Eq. 3 (sampled at the forward mask) and MaxK's scatter."""

    @staticmethod
    def forward(ctx, z: torch.Tensor, graph: Graph, k: int):
        z = z.contiguous()
        h = z.shape[1]
        if maxk.pairs_default(h, k) and z.data_ptr() % 16 == 0:  # k in {8, 16}: the forward gathers the pair layout
            sp_data, sp_idx, sp_pairs = maxk.maxk_topk_cbsr_pairs(
                z, k, banked=maxk.banked_default(h, k, graph.n_rows, graph.nnz))  # k = 16: the balanced order
            y = maxk.maxk_spgemm_fwd_pairs(graph.row_ptr, graph.col_idx, graph.val, graph.n_cols, graph.nnz, sp_pairs,
                                           h, plan=graph.plan)
        elif maxk.banked_default(h, k, graph.n_rows, graph.nnz) and maxk.float4_rows(z):  # k in {32, 64, 128}: the bank-balanced copy
            sp_data, sp_idx, sp_bdata, sp_bidx = maxk.maxk_topk_cbsr_banked(z, k)
            y = maxk.maxk_spgemm_fwd(graph.row_ptr, graph.col_idx, graph.val, graph.n_cols, graph.nnz, sp_bdata,
                                     sp_bidx, h, plan=graph.plan)
        else:
            sp_data, sp_idx = maxk.maxk_topk_cbsr(z, k)
            y = maxk.maxk_spgemm_fwd(graph.row_ptr, graph.col_idx, graph.val, graph.n_cols, graph.nnz, sp_data,
                                     sp_idx, h, plan=graph.plan)
        ctx.save_for_backward(sp_idx)
        ctx.graph, ctx.h = graph, z.shape[1]
        return y

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        (sp_idx,) = ctx.saved_tensors
        g = ctx.graph
        d_sp = maxk.maxk_sspmm_bwd(g.row_ptr, g.col_idx, g.val, g.n_cols, g.nnz, dy.contiguous(), sp_idx, plan=g.plan)
        dz = maxk.maxk_cbsr_scatter(d_sp, sp_idx, ctx.h)
        return dz, None, None


class MaxKLinearAggregate(torch.autograd.Function):
    """Y = A · max-k(X W + b) with X, W in bf16: the forward's GEMM and top-k are ONE fused tcgen05 kernel
    (maxk_linear_topk_cbsr), so Z never reaches HBM; the backward uses cuBLAS for dW, dX."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, w_t: torch.Tensor, b: torch.Tensor, graph: Graph, k: int):
        sp_data, sp_idx = maxk.maxk_linear_topk_cbsr(x.contiguous(), w_t.contiguous(), k, bias=b)
        h = w_t.shape[0]
        y = maxk.maxk_spgemm_fwd(graph.row_ptr, graph.col_idx, graph.val, graph.n_cols, graph.nnz, sp_data, sp_idx,
                                 h, plan=graph.plan)
        ctx.save_for_backward(x, w_t, sp_idx)
        ctx.graph, ctx.h = graph, h
        return y

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        x, w_t, sp_idx = ctx.saved_tensors
        g = ctx.graph
        d_sp = maxk.maxk_sspmm_bwd(g.row_ptr, g.col_idx, g.val, g.n_cols, g.nnz, dy.contiguous(), sp_idx, plan=g.plan)
        dz = maxk.maxk_cbsr_scatter(d_sp, sp_idx, ctx.h)          # fp32 [n, h]
        dz16 = dz.to(torch.bfloat16)
        dx = dz16 @ w_t                                            # [n, f]
        dw_t = dz16.t() @ x                                        # [h, f]
        db = dz.sum(0)
        return dx, dw_t, db, None, None


class MaxKGraphConv(torch.nn.Module):
    """One MaxK-GNN layer: Linear(f_in -> h) -> MaxK(k) -> aggregation over the graph (SAGE-mean values).

    fused=True keeps X/W in bf16 and runs the forward GEMM + top-k as the fused tcgen05 kernel (h in {128, 256},
    f_in % 64 == 0, k <= 64); otherwise a cuBLAS fp32 GEMM feeds maxk_topk_cbsr.
    """

    def __init__(self, f_in: int, h: int, k: int, fused: bool = False, device=None):
        super().__init__()
        self.f_in, self.h, self.k, self.fused = f_in, h, k, fused
        dt = torch.bfloat16 if fused else torch.float32
        self.w_t = torch.nn.Parameter((torch.randn(h, f_in, device=device) / f_in ** 0.5).to(dt))
        self.b = torch.nn.Parameter(torch.zeros(h, device=device))

    def forward(self, x: torch.Tensor, graph: Graph) -> torch.Tensor:
        if self.fused:
            return MaxKLinearAggregate.apply(x.to(torch.bfloat16), self.w_t, self.b, graph, self.k)
        z = torch.addmm(self.b, x, self.w_t.t())
        return MaxKAggregate.apply(z, graph, self.k)
