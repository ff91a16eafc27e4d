"""B200-native MaxK-GNN layer hot path (arXiv 2312.08656).

The product is libmaxk.so (csrc/, C-ABI in include/maxk.h). This package is its thin Python face:
  maxk       ctypes binding with the C-ABI's names (argument marshalling only)
  layer      a graph-resident aggregation object running top-k -> SpGEMM fwd and SSpMM bwd
  partition  the nnz-balanced row partitioner and slot remap for multi-GPU (host logic)
  dist       the NCCL all-gather / reduce-scatter glue (torch.distributed)
  traffic    the paper's byte model (§4.3) used for roofline accounting
There is no CPU fallback anywhere on this path.
"""
from .maxk import (MaxkError, Plan, launch_count, load, maxk_cbsr_scatter, maxk_plan_create,  # noqa: F401
                   maxk_spgemm_fwd, maxk_sspmm_bwd, maxk_topk_cbsr, version)

__all__ = ["MaxkError", "Plan", "launch_count", "load", "maxk_cbsr_scatter", "maxk_plan_create", "maxk_spgemm_fwd", "maxk_sspmm_bwd",
           "maxk_topk_cbsr", "version"]
