"""Multi-GPU path on ONE GPU (SURVEY.md §4 layer 3, "virtual-rank test"): partition -> slot remap -> per-rank
CUDA kernels on n_rows x Nc row blocks -> emulated all-gather / reduce-scatter (device copies / sums), for
G in {2, 4, 8}. The CBSR must equal the 1-GPU CBSR bit-exactly, Y and dXs must match the 1-GPU result and
the oracle within tolerance. (The NCCL calls themselves are covered by tests/test_dist_gloo.py.)"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200.dist import CudaOps
from paper_2312_08656_b200.layer import MaxkAggregation
from paper_2312_08656_b200.partition import partition_rows_by_nnz, remap_columns, split_local_remote

pytestmark = pytest.mark.gpu

N, NNZ, H, K, SEED = 20000, 800000, 256, 32, 99


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rows_close(gpu, ref, what):
    err = np.abs(gpu.astype(np.float64) - ref).max(axis=1)
    tol = 1e-5 * (1.0 + np.abs(ref).max(axis=1))
    assert np.all(err <= tol), f"{what}: worst {float((err / tol).max()):.2f} x tol"


@pytest.mark.parametrize("world,split", [(2, False), (4, False), (8, False), (2, True), (8, True)])
def test_virtual_ranks_match_single_gpu(world, split):
    full = synth.power_law_graph(N, NNZ, SEED)
    x = synth.normal_f32((N, H), 1)
    dy = synth.normal_f32((N, H), 2)
    # 1-GPU reference run
    one = MaxkAggregation(_cuda(full.row_ptr), _cuda(full.col_idx), _cuda(full.val), N, H, K)
    y1, d1 = one.step(_cuda(x), _cuda(dy))
    y1, d1 = y1.cpu().numpy(), d1.cpu().numpy()
    cb1 = one.sp_idx.cpu().numpy()
    one.close()

    part = partition_rows_by_nnz(full.row_ptr, world)
    R, Nc = part.r_max, part.n_slots
    ranks = []
    for g in range(world):
        r0, r1 = part.rows(g)
        blk = synth.power_law_graph(N, NNZ, SEED, rows=(r0, r1))
        col = remap_columns(blk.col_idx, part)
        ops = CudaOps(_cuda(blk.row_ptr), _cuda(col), _cuda(blk.val), Nc, H, K)
        sd = torch.zeros((Nc, K), dtype=torch.float32, device="cuda")
        si = torch.zeros((Nc, K), dtype=torch.uint8, device="cuda")
        rk = dict(r0=r0, r1=r1, ops=ops, sd=sd, si=si, x=_cuda(x[r0:r1]), dy=_cuda(dy[r0:r1]))
        if split:  # f2: local-column edges (own slot block only) and remote-column edges as separate ops
            (lr, lc, lv), (rr, rc, rv) = split_local_remote(blk.row_ptr, col, blk.val, part, g)
            rk["ops_l"] = CudaOps(_cuda(lr), _cuda(lc), _cuda(lv), R, H, K)
            rk["ops_r"] = CudaOps(_cuda(rr), _cuda(rc), _cuda(rv), Nc, H, K)
        ranks.append(rk)
    for g, rk in enumerate(ranks):  # local top-k into the rank's slot block
        n = rk["r1"] - rk["r0"]
        rk["ops"].topk(rk["x"], rk["sd"][g * R:g * R + n], rk["si"][g * R:g * R + n])
    if split:  # the local-column forward runs BEFORE the all-gather: it may only need the rank's own block
        for g, rk in enumerate(ranks):
            rk["y"] = torch.empty((rk["r1"] - rk["r0"], H), dtype=torch.float32, device="cuda")
            rk["ops_l"].forward(rk["sd"][g * R:(g + 1) * R], rk["si"][g * R:(g + 1) * R], rk["y"])
    for rk in ranks:  # emulated all_gather_into_tensor
        for g, src in enumerate(ranks):
            rk["sd"][g * R:(g + 1) * R].copy_(src["sd"][g * R:(g + 1) * R])
            rk["si"][g * R:(g + 1) * R].copy_(src["si"][g * R:(g + 1) * R])
    ys, parts = [], []
    for g, rk in enumerate(ranks):
        dp = torch.empty((Nc, K), dtype=torch.float32, device="cuda")
        if split:
            y = rk["y"]
            rk["ops_r"].forward(rk["sd"], rk["si"], y, accumulate=True)
            rk["ops_r"].backward(rk["dy"], rk["si"], dp)
            rk["dt"] = torch.empty((R, K), dtype=torch.float32, device="cuda")
            rk["ops_l"].backward(rk["dy"], rk["si"][g * R:(g + 1) * R], rk["dt"])
        else:
            y = torch.empty((rk["r1"] - rk["r0"], H), dtype=torch.float32, device="cuda")
            rk["ops"].forward(rk["sd"], rk["si"], y)
            rk["ops"].backward(rk["dy"], rk["si"], dp)
        ys.append(y)
        parts.append(dp)
    red = torch.stack(parts).sum(0)  # emulated reduce_scatter_tensor (sum)
    if split:  # each rank adds its local-target partial to its reduce-scatter block
        for g, rk in enumerate(ranks):
            blkv = red[g * R:(g + 1) * R].contiguous()
            rk["ops_l"].add(blkv, rk["dt"])
            red[g * R:(g + 1) * R] = blkv
    y_all = torch.cat(ys).cpu().numpy()
    slots = part.slot_of(np.arange(N))
    d_all = red.cpu().numpy()[slots]
    # the gathered mask at every real slot is the 1-GPU mask (bit-exact)
    assert np.array_equal(ranks[0]["si"].cpu().numpy()[slots], cb1)
    _rows_close(y_all, y1.astype(np.float64), "Y vs 1-GPU")
    _rows_close(d_all, d1.astype(np.float64), "dXs vs 1-GPU")
    rows = np.unique(np.concatenate([np.argsort(-np.diff(full.row_ptr))[:20], np.arange(0, N, 97)]))
    rd, ri = oracle.topk_cbsr(x, K)
    _rows_close(y_all[rows], oracle.spgemm_fwd(full.row_ptr, full.col_idx, full.val, rd, ri, H, rows=rows), "Y vs oracle")
    _rows_close(d_all[rows], oracle.sspmm_bwd(full.row_ptr, full.col_idx, full.val, dy, ri, rows=rows),
                "dXs vs oracle")
    for rk in ranks:
        rk["ops"].close()
        if split:
            rk["ops_l"].close()
            rk["ops_r"].close()
