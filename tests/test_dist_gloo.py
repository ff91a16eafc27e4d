"""Multi-GPU path on CPU: world_size-2 gloo run of the partition -> slot remap -> all-gather ->
per-rank compute -> reduce-scatter sequence (paper_2312_08656_b200.dist), with the CPU oracle injected
as the per-rank compute. Each rank's Y rows and dXs rows must equal the single-process oracle result
for the whole graph; the gathered mask must equal the 1-process top-k mask."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2312_08656_b200.dist import DistributedMaxk
from paper_2312_08656_b200.partition import nnz_balance, partition_rows_by_nnz, remap_columns, split_local_remote

N, NNZ, H, K, SEED = 700, 9000, 32, 8, 77


class OracleOps:
    """CPU oracle in the role of the per-rank kernels (tests only)."""

    def __init__(self, row_ptr, col, val, part, h, k, own_block_of=None):
        """own_block_of=g: the CBSR passed in is rank g's R_max-row slot block only (split local ops)."""
        self.row_ptr, self.col, self.val, self.part, self.h, self.k = row_ptr, col, val, part, h, k
        real = np.zeros(part.n_slots, dtype=bool)
        for g in range(part.world):
            r0, r1 = part.rows(g)
            real[g * part.r_max: g * part.r_max + (r1 - r0)] = True
        if own_block_of is not None:
            real = real[own_block_of * part.r_max: (own_block_of + 1) * part.r_max]
        self.real = real

    def topk(self, x, data_out, idx_out):
        d, i = oracle.topk_cbsr(x.numpy(), self.k)
        data_out.copy_(torch.from_numpy(d))
        idx_out.copy_(torch.from_numpy(i.astype(np.uint8)))

    def _dense(self, sp_data, sp_idx):
        d = sp_data.numpy().copy()
        i = sp_idx.numpy().astype(np.int32)
        d[~self.real] = 0.0
        i[~self.real] = np.arange(self.k)  # padding slots: any valid, distinct pattern with zero data
        return d, i

    def forward(self, sp_data, sp_idx, y, accumulate=False):
        d, i = self._dense(sp_data, sp_idx)
        out = torch.from_numpy(oracle.spgemm_fwd(self.row_ptr, self.col, self.val, d, i, self.h).astype(np.float32))
        y.add_(out) if accumulate else y.copy_(out)

    def backward(self, dy, sp_idx, d_out, accumulate=False):
        _, i = self._dense(torch.zeros(sp_idx.shape), sp_idx)
        out = torch.from_numpy(oracle.sspmm_bwd(self.row_ptr, self.col, self.val, dy.numpy(), i).astype(np.float32))
        d_out.add_(out) if accumulate else d_out.copy_(out)

    def add(self, dst, src):
        dst.add_(src)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results, split=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        deg, _ = synth.power_law_degrees(N, NNZ, SEED)
        rp_full = np.zeros(N + 1, np.int64)
        np.cumsum(deg, out=rp_full[1:])
        part = partition_rows_by_nnz(rp_full, world)
        r0, r1 = part.rows(rank)
        g = synth.power_law_graph(N, NNZ, SEED, rows=(r0, r1))
        col = remap_columns(g.col_idx, part)
        x = synth.normal_f32((r1 - r0, H), 1, row_offset=r0)
        dy = synth.normal_f32((r1 - r0, H), 2, row_offset=r0)
        ops = OracleOps(g.row_ptr, col, g.val, part, H, K)
        split_ops = None
        if split:  # f2: local-column edges overlap the all-gather / reduce-scatter
            (lr, lc, lv), (rr, rc, rv) = split_local_remote(g.row_ptr, col, g.val, part, rank)
            split_ops = (OracleOps(lr, lc, lv, part, H, K, own_block_of=rank), OracleOps(rr, rc, rv, part, H, K))
        agg = DistributedMaxk(part, rank, ops, H, K, torch.device("cpu"), idx_dtype=torch.uint8, split_ops=split_ops)
        agg.sp_data.zero_()
        agg.sp_idx.zero_()
        y, d = agg.step(torch.from_numpy(x), torch.from_numpy(dy))
        results[rank] = (r0, r1, y.numpy().copy(), d.numpy().copy(), agg.sp_idx.numpy().copy(), part.bounds.copy(),
                         part.r_max)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,split", [(2, False), (3, False), (2, True), (3, True), (4, True)])
def test_distributed_matches_single_process(world, split):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), results, split), nprocs=world, join=True,
                       start_method="spawn")
    full = synth.power_law_graph(N, NNZ, SEED)
    x = synth.normal_f32((N, H), 1)
    dy = synth.normal_f32((N, H), 2)
    d_ref, i_ref = oracle.topk_cbsr(x, K)
    y_ref = oracle.spgemm_fwd(full.row_ptr, full.col_idx, full.val, d_ref, i_ref, H)
    dx_ref = oracle.sspmm_bwd(full.row_ptr, full.col_idx, full.val, dy, i_ref)
    covered = 0
    for rank in range(world):
        r0, r1, y, d, idx_slots, bounds, r_max = results[rank]
        covered += r1 - r0
        np.testing.assert_allclose(y, y_ref[r0:r1], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(d, dx_ref[r0:r1], rtol=1e-5, atol=1e-5)
        # the all-gathered mask is the 1-process mask at every real slot (bit-exact)
        for g in range(world):
            a, b = bounds[g], bounds[g + 1]
            assert np.array_equal(idx_slots[g * r_max: g * r_max + (b - a)].astype(np.int32), i_ref[a:b])
    assert covered == N


def test_partition_balances_nnz_and_maps_slots():
    g = synth.power_law_graph(5000, 200000, seed=4)
    for world in (1, 2, 4, 8):
        part = partition_rows_by_nnz(g.row_ptr, world)
        assert part.bounds[0] == 0 and part.bounds[-1] == 5000 and np.all(np.diff(part.bounds) > 0)
        per = nnz_balance(g.row_ptr, part)
        assert per.sum() == g.nnz
        dmax = int(np.diff(g.row_ptr).max())
        assert per.max() - per.min() <= 2 * dmax + 1  # a row is never split: balance within a hub's size
        slots = part.slot_of(np.arange(5000))
        assert np.unique(slots).size == 5000 and slots.max() < part.n_slots
        assert np.array_equal(part.node_of_slot(slots), np.arange(5000))
        assert np.array_equal(remap_columns(g.col_idx, part), slots[g.col_idx])
