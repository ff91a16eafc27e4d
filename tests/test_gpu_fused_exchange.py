"""The row-partitioned layer with its exchanges fused into the compute kernels:
the all-gather into the top-k (maxk_topk_cbsr_multi writes each rank's CBSR block into every replica) and the
reduce-scatter into the backward (maxk_sspmm_bwd_owners reduces each slot's dXs straight into its owner's block).

On the one GPU this run has, the G virtual ranks' replicas and owner blocks are buffers of this device and the
ranks' kernels run one after another (none waits on another); on an NVLink node the same pointers would be peers'
memory mapped into the process. Bar: every replica's mask bit-exact against the oracle at every real slot, the
ranks' Y rows and the owners' dXs rows against the fp64 oracle (north-star tolerance)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200 import maxk
from paper_2312_08656_b200.partition import partition_rows_by_nnz, remap_columns

pytestmark = pytest.mark.gpu

N, NNZ, H, SEED = 20000, 800000, 256, 123


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rows_close(gpu, ref, what):
    err = np.abs(gpu.astype(np.float64) - ref).max(axis=1)
    tol = 1e-5 * (1.0 + np.abs(ref).max(axis=1))
    assert np.all(err <= tol), f"{what}: worst {float(np.nanmax(err / tol)):.2f} x tol"


@pytest.mark.parametrize("world,k", [(2, 32), (4, 32), (8, 16), (3, 64)])
@pytest.mark.parametrize("use_plan", [True, False])
def test_fused_allgather_and_reducescatter(world, k, use_plan):
    full = synth.power_law_graph(N, NNZ, SEED)
    x = synth.normal_f32((N, H), 11)
    dy = synth.normal_f32((N, H), 12)
    part = partition_rows_by_nnz(full.row_ptr, world)
    R, Nc = part.r_max, part.n_slots
    sd = [torch.full((Nc, k), float("nan"), device="cuda") for _ in range(world)]  # each rank's replica
    si = [torch.zeros((Nc, k), dtype=torch.uint8, device="cuda") for _ in range(world)]
    ranks = []
    for g in range(world):
        r0, r1 = part.rows(g)
        blk = synth.power_law_graph(N, NNZ, SEED, rows=(r0, r1))
        rp, ci, va = _cuda(blk.row_ptr), _cuda(remap_columns(blk.col_idx, part)), _cuda(blk.val)
        plan = maxk.maxk_plan_create(rp, H, k) if use_plan else None
        ranks.append(dict(r0=r0, r1=r1, rp=rp, ci=ci, va=va, nnz=int(blk.row_ptr[-1]), plan=plan))
    # top-k with the all-gather fused: rank g's rows go to its slot block of EVERY replica (its own first)
    for g, rk in enumerate(ranks):
        n = rk["r1"] - rk["r0"]
        order = [g] + [h for h in range(world) if h != g]
        maxk.maxk_topk_cbsr_multi(_cuda(x[rk["r0"]:rk["r1"]]), k, [sd[h][g * R:g * R + n] for h in order],
                                  [si[h][g * R:g * R + n] for h in order])
    # forward on each rank's own replica; backward with the reduce-scatter fused (owners' blocks zeroed first)
    d_local = [torch.zeros((R, k), device="cuda") for _ in range(world)]
    ptrs = torch.tensor([t.data_ptr() for t in d_local], dtype=torch.int64, device="cuda")
    ys = []
    for g, rk in enumerate(ranks):
        ys.append(maxk.maxk_spgemm_fwd(rk["rp"], rk["ci"], rk["va"], Nc, rk["nnz"], sd[g], si[g], H, plan=rk["plan"]))
        maxk.maxk_sspmm_bwd_owners(rk["rp"], rk["ci"], rk["va"], Nc, rk["nnz"], _cuda(dy[rk["r0"]:rk["r1"]]), si[g], R,
                                   ptrs, plan=rk["plan"])
    torch.cuda.synchronize()
    slots = part.slot_of(np.arange(N))
    rd, ri = oracle.topk_cbsr(x, k)
    for g in range(world):  # every replica holds the full mask and data, bit-exact
        assert np.array_equal(si[g].cpu().numpy()[slots].astype(np.int64), ri)
        assert np.array_equal(sd[g].cpu().numpy()[slots].view(np.uint32), rd.view(np.uint32))
    y_all = torch.cat(ys).cpu().numpy()
    d_all = torch.cat(d_local).cpu().numpy()[slots]
    rows = np.unique(np.concatenate([np.argsort(-np.diff(full.row_ptr))[:20], np.arange(0, N, 53)]))
    _rows_close(y_all[rows], oracle.spgemm_fwd(full.row_ptr, full.col_idx, full.val, rd, ri, H, rows=rows), "Y")
    _rows_close(d_all[rows], oracle.sspmm_bwd(full.row_ptr, full.col_idx, full.val, dy, ri, rows=rows), "dXs")
    for rk in ranks:
        if rk["plan"] is not None:
            rk["plan"].close()


def test_fused_exchange_argument_errors():
    lib = maxk.load()
    x = torch.zeros((16, 256), device="cuda")
    d = torch.empty((16, 32), device="cuda")
    i = torch.empty((16, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):  # more than 8 destinations
        maxk.maxk_topk_cbsr_multi(x, 32, [d] * 9, [i] * 9)
    with pytest.raises(maxk.MaxkError):  # k = 96: no multi-destination top-k
        maxk.maxk_topk_cbsr_multi(x, 96, [torch.empty((16, 96), device="cuda")],
                                  [torch.empty((16, 96), dtype=torch.uint8, device="cuda")])
    rp = torch.zeros(5, dtype=torch.int64, device="cuda")
    ci = torch.zeros(0, dtype=torch.int32, device="cuda")
    va = torch.zeros(0, device="cuda")
    dy = torch.zeros((4, 256), device="cuda")
    si = torch.zeros((8, 32), dtype=torch.uint8, device="cuda")
    ptrs = torch.zeros(3, dtype=torch.int64, device="cuda")
    with pytest.raises(maxk.MaxkError):  # n_cols (8) != n_owners (3) x owner_rows (2)
        maxk.maxk_sspmm_bwd_owners(rp, ci, va, 8, 0, dy, si, 2, ptrs)
    assert lib.maxk_sspmm_bwd_owners(rp.data_ptr(), ci.data_ptr(), va.data_ptr(), 4, 8, 0, dy.data_ptr(), 256,
                                     si.data_ptr(), 256, 32, 1, 4, 2, None, None, None) == 1  # NULL d_owner


class _VirtualPeers:
    """PeerMemoryMaxk's peers on one GPU: every virtual rank's replica and dXs block are buffers of this device;
    the phases run rank after rank, so the barrier has nothing to wait for."""

    def __init__(self, shared, rank):
        self.replicas, self.owner_ptrs, self.dl = shared["replicas"], shared["owner_ptrs"], shared["dls"][rank]

    def barrier(self):
        pass


@pytest.mark.parametrize("world", [2, 4])
def test_peer_memory_layer_pass(world):
    """dist.PeerMemoryMaxk (the layer pass with both exchanges fused into the kernels) with virtual peers: the
    phases of all ranks interleaved in the order its barriers enforce, two passes (buffer reuse)."""
    from paper_2312_08656_b200.dist import CudaOps, PeerMemoryMaxk
    k = 32
    full = synth.power_law_graph(N, NNZ, SEED)
    part = partition_rows_by_nnz(full.row_ptr, world)
    R, Nc = part.r_max, part.n_slots
    shared = {"replicas": [(torch.zeros((Nc, k), device="cuda"), torch.zeros((Nc, k), dtype=torch.uint8, device="cuda"))
                           for _ in range(world)],
              "dls": [torch.zeros((R, k), device="cuda") for _ in range(world)]}
    shared["owner_ptrs"] = torch.tensor([t.data_ptr() for t in shared["dls"]], dtype=torch.int64, device="cuda")
    ranks = []
    for g in range(world):
        r0, r1 = part.rows(g)
        blk = synth.power_law_graph(N, NNZ, SEED, rows=(r0, r1))
        ops = CudaOps(_cuda(blk.row_ptr), _cuda(remap_columns(blk.col_idx, part)), _cuda(blk.val), Nc, H, k)
        ranks.append(PeerMemoryMaxk(part, g, ops, H, k, _VirtualPeers(shared, g)))
    for seed in (21, 22):
        x = synth.normal_f32((N, H), seed)
        dy = synth.normal_f32((N, H), seed + 100)
        for rk in ranks:
            r0, r1 = part.rows(rk.rank)
            rk.topk(_cuda(x[r0:r1]))
        ys = [rk.forward() for rk in ranks]
        ds = [rk.backward(_cuda(dy[slice(*part.rows(rk.rank))])) for rk in ranks]
        torch.cuda.synchronize()
        rd, ri = oracle.topk_cbsr(x, k)
        slots = part.slot_of(np.arange(N))
        for g in range(world):
            assert np.array_equal(shared["replicas"][g][1].cpu().numpy()[slots].astype(np.int64), ri)
        y_all = torch.cat([y.clone() for y in ys]).cpu().numpy()
        d_all = torch.cat([d.clone() for d in ds]).cpu().numpy()
        rows = np.unique(np.concatenate([np.argsort(-np.diff(full.row_ptr))[:20], np.arange(0, N, 71)]))
        _rows_close(y_all[rows], oracle.spgemm_fwd(full.row_ptr, full.col_idx, full.val, rd, ri, H, rows=rows), "Y")
        _rows_close(d_all[rows], oracle.sspmm_bwd(full.row_ptr, full.col_idx, full.val, dy, ri, rows=rows), "dXs")
    for rk in ranks:
        rk.ops.close()
