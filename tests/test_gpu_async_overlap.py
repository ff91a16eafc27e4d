"""The f2 comm/compute overlap under REAL asynchrony on one GPU.

G virtual ranks run in one process, one host thread and one CUDA stream each, every rank a full
DistributedMaxk with the local/remote edge split. Their collectives (VirtualGroup) are issued once every rank
has called them and run on a dedicated side stream, after events recorded on every rank's stream and after a
deliberate ~1 ms device delay; the handle's wait() orders the caller's stream after the side stream. So the
local forward really runs while the CBSR all-gather is in flight, and the local backward while the
reduce-scatter is in flight. Every buffer the collectives fill is poisoned with NaN first: a consumer that
does not wait() reads NaN and fails the oracle comparison. (Under gloo, tests/test_dist_gloo.py, the
collectives are synchronous host bounces.)"""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200.dist import CudaOps, DistributedMaxk
from paper_2312_08656_b200.partition import partition_rows_by_nnz, remap_columns, split_local_remote

pytestmark = pytest.mark.gpu

N, NNZ, H, K, SEED = 20000, 800000, 256, 32, 77
DELAY_CYCLES = 2_000_000  # ~1 ms at ~2 GHz before every collective's copies


class _Handle:
    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)


class VirtualGroup:
    """Collectives of G virtual ranks (threads) on one GPU, executed on a side stream."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.side = torch.cuda.Stream()
        self.pending = [None] * world
        self.done = None
        self.issued = {"ag": 0, "rs": 0}

    def member(self, rank: int):
        grp = self

        class _Member:
            def all_gather_async(self, out, inp):
                return grp._collective(rank, "ag", out, inp)

            def reduce_scatter_async(self, out, inp):
                return grp._collective(rank, "rs", out, inp)

        return _Member()

    def _collective(self, rank, kind, out, inp):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.pending[rank] = (out, inp, ev)
        self.barrier.wait()
        if rank == 0:
            with torch.cuda.stream(self.side):
                for _, _, e in self.pending:
                    self.side.wait_event(e)
                torch.cuda._sleep(DELAY_CYCLES)
                if kind == "ag":  # out_d[block s] = inp_s for every pair (in-place all_gather_into_tensor)
                    R = inp.shape[0]
                    for d in range(self.world):
                        for s in range(self.world):
                            if s != d:
                                self.pending[d][0][s * R:(s + 1) * R].copy_(self.pending[s][1])
                else:  # out_d = sum_s inp_s[block d] (reduce_scatter_tensor, sum)
                    R = self.pending[0][0].shape[0]
                    for d in range(self.world):
                        acc = self.pending[0][1][d * R:(d + 1) * R].clone()
                        for s in range(1, self.world):
                            acc += self.pending[s][1][d * R:(d + 1) * R]
                        self.pending[d][0].copy_(acc)
                self.done = torch.cuda.Event()
                self.done.record(self.side)
                self.issued[kind] += 1
        self.barrier.wait()
        return _Handle(self.done)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rows_close(gpu, ref, what):
    err = np.abs(gpu.astype(np.float64) - ref).max(axis=1)
    tol = 1e-5 * (1.0 + np.abs(ref).max(axis=1))
    assert np.all(err <= tol), f"{what}: worst {float(np.nanmax(err / tol)):.2f} x tol (NaN: a missing wait)"


@pytest.mark.parametrize("banked", ["0", "2"], ids=["column", "banked"])
@pytest.mark.parametrize("world", [2, 4])
def test_overlapped_split_path_under_async_collectives(world, banked, monkeypatch):
    # banked: the forward reads the bank-balanced copy (forced; the default where the forward uses NC = 16), and the
    # all-gather moves it plus the column-ordered mask (three collectives per pass instead of two)
    monkeypatch.setenv("MAXK_BANKED", banked)
    full = synth.power_law_graph(N, NNZ, SEED)
    x = synth.normal_f32((N, H), 1)
    dy = synth.normal_f32((N, H), 2)
    part = partition_rows_by_nnz(full.row_ptr, world)
    R, Nc = part.r_max, part.n_slots
    dev = torch.device("cuda", torch.cuda.current_device())
    grp = VirtualGroup(world)
    ranks = []
    for g in range(world):
        r0, r1 = part.rows(g)
        blk = synth.power_law_graph(N, NNZ, SEED, rows=(r0, r1))
        col = remap_columns(blk.col_idx, part)
        (lr, lc, lv), (rr, rc, rv) = split_local_remote(blk.row_ptr, col, blk.val, part, g)
        ops = CudaOps(_cuda(blk.row_ptr), _cuda(col), _cuda(blk.val), Nc, H, K)
        split = (CudaOps(_cuda(lr), _cuda(lc), _cuda(lv), R, H, K), CudaOps(_cuda(rr), _cuda(rc), _cuda(rv), Nc, H, K))
        agg = DistributedMaxk(part, g, ops, H, K, dev, split_ops=split, comm=grp.member(g))
        ranks.append(dict(agg=agg, ops=[ops, *split], x=_cuda(x[r0:r1]), dy=_cuda(dy[r0:r1]),
                          stream=torch.cuda.Stream(), out=None))
    torch.cuda.synchronize()
    errors = []

    def run(g):
        rk = ranks[g]
        try:
            with torch.cuda.stream(rk["stream"]):
                agg = rk["agg"]
                for _ in range(2):  # two passes: the second reuses every buffer of the first
                    agg.sp_data.fill_(float("nan"))
                    if agg.sp_banked is not None:
                        agg.sp_banked[0].fill_(float("nan"))
                    agg.d_local.fill_(float("nan"))
                    agg.y.fill_(float("nan"))
                    y = agg.forward(rk["x"])
                    d = agg.backward(rk["dy"])
                rk["out"] = (y.clone(), d.clone(), agg.sp_idx.clone())
                rk["stream"].synchronize()
        except Exception as e:  # surfaced on the main thread
            errors.append((g, repr(e)))
            grp.barrier.abort()

    threads = [threading.Thread(target=run, args=(g,)) for g in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    n_ag = 3 if banked == "2" else 2  # per pass: data + idx (+ the mask when banked) all-gathers, one reduce-scatter
    assert all(rk["agg"].sp_banked is not None for rk in ranks) == (banked == "2")
    assert grp.issued == {"ag": 2 * n_ag, "rs": 2}
    torch.cuda.synchronize()
    y_all = torch.cat([rk["out"][0] for rk in ranks]).cpu().numpy()
    d_all = torch.cat([rk["out"][1] for rk in ranks]).cpu().numpy()
    slots = part.slot_of(np.arange(N))
    rd, ri = oracle.topk_cbsr(x, K)
    for rk in ranks:  # every rank holds the full gathered mask, bit-exact
        assert np.array_equal(rk["out"][2].cpu().numpy()[slots].astype(np.int32), ri)
    _rows_close(y_all, oracle.spgemm_fwd(full.row_ptr, full.col_idx, full.val, rd, ri, H), "Y (all rows)")
    _rows_close(d_all, oracle.sspmm_bwd(full.row_ptr, full.col_idx, full.val, dy, ri), "dXs (all rows)")
    for rk in ranks:
        for o in rk["ops"]:
            o.close()
