"""Multi-GPU glue: one process per GPU, NCCL over NVLink through torch.distributed.

Rank g owns rows [r_g, r_{g+1}) of A, X, Y and dY (partition.py). One layer pass:
  1. top-k of the local X rows, written straight into the rank's slot block of the full CBSR buffers;
  2. in-place all_gather_into_tensor of sp_data (fp32) and sp_idx (uint8/16): every rank now holds the
     CBSR of all Nc slots — the compact (4+b)*k bytes/row exchange the paper's format enables;
  3. forward SpGEMM of the local row block against the gathered CBSR -> local Y rows;
  4. backward SSpMM of the local dY rows -> partial d_sp_data over ALL Nc slots (the outer product
     pushes to every column j, Eq. 4);
  5. reduce_scatter_tensor (sum) of the Nc x k partials -> each rank keeps its own R_max x k block.
The mask is the gathered sp_idx, identical in forward and backward by construction.

The compute steps are an `ops` object; production uses CudaOps (the C-ABI kernels). Tests may inject
other ops (e.g. the CPU oracle under gloo) to check the partition/exchange logic on CPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import maxk
from .partition import RowPartition


class CudaOps:
    """The product compute path: libmaxk.so kernels on the current CUDA stream."""

    def __init__(self, row_ptr, col_idx, val, n_cols: int, h: int, k: int, use_plan: bool = True):
        self.row_ptr, self.col_idx, self.val = row_ptr, col_idx, val
        self.n_cols, self.h, self.k = n_cols, h, k
        rp = row_ptr[[0, -1]].tolist()
        self.nnz = int(rp[1] - rp[0])
        self.plan = maxk.maxk_plan_create(row_ptr, h, k) if use_plan else None
        # the CBSR pair layout (k in {8, 16}) for the forward's gathers; used by 1-rank passes (maxk.pairs_default)
        self.use_pairs = maxk.pairs_default(h, k)
        # the bank-balanced CBSR copy (k in {32, 64, 128}) for the forward's gathers; used by 1-rank passes
        banked = maxk.banked_default(h, k, row_ptr.shape[0] - 1, self.nnz)
        self.use_banked = banked and k != 16                   # two-block copy, k in {32, 64, 128}
        self.pairs_banked = banked and self.use_pairs          # k = 16: the balanced pair order

    def topk(self, x, data_out, idx_out, pairs_out=None, banked_out=None):
        """Top-k into (data_out, idx_out); also the pair layout into pairs_out or the bank-balanced copy into
        banked_out = (bdata, bidx) when given (x rows must then be 16-byte aligned). Returns whether the
        companion layout was written."""
        with maxk.nvtx_range("maxk/topk"):
            if pairs_out is not None and maxk.float4_rows(x):
                maxk.maxk_topk_cbsr_pairs(x, self.k, data_out, idx_out, pairs_out, banked=self.pairs_banked)
                return True
            if banked_out is not None and maxk.float4_rows(x):
                maxk.maxk_topk_cbsr_banked(x, self.k, data_out, idx_out, *banked_out)
                return True
            maxk.maxk_topk_cbsr(x, self.k, data_out, idx_out)
            return False

    def forward(self, sp_data, sp_idx, y, accumulate=False, pairs=None):
        with maxk.nvtx_range("maxk/spgemm_fwd"):
            if pairs is not None and not accumulate:
                maxk.maxk_spgemm_fwd_pairs(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz, pairs,
                                           self.h, y=y, plan=self.plan)
            else:
                maxk.maxk_spgemm_fwd(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz, sp_data, sp_idx,
                                     self.h, y=y, plan=self.plan, accumulate=accumulate)

    def backward(self, dy, sp_idx, d_out, accumulate=False):
        with maxk.nvtx_range("maxk/sspmm_bwd"):
            maxk.maxk_sspmm_bwd(self.row_ptr, self.col_idx, self.val, self.n_cols, self.nnz, dy, sp_idx,
                                d_sp_data=d_out, plan=self.plan, accumulate=accumulate)

    def add(self, dst, src):
        maxk.maxk_add_f32(dst, src)

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None


def _host_bounce(group) -> bool:
    """gloo (the CPU test backend) has no CUDA all-gather / reduce-scatter: bounce through host memory."""
    return dist.get_backend(group) == "gloo"


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    if out.is_cuda and _host_bounce(group):
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def reduce_scatter_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    if out.is_cuda and _host_bounce(group):
        o = out.cpu()
        dist.reduce_scatter_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.reduce_scatter_tensor(out, inp, group=group)


class _Done:
    def wait(self):
        pass


def all_gather_async(out: torch.Tensor, inp: torch.Tensor, group=None):
    """In-place all-gather issued asynchronously (NCCL: on its own stream, after the caller's stream); the
    returned handle's wait() orders the caller's stream after it. The gloo test backend runs it synchronously."""
    if out.is_cuda and _host_bounce(group):
        all_gather_into(out, inp, group=group)
        return _Done()
    return dist.all_gather_into_tensor(out, inp, group=group, async_op=True)


def reduce_scatter_async(out: torch.Tensor, inp: torch.Tensor, group=None):
    if out.is_cuda and _host_bounce(group):
        reduce_scatter_into(out, inp, group=group)
        return _Done()
    return dist.reduce_scatter_tensor(out, inp, group=group, async_op=True)


def max_over_ranks(v: float, device, group=None) -> float:
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if _host_bounce(group) else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class DistributedMaxk:
    """One rank of the row-partitioned layer pass.

    split_ops = (ops_local, ops_remote) enables the comm/compute overlap of SURVEY §8(f) f2: ops_local holds the
    edges whose column is one of this rank's own slots (columns shifted to [0, R_max), partition.split_local_remote)
    and ops_remote the rest. Forward: the local edges run while the CBSR all-gather is in flight, then the remote
    edges accumulate into Y. Backward: the remote-target edges reduce into the Nc x k partial, whose
    reduce-scatter then runs while the local-target edges reduce into a private R_max x k block, added at the end.
    Same results as the unsplit pass (fp32 summation order aside)."""

    def __init__(self, part: RowPartition, rank: int, ops, h: int, k: int, device, idx_dtype=None, group=None,
                 split_ops=None, comm=None):
        self.part, self.rank, self.ops, self.h, self.k = part, rank, ops, h, k
        self.group = group
        # comm: an object with all_gather_async(out, inp) / reduce_scatter_async(out, inp) returning handles with
        # wait() (default: torch.distributed on `group`). Tests inject virtual ranks on one GPU whose collectives
        # run on a side CUDA stream, so the overlapped path runs under real asynchrony.
        self.comm = comm
        self.split_ops = split_ops if part.world > 1 else None
        r0, r1 = part.rows(rank)
        self.n_local = r1 - r0
        R, Nc = part.r_max, part.n_slots
        idt = idx_dtype if idx_dtype is not None else maxk.idx_dtype(h)
        self.sp_data = torch.empty((Nc, k), dtype=torch.float32, device=device)
        self.sp_idx = torch.empty((Nc, k), dtype=idt, device=device)
        self.y = torch.empty((self.n_local, h), dtype=torch.float32, device=device)
        self.d_partial = torch.empty((Nc, k), dtype=torch.float32, device=device)
        self.d_local = torch.empty((R, k), dtype=torch.float32, device=device)
        self._blk = slice(rank * R, (rank + 1) * R)
        # one rank: the forward gathers the pair layout where it exists (CudaOps.use_pairs); with several ranks the
        # two-block CBSR is what the all-gather moves (5k instead of 8k bytes per row)
        self.sp_pairs = (torch.empty((Nc, k, 2), dtype=torch.int32, device=device)
                         if part.world == 1 and getattr(ops, "use_pairs", False) else None)
        # k in {32, 64, 128} on high-degree graphs: the forward reads the bank-balanced copy (CudaOps.use_banked).
        # With several ranks the all-gather then moves the banked data and indices (for the forward) and the
        # column-ordered indices (the mask the backward and the caller use) instead of sp_data + sp_idx: 6k instead of
        # 5k bytes per row; the gathered sp_data then holds only this rank's block
        banked = getattr(ops, "use_banked", False)
        self.sp_banked = ((torch.empty((Nc, k), dtype=torch.float32, device=device),
                           torch.empty((Nc, k), dtype=idt, device=device)) if banked else None)
        self.d_tmp = torch.empty((R, k), dtype=torch.float32, device=device) if self.split_ops else None

    def _all_gather_async(self, out, inp):
        if self.comm is not None:
            return self.comm.all_gather_async(out, inp)
        return all_gather_async(out, inp, group=self.group)

    def _reduce_scatter_async(self, out, inp):
        if self.comm is not None:
            return self.comm.reduce_scatter_async(out, inp)
        return reduce_scatter_async(out, inp, group=self.group)

    def forward(self, x_local):
        R = self.part.r_max
        s0 = self.rank * R
        pairs, banked = self.sp_pairs, self.sp_banked
        kw = {}
        if pairs is not None:
            kw["pairs_out"] = pairs[s0:s0 + self.n_local]
        if banked is not None:
            kw["banked_out"] = tuple(b[s0:s0 + self.n_local] for b in banked)
        if not self.ops.topk(x_local, self.sp_data[s0:s0 + self.n_local], self.sp_idx[s0:s0 + self.n_local], **kw):
            pairs = banked = None  # x could not feed the companion layout: the forward reads the two blocks
        data, idx = banked if banked is not None else (self.sp_data, self.sp_idx)  # what the forward reads
        gathered = (data, idx) + ((self.sp_idx,) if banked is not None else ())  # + the backward's mask
        if self.split_ops is not None:
            ops_l, ops_r = self.split_ops
            waits = [self._all_gather_async(t, t[self._blk]) for t in gathered]
            ops_l.forward(data[self._blk], idx[self._blk], self.y)  # overlaps the all-gather
            for w in waits:
                w.wait()
            ops_r.forward(data, idx, self.y, accumulate=True)
            return self.y
        if self.part.world > 1:
            for t in gathered:
                all_gather_into(t, t[self._blk], group=self.group)
        self.ops.forward(data, idx, self.y, **({} if pairs is None else {"pairs": pairs}))
        return self.y

    def backward(self, dy_local):
        if self.split_ops is not None:
            ops_l, ops_r = self.split_ops
            ops_r.backward(dy_local, self.sp_idx, self.d_partial)  # this rank's own block stays zero
            w = self._reduce_scatter_async(self.d_local, self.d_partial)
            ops_l.backward(dy_local, self.sp_idx[self._blk], self.d_tmp)  # overlaps the reduce-scatter
            w.wait()
            ops_l.add(self.d_local, self.d_tmp)
            return self.d_local[: self.n_local]
        self.ops.backward(dy_local, self.sp_idx, self.d_partial)
        if self.part.world == 1:
            return self.d_partial[: self.n_local]
        reduce_scatter_into(self.d_local, self.d_partial, group=self.group)
        return self.d_local[: self.n_local]

    def step(self, x_local, dy_local):
        y = self.forward(x_local)
        d = self.backward(dy_local)
        return y, d

    def step_host(self, x_h, dy_h, y_h, d_h, x_d, dy_d):
        """One pass from pinned HOST inputs to pinned HOST outputs (the end-to-end public call).

        Copies overlap compute on side streams: dY's upload runs during top-k + forward, and Y's
        download runs during the backward. Everything is ordered on the caller's current stream at the
        end (no host synchronisation here)."""
        main = torch.cuda.current_stream()
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(device=x_d.device)
            self._d2h = torch.cuda.Stream(device=x_d.device)
        h2d, d2h = self._h2d, self._d2h
        x_d.copy_(x_h, non_blocking=True)
        h2d.wait_stream(main)
        with torch.cuda.stream(h2d):
            dy_d.copy_(dy_h, non_blocking=True)
        y = self.forward(x_d)
        d2h.wait_stream(main)
        with torch.cuda.stream(d2h):
            y_h.copy_(y, non_blocking=True)
        main.wait_stream(h2d)
        d = self.backward(dy_d)
        d_h.copy_(d, non_blocking=True)
        main.wait_stream(d2h)
        return y_h, d_h


class HostPipeline:
    """A sequence of layer passes from pinned HOST inputs to pinned HOST outputs with every copy overlapped:
    the end-to-end public call for a stream of batches (a training or serving loop).

    Step i's X and dY upload on an H2D stream while step i-1 computes; step i's Y downloads on a D2H stream as
    soon as its forward is done and its dXs after its backward, while step i+1 computes. PCIe is full duplex,
    so uploads and downloads also overlap each other. Device inputs and outputs are double-buffered (the
    buffers of step i are reused by step i+2 once step i's compute and downloads are done). Nothing
    synchronises the host; call flush() to order everything on the caller's current stream."""

    def __init__(self, agg: "DistributedMaxk"):
        self.agg = agg
        dev = agg.y.device
        n, h = agg.n_local, agg.h
        self.x = [torch.empty((n, h), dtype=torch.float32, device=dev) for _ in range(2)]
        self.dy = [torch.empty((n, h), dtype=torch.float32, device=dev) for _ in range(2)]
        self.y = [agg.y, torch.empty_like(agg.y)]
        self.dp = [agg.d_partial, torch.empty_like(agg.d_partial)]
        self.dl = [agg.d_local, torch.empty_like(agg.d_local)]
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.uploaded, self.fwd_done, self.computed, self.downloaded = ev(), ev(), ev(), ev()
        self.i = 0

    def begin(self):
        """Order the side streams after everything already queued on the caller's stream (e.g. a timing event)."""
        main = torch.cuda.current_stream()
        self.h2d.wait_stream(main)
        self.d2h.wait_stream(main)

    def submit(self, x_h, dy_h, y_h, d_h):
        s, agg, main = self.i % 2, self.agg, torch.cuda.current_stream()
        with torch.cuda.stream(self.h2d):
            if self.i >= 2:
                self.h2d.wait_event(self.computed[s])  # step i-2 has finished reading this input set
            self.x[s].copy_(x_h, non_blocking=True)
            self.dy[s].copy_(dy_h, non_blocking=True)
            self.uploaded[s].record(self.h2d)
        main.wait_event(self.uploaded[s])
        if self.i >= 2:
            main.wait_event(self.downloaded[s])  # step i-2's outputs have left this output set
        agg.y, agg.d_partial, agg.d_local = self.y[s], self.dp[s], self.dl[s]
        y = agg.forward(self.x[s])
        self.fwd_done[s].record(main)
        d = agg.backward(self.dy[s])
        self.computed[s].record(main)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.fwd_done[s])
            y_h.copy_(y, non_blocking=True)
            self.d2h.wait_event(self.computed[s])
            d_h.copy_(d, non_blocking=True)
            self.downloaded[s].record(self.d2h)
        self.i += 1

    def flush(self):
        main = torch.cuda.current_stream()
        main.wait_stream(self.h2d)
        main.wait_stream(self.d2h)



class SymmetricPeers:
    """The replicas and owner blocks of PeerMemoryMaxk in torch symmetric memory: every rank's [Nc x k] CBSR replica
    and [R_max x k] dXs block, mapped into every rank's address space (peer memory over NVLink), plus a device-side
    barrier. Needs one GPU per rank with peer access (an NVLink node)."""

    def __init__(self, group, n_slots: int, r_max: int, k: int, idx_dtype, device):
        import torch.distributed._symmetric_memory as symm
        world = dist.get_world_size(group)
        self.sd = symm.empty(n_slots, k, dtype=torch.float32, device=device)
        self.si = symm.empty(n_slots, k, dtype=idx_dtype, device=device)
        self.dl = symm.empty(r_max, k, dtype=torch.float32, device=device)
        hs = [symm.rendezvous(t, group) for t in (self.sd, self.si, self.dl)]
        self._barrier_handle = hs[2]
        self.replicas = [(hs[0].get_buffer(r, (n_slots, k), torch.float32), hs[1].get_buffer(r, (n_slots, k), idx_dtype))
                         for r in range(world)]
        self.owner_ptrs = torch.tensor(list(hs[2].buffer_ptrs), dtype=torch.int64, device=device)

    def barrier(self):
        self._barrier_handle.barrier(channel=0)


class PeerMemoryMaxk:
    """One rank of the row-partitioned layer pass with the exchanges fused into the kernels over peer memory
     instead of NCCL collectives: the top-k writes the rank's CBSR block into every
    rank's replica (maxk_topk_cbsr_multi) and the backward reduces each slot's dXs straight into its owner's block
    (maxk_sspmm_bwd_owners). peers: SymmetricPeers (an NVLink node), or any object with .replicas (per rank: the
    (sp_data, sp_idx) [Nc x k] replica), .owner_ptrs (int64 device tensor of the ranks' [R_max x k] dXs block
    addresses), .dl (this rank's block) and .barrier() (tests: virtual ranks on one GPU).
    Per pass: barrier (the replicas are free) -> top-k into every replica -> barrier -> forward from this rank's
    replica, zero this rank's dXs block -> barrier -> backward into the owners -> barrier (the blocks are complete).
    The phases are separate methods so that virtual ranks on one GPU can interleave them."""

    def __init__(self, part: RowPartition, rank: int, ops, h: int, k: int, peers):
        self.part, self.rank, self.ops, self.h, self.k, self.peers = part, rank, ops, h, k, peers
        r0, r1 = part.rows(rank)
        self.n_local = r1 - r0
        self.sp_data, self.sp_idx = peers.replicas[rank]
        self.d_local = peers.dl
        self.y = torch.empty((self.n_local, h), dtype=torch.float32, device=self.sp_data.device)

    def topk(self, x_local):
        s0, n = self.rank * self.part.r_max, self.n_local
        order = [self.rank] + [r for r in range(self.part.world) if r != self.rank]
        with maxk.nvtx_range("maxk/topk_multi"):
            maxk.maxk_topk_cbsr_multi(x_local, self.k, [self.peers.replicas[r][0][s0:s0 + n] for r in order],
                                      [self.peers.replicas[r][1][s0:s0 + n] for r in order])

    def forward(self):
        with maxk.nvtx_range("maxk/spgemm_fwd"):
            maxk.maxk_spgemm_fwd(self.ops.row_ptr, self.ops.col_idx, self.ops.val, self.ops.n_cols, self.ops.nnz,
                                 self.sp_data, self.sp_idx, self.h, y=self.y, plan=self.ops.plan)
        self.d_local.zero_()
        return self.y

    def backward(self, dy_local):
        with maxk.nvtx_range("maxk/sspmm_bwd_owners"):
            maxk.maxk_sspmm_bwd_owners(self.ops.row_ptr, self.ops.col_idx, self.ops.val, self.ops.n_cols,
                                       self.ops.nnz, dy_local, self.sp_idx, self.part.r_max, self.peers.owner_ptrs,
                                       plan=self.ops.plan)
        return self.d_local[: self.n_local]

    def step(self, x_local, dy_local):
        self.peers.barrier()
        self.topk(x_local)
        self.peers.barrier()
        y = self.forward()
        self.peers.barrier()
        d = self.backward(dy_local)
        self.peers.barrier()
        return y, d
