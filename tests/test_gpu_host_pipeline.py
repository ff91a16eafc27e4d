"""HostPipeline (the end-to-end public call for a stream of host batches): with copies
overlapped across steps and double-buffered device sets, every step's host outputs equal what the same pass
computes from device-resident inputs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200.dist import CudaOps, DistributedMaxk, HostPipeline
from paper_2312_08656_b200.partition import partition_rows_by_nnz

pytestmark = pytest.mark.gpu


def test_pipeline_matches_per_step_results():
    h, k, n = 256, 32, 3000
    g = synth.power_law_graph(n, 90_000, seed=21)
    dev = torch.device("cuda")
    part = partition_rows_by_nnz(g.row_ptr, 1)
    rp, ci, va = (torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val))
    ops = CudaOps(rp, ci, va, part.n_slots, h, k)
    agg = DistributedMaxk(part, 0, ops, h, k, dev)
    steps = 5  # distinct inputs per step: a buffer mix-up between double-buffered sets would show
    xs = [synth.normal_f32((n, h), 100 + i) for i in range(steps)]
    dys = [synth.normal_f32((n, h), 200 + i) for i in range(steps)]
    pipe = HostPipeline(agg)
    outs = []
    for i in range(steps):
        y_h = torch.empty((n, h), dtype=torch.float32).pin_memory()
        d_h = torch.empty((n, k), dtype=torch.float32).pin_memory()
        pipe.submit(torch.from_numpy(xs[i]).pin_memory(), torch.from_numpy(dys[i]).pin_memory(), y_h, d_h)
        outs.append((y_h, d_h))
    pipe.flush()
    torch.cuda.synchronize()
    for i in range(steps):
        rd, ri = oracle.topk_cbsr(xs[i], k)
        y_ref = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h)
        d_ref = oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dys[i], ri)
        for got, ref, what in ((outs[i][0].numpy(), y_ref, "Y"), (outs[i][1].numpy(), d_ref, "dXs")):
            err = np.abs(got.astype(np.float64) - ref).max(axis=1)
            assert np.all(err <= 1e-5 * (1 + np.abs(ref).max(axis=1))), (i, what)
    ops.close()
