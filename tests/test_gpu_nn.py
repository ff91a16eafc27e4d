"""MaxK-GNN layer autograd (paper_2312_08656_b200.nn) vs a dense fp64 torch reference on a small graph.

The reference uses the MASK the kernel selected (the top-k decision is taken in the kernel's fp32 precision,
DESIGN §2) and recomputes everything else densely in fp64: Y = A · (Z ⊙ M), then autograd for dX, dW, db.
"""
import numpy as np
import pytest
import torch

import synth
from paper_2312_08656_b200 import maxk
from paper_2312_08656_b200.nn import Graph, MaxKGraphConv

pytestmark = pytest.mark.gpu


def _graph(n, seed):
    g = synth.random_csr(n, n, avg_deg=7.0, seed=seed, weights="mean")
    A = torch.zeros((n, n), dtype=torch.float64)
    for i in range(n):
        for e in range(g.row_ptr[i], g.row_ptr[i + 1]):
            A[i, g.col_idx[e]] += float(g.val[e])
    return g, A


def _close(a, b, what, tol=2e-3):
    a = a.double().cpu()
    b = b.double().cpu()
    err = (a - b).abs().max().item()
    scale = 1.0 + b.abs().max().item()
    assert err <= tol * scale, f"{what}: err {err:.3e} vs scale {scale:.3e}"


@pytest.mark.parametrize("fused", [False, True])
def test_layer_gradients_match_dense_reference(fused):
    n, f_in, h, k = 400, 64, 128, 16
    g, A = _graph(n, seed=7)
    dev = torch.device("cuda")
    graph = Graph(*(torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val)), n_cols=n, h=h, k=k)
    torch.manual_seed(0)
    layer = MaxKGraphConv(f_in, h, k, fused=fused, device=dev)
    with torch.no_grad():
        layer.b.copy_(torch.randn(h) * 0.1)
    x = torch.randn((n, f_in), device=dev, requires_grad=True)
    r = torch.randn((n, h), device=dev)
    y = layer(x, graph)
    (y * r).sum().backward()

    # the kernel's mask, from the same fp32 z the layer selected on
    with torch.no_grad():
        if fused:
            z = torch.empty((n, h), device=dev)
            maxk.maxk_linear_topk_cbsr(x.detach().to(torch.bfloat16), layer.w_t.detach(), k, bias=layer.b.detach(),
                                       z_out=z)
        else:
            z = torch.addmm(layer.b, x, layer.w_t.t())
        _, si = maxk.maxk_topk_cbsr(z, k)
    mask = torch.zeros((n, h), dtype=torch.float64)
    mask.scatter_(1, si.long().cpu(), 1.0)

    # dense fp64 reference with that mask
    xr = (x.detach().to(torch.bfloat16) if fused else x.detach()).double().cpu().requires_grad_(True)
    wr = layer.w_t.detach().double().cpu().requires_grad_(True)
    br = layer.b.detach().double().cpu().requires_grad_(True)
    zr = xr @ wr.t() + br
    yr = A @ (zr * mask)
    (yr * r.double().cpu()).sum().backward()
    _close(y.detach(), yr.detach(), "Y", tol=1e-4 if not fused else 1e-4)
    _close(layer.b.grad, br.grad, "db")
    _close(layer.w_t.grad, wr.grad, "dW", tol=1e-2 if fused else 1e-3)  # fused: bf16 GEMMs in the backward
    _close(x.grad, xr.grad, "dX", tol=1e-2 if fused else 1e-3)
