"""Eq. 1 fused on tcgen05 (maxk_linear_topk_cbsr) against the oracle.

The argmax-like selection is decided in the kernel's precision (fp32 z from bf16 products accumulated on the
tensor cores), so (DESIGN.md §2 comparison rule): z_out must match the fp64 oracle z = X·W + b within
1e-5·(1 + max|ref|) per row, and the CBSR must equal the oracle's exact top-k OF THE KERNEL'S z bit-exactly.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2312_08656_b200 import maxk

pytestmark = pytest.mark.gpu


def _case(n, f, h, k, seed, quantized=False, with_bias=True):
    g = torch.Generator().manual_seed(seed)
    if quantized:  # small integers -> exact z with many ties at the k-boundary (exercises the exact fallback)
        x = torch.randint(-2, 3, (n, f), generator=g).to(torch.bfloat16)
        w_t = torch.randint(-2, 3, (h, f), generator=g).to(torch.bfloat16)
        b = torch.randint(-2, 3, (h,), generator=g).float() if with_bias else None
    else:
        x = torch.randn((n, f), generator=g).to(torch.bfloat16)
        w_t = (torch.randn((h, f), generator=g) / 16).to(torch.bfloat16)
        b = torch.randn((h,), generator=g) if with_bias else None
    xd, wd = x.cuda(), w_t.cuda()
    bd = b.cuda() if b is not None else None
    z = torch.full((n, h), float("nan"), device="cuda")
    sd, si = maxk.maxk_linear_topk_cbsr(xd, wd, k, bias=bd, z_out=z)
    torch.cuda.synchronize()
    z_np = z.cpu().numpy()
    ref = oracle.linear(x.float().numpy(), w_t.float().numpy(), None if b is None else b.numpy())
    err = np.abs(z_np.astype(np.float64) - ref).max(axis=1)
    tol = 1e-5 * (1.0 + np.abs(ref).max(axis=1))
    assert np.all(err <= tol), f"z: worst {float((err / tol).max()):.2f} x tol"
    rd, ri = oracle.topk_cbsr(z_np, k)
    assert np.array_equal(si.cpu().numpy().astype(np.int32), ri)
    assert np.array_equal(sd.cpu().numpy().view(np.uint32), rd.view(np.uint32))
    return sd, si


@pytest.mark.parametrize("n,f,h,k", [
    (128, 256, 256, 32), (1000, 256, 256, 32), (5000, 256, 256, 8), (300, 128, 256, 16), (4097, 64, 256, 64),
    (1, 256, 256, 32), (129, 256, 128, 32), (2000, 256, 128, 1), (777, 192, 256, 64),
    # more tiles than CTAs: both TMEM accumulator stages and several mbarrier phases per CTA, ragged last tile
    (40001, 256, 256, 32), (25000, 128, 128, 16),
])
def test_linear_topk_matches_oracle(n, f, h, k):
    _case(n, f, h, k, seed=n + f + h + k)


@pytest.mark.parametrize("k", [1, 8, 32, 64])
def test_linear_topk_ties_exact_fallback(k):
    _case(1500, 128, 256, k, seed=k, quantized=True)


def test_linear_topk_no_bias_and_matches_unfused_path():
    n, f, h, k = 3000, 256, 256, 32
    sd, si = _case(n, f, h, k, seed=5, with_bias=False)
    # the fused selection equals maxk_topk_cbsr applied to the same z
    g = torch.Generator().manual_seed(5)
    x = torch.randn((n, f), generator=g).to(torch.bfloat16).cuda()
    w_t = (torch.randn((h, f), generator=g) / 16).to(torch.bfloat16).cuda()
    z = torch.empty((n, h), device="cuda")
    maxk.maxk_linear_topk_cbsr(x, w_t, k, z_out=z)
    d2, i2 = maxk.maxk_topk_cbsr(z, k)
    assert torch.equal(i2, si) and torch.equal(d2.view(torch.int32), sd.view(torch.int32))


def test_linear_topk_argument_errors():
    x = torch.zeros((10, 100), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((256, 100), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(maxk.MaxkError):
        maxk.maxk_linear_topk_cbsr(x, w, 8)  # f_in not a multiple of 64
    x = torch.zeros((10, 128), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros((192, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(maxk.MaxkError):
        maxk.maxk_linear_topk_cbsr(x, w, 8)  # h not in {128, 256}
