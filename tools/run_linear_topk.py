"""Launch the fused Eq. 1 kernel on the Reddit-shaped row count (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08656_b200 import maxk  # noqa: E402

n, f, h, k = 232965, 256, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 32
x = torch.randn((n, f), device="cuda").to(torch.bfloat16)
w = (torch.randn((h, f), device="cuda") / 16).to(torch.bfloat16)
b = torch.randn((h,), device="cuda")
for _ in range(3):
    maxk.maxk_linear_topk_cbsr(x, w, k, bias=b)
torch.cuda.synchronize()
print("ok")
