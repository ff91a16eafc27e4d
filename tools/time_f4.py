import sys, os, torch
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo') else '.')
from paper_2312_08656_b200 import maxk
n, f, h, k = 232965, 256, 256, 32
x = torch.randn((n, f), device="cuda").to(torch.bfloat16)
w = (torch.randn((h, f), device="cuda") / 16).to(torch.bfloat16)
b = torch.randn((h,), device="cuda")
for _ in range(3): maxk.maxk_linear_topk_cbsr(x, w, k, bias=b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): maxk.maxk_linear_topk_cbsr(x, w, k, bias=b)
e1.record(); torch.cuda.synchronize()
print("f4 ms", e0.elapsed_time(e1) / 50)
sd = torch.empty((n, k), device="cuda")
si = torch.empty((n, k), device="cuda", dtype=torch.uint8)


def unfused():
    z = torch.addmm(b, x, w.t(), out_dtype=torch.float32)
    maxk.maxk_topk_cbsr(z, k, sd, si)


for _ in range(3): unfused()
torch.cuda.synchronize()
e0.record()
for _ in range(50): unfused()
e1.record(); torch.cuda.synchronize()
print("unfused (cuBLAS addmm bf16->fp32 + maxk_topk_cbsr) ms", e0.elapsed_time(e1) / 50)
