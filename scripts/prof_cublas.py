"""cuBLAS fp16 GeMM of one shape, a few launches (for ncu). Usage:
python scripts/prof_cublas.py M N K [iters]"""
import sys

import torch

m, n, k = (int(v) for v in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
x = torch.randn(m, k, device="cuda").half()
w = (torch.randn(n, k, device="cuda") / k ** 0.5).half()
c = torch.empty(m, n, device="cuda", dtype=torch.half)
for _ in range(iters):
    torch.matmul(x, w.t(), out=c)
torch.cuda.synchronize()
