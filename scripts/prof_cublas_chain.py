"""cuBLAS GPT-3 MLP shard chain (x @ W1^T -> GeLU -> @ W2^T), a few iterations (for ncu)."""
import sys

import torch

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
H = 12288
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
for _ in range(4):
    torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t()
torch.cuda.synchronize()
