"""Planner candidates for the GPT-3 MLP shard at batch B, fastest first (fused mode)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402

H, FFN = 12288, 6144
for b in [int(a) for a in sys.argv[1:]] or [1024]:
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
    best, cands = planner.pick_mlp(x, w1, w2, mode="fused")
    print(f"B={b}: pick {planner.describe(best)}")
    for d in sorted(cands, key=lambda c: c["us"])[:12]:
        print(f"   {d['us']:7.1f} us  " + str({k: v for k, v in d.items() if k != 'us'}))
