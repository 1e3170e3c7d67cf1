"""Run one chain configuration a few times (for ncu). Usage:
python scripts/prof_one.py B MODE POLICY TILE_N [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

b, mode, pol, tn = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
H = 12288
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
policy = {"row": ts.RowSync(), "tile": ts.TileSync()}[pol]
ch = ts.MlpChain(x, w1, w2, policy=policy, mode=mode, tile_n=tn)
for _ in range(iters):
    ch()
torch.cuda.synchronize()
print("done", ch.cs.watchdog_fired())
