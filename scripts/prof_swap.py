"""Run the swapped small-batch chain a few times (for ncu).
python scripts/prof_swap.py B TN Z1 Z2 MODE"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

b, tn, z1, z2, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
H = 12288
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
ch = ts.MlpChain(x, w1, w2, policy=ts.RowSync(), mode=mode, tile_n=tn, swap_ab=True,
                 prod_splits=z1, cons_splits=z2)
for _ in range(3):
    ch()
torch.cuda.synchronize()
print("done")
