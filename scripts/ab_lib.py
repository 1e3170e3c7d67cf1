"""Times a few fixed MLP plans with whichever library TS_LIB_PATH selects (A/B of builds)."""
import os
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner

H, F = 12288, 6144
torch.manual_seed(0)
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
lib = os.path.basename(os.environ.get("TS_LIB_PATH", "tree"))
for b, z, order in ((1024, 2, ts.BandedColumnMajor(4)), (1024, 1, ts.RowMajor()), (2048, 1, ts.RowMajor()), (256, 3, ts.RowMajor())):
    x = torch.randn(b, H, device="cuda").half()
    ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                     prod_splits=z, cons_order=order)
    r = [planner._time(ch, iters=20, warm=3) for _ in range(5)]
    print(f"{lib:14s} B={b} z{z} {type(order).__name__}: {statistics.median(r):.1f} us", flush=True)
