"""Run one GPT-3 MLP chain configuration a few times (for ncu). Usage:
python scripts/prof_one.py B MODE POLICY [PROD_TILE_N CONS_TILE_N BAND ITERS PROD_SPLITS PROD_BAND TAIL]"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

b, mode, pol = int(sys.argv[1]), sys.argv[2], sys.argv[3]
pt = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ct = int(sys.argv[5]) if len(sys.argv) > 5 else 0
band = int(sys.argv[6]) if len(sys.argv) > 6 else 1
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 3
z1 = int(sys.argv[8]) if len(sys.argv) > 8 else 1
pband = int(sys.argv[9]) if len(sys.argv) > 9 else 1
tail = tuple(int(v) for v in sys.argv[10].split(",")) if len(sys.argv) > 10 else (0, 1)
H = 12288
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
policy = {"row": ts.RowSync(), "tile": ts.TileSync()}[pol]
order = ts.BandedColumnMajor(band) if band > 1 else ts.RowMajor()
ch = ts.MlpChain(x, w1, w2, policy=policy, mode=mode, tile_n=256, cta_group=2,
                 prod_tile_n=pt, cons_tile_n=ct, cons_order=order, prod_splits=z1,
                 prod_order=ts.BandedColumnMajor(pband) if pband > 1 else ts.RowMajor(),
                 extra_flags=int(os.environ.get("TS_EXTRA_FLAGS", "0"), 0), cons_tail=tail)
for _ in range(iters):
    ch()
torch.cuda.synchronize()
print("done", ch.cs.watchdog_fired())
