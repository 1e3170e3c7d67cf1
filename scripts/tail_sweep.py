"""Last-wave balancing sweep for the GPT-3 MLP shard: GeMM2 tail tiles x slices on top of
the planner's large-batch configurations. argv: B"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
torch.manual_seed(0)
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
x = torch.randn(b, H, device="cuda").half()
tiles2 = (b // 256) * (H // 512)
rem = tiles2 % 74
res = []
for z1 in (1, 2):
    for band in (1, 4):
        for tail in ((0, 1), (rem, 2), (rem, 3), (rem, 4), (rem + 74, 2), (2 * rem, 2),
                     (2 * rem, 3)):
            if tail[0] > tiles2:
                continue
            for mode in ("fused", "stream"):
                ch = ts.MlpChain(x, w1, w2, policy=ts.RowSync(), mode=mode, tile_n=256,
                                 cta_group=2, prod_tile_n=512, cons_tile_n=512, prod_splits=z1,
                                 cons_order=ts.BandedColumnMajor(band) if band > 1 else ts.RowMajor(),
                                 cons_tail=tail)
                us = time_fn(ch, iters=30)
                res.append((us, f"B={b} z1={z1} band{band} tail={tail} {mode}: {us:.1f} us "
                                f"wd={ch.cs.watchdog_fired()}"))
for us, line in sorted(res)[:16]:
    print(line, flush=True)
