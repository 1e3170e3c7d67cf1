"""A/B of two library builds (TS_LIB_PATH) on chains whose consumers wait: GPT-3 MLP
(RowSync / TileSync), attention, conv pairs. Run once per library; medians of 5.
usage: TS_LIB_PATH=variants/x.so python scripts/ab_wait.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from paper_2305_13450_b200 import planner  # noqa: E402
from paper_2305_13450_b200.chains import AttentionChain, ConvChain  # noqa: E402

lib = os.path.basename(os.environ.get("TS_LIB_PATH", "tree"))
H, F = 12288, 6144
torch.manual_seed(0)
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()


def report(name, ch):
    r = [planner._time(ch, iters=20, warm=3) for _ in range(5)]
    assert not ch.cs.watchdog_fired(), name
    print(f"{lib:12s} {name:48s} {statistics.median(r):7.1f} us", flush=True)


for b, pol, z, order in ((1024, ts.RowSync(), 2, ts.BandedColumnMajor(4)),
                         (1024, ts.TileSync(), 2, ts.RowMajor()),
                         (2048, ts.RowSync(), 1, ts.RowMajor()),
                         (256, ts.RowSync(), 3, ts.RowMajor()),
                         (256, ts.TileSync(), 3, ts.RowMajor())):
    x = torch.randn(b, H, device="cuda").half()
    report(f"mlp B={b} {type(pol).__name__} z{z} {type(order).__name__}",
           ts.MlpChain(x, w1, w2, policy=pol, tile_n=256, cta_group=2, prod_tile_n=512,
                       cons_tile_n=512, prod_splits=z, cons_order=order))
wqkv = (torch.randn(3 * 1536, H, device="cuda") / H ** 0.5).half()
wo = (torch.randn(H, 1536, device="cuda") / 1536 ** 0.5).half()
for s in (512, 2048):
    x = torch.randn(s, H, device="cuda").half()
    report(f"attention S={s}", AttentionChain(x, wqkv, wo))
for hw, c, b, tn, z, halo in ((28, 128, 256, 128, 1, False), (28, 128, 32, 128, 1, False),
                              (14, 256, 256, 256, 1, False), (7, 512, 32, 128, 2, False),
                              (7, 512, 1, 256, 4, False), (56, 64, 256, 64, 1, True),
                              (56, 64, 32, 64, 1, True)):
    cw1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    cw2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    for mode in ("fused", "stream"):
        report(f"conv {hw}x{hw}x{c} B={b} tn{tn} z{z}{' halo' if halo else ''} {mode}",
               ConvChain(x, cw1, cw2, mode=mode, tile_n=tn, cta_group=1, prod_splits=z,
                         cons_splits=z, halo=halo))
