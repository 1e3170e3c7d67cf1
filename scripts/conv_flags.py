"""Untraced ResNet conv pair timings under diagnostic flag bits (which mechanism costs the
fused chain its time at small batch). argv: N HW C tile_n z"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

n, hw, c, tn, z = (int(v) for v in sys.argv[1:6])
x = torch.randn(n, hw, hw, c, device="cuda").half()
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for name, mode, fl in (("stream", "stream", 0), ("fused", "fused", 0),
                       ("fused no-wait (bit 12, wrong results)", "fused", 1 << 12),
                       ("fused no deep+R (bit 21)", "fused", 1 << 21),
                       ("fused no watermark (bit 23)", "fused", 1 << 23),
                       ("fused no reorder", "fused", 2)):
    ch = ts.ConvChain(x, w1, w2, mode=mode, tile_n=tn, cta_group=1, extra_flags=fl,
                      prod_splits=z, cons_splits=z)
    print(f"{n}x{hw}x{c} tn{tn} z{z} {name}: {time_fn(ch, iters=50):.1f} us", flush=True)
