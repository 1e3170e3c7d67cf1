"""End-to-end (pinned host X -> chain -> pinned host Y) latency of MlpChain.run_host for a
few configurations, next to the unoverlapped copy-chain-copy sequence."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
xh = x.cpu().pin_memory()
yh = torch.empty(b, H, dtype=torch.half).pin_memory()
for name, kw in (("512/512 row", dict(prod_tile_n=512, cons_tile_n=512)),
                 ("512/512 row interleaved", dict(prod_tile_n=512, cons_tile_n=512, row_interleave=True)),
                 ("512/512 row z2/1 interleaved", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=2,
                                                       row_interleave=True)),
                 ("512/512 row z3/1 interleaved", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=3,
                                                       row_interleave=True)),
                 ("256/512 row z2/1 interleaved", dict(cons_tile_n=512, prod_splits=2, row_interleave=True)),
                 ("512/512 row z2/1", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=2)),
                 ("512/512 row z3/1", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=3)),
                 ("cg1 256/256 row z3/1", dict(cta_group=1, prod_splits=3)),
                 ("512/512 row z4/2", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=4, cons_splits=2)),
                 ("512/512 row z2/2", dict(prod_tile_n=512, cons_tile_n=512, prod_splits=2, cons_splits=2)),
                 ("256/256 row z4/2", dict(prod_splits=4, cons_splits=2)),
                 ("cg1 256/256 row z2/1", dict(cta_group=1, prod_splits=2)),
                 ("cg1 256/256 row", dict(cta_group=1))):
    kw = dict(dict(tile_n=256, cta_group=2), **kw)
    ch = ts.MlpChain(x.clone(), w1, w2, **kw)
    plain = time_fn(lambda: (ch.x.copy_(xh, non_blocking=True), ch(), yh.copy_(ch.y, non_blocking=True)))
    over = time_fn(lambda: ch.run_host(xh, yh))
    kern = time_fn(ch)
    print(f"B={b} {name}: kernel {kern:.1f} us, copy+chain+copy {plain:.1f} us, "
          f"overlapped run_host {over:.1f} us", flush=True)
h2d = time_fn(lambda: x.copy_(xh, non_blocking=True))
d2h = time_fn(lambda: yh.copy_(x, non_blocking=True))
print(f"H2D {h2d:.1f} us, D2H {d2h:.1f} us for {b * H * 2 / 1e6:.1f} MB each")
