"""Small chains of every kind, once each (for compute-sanitizer)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

torch.manual_seed(0)
d = "cuda"
x = torch.randn(300, 512, device=d).half()
w1 = (torch.randn(1024, 512, device=d) / 23).half()
w2 = (torch.randn(512, 1024, device=d) / 32).half()
for kw in (dict(tile_n=256, cta_group=2), dict(tile_n=128, cta_group=1),
           dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512, prod_splits=2),
           dict(tile_n=64, swap_ab=True, prod_splits=2)):
    ts.MlpChain(x, w1, w2, policy=ts.TileSync(), **kw)()
xa = torch.randn(256, 512, device=d).half()
ts.AttentionChain(xa, (torch.randn(768, 512, device=d) / 23).half(),
                  (torch.randn(512, 256, device=d) / 16).half(), cta_group=2)()
xc = torch.randn(1, 14, 14, 128, device=d).half()
wc = (torch.randn(128, 3, 3, 128, device=d) / 34).half()
ts.ConvChain(xc, wc, wc.clone(), tile_n=128, cta_group=1)()
ts.MlpChain(x, w1, w2, policy=ts.RowSync(), tile_n=256, cta_group=2, prod_splits=2,
            row_interleave=True)()
from paper_2305_13450_b200 import tp  # noqa: E402
ar = tp.FusedTPMlp(x, w1, w2, tile_n=256, cta_group=2, cons_splits=2)  # world 1
tp.connect_group([ar])
ar()
torch.cuda.synchronize()
assert not ar.chain.cs.watchdog_fired()
print("ok")
