"""A/B of split-K reduction paths on the same box: tensor-core owner (default) vs the
all-planes last-arriver path (flag bit 29), GPT-3 MLP shard plans with split slices."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
H, FFN = 12288, 6144
cases = [(512, dict(prod_splits=3, cons_order=ts.BandedColumnMajor(2))),
         (512, dict(prod_splits=2)),
         (1024, dict(prod_splits=2, cons_order=ts.BandedColumnMajor(4))),
         (1024, dict(prod_splits=3)),
         (1024, dict(cons_tail=(22, 3), cons_order=ts.BandedColumnMajor(4))),
         (256, dict(prod_splits=4, cons_splits=2)),
         (256, dict(prod_splits=6, cons_splits=3))]
for b, kw in cases:
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
    res = []
    for rep in range(2):
        for fl in (0, 1 << 29):
            ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                             extra_flags=fl, **kw)
            res.append(planner._time(ch, iters=20, warm=5))
    print(f"B={b} {kw}: tensor-core {res[0]:.1f} / {res[2]:.1f} us, all-planes {res[1]:.1f} / {res[3]:.1f} us")
