"""Mid-batch GPT-3 MLP plans with 256x384 pair tiles (more tiles than 256x512) and split-K."""
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
for b in (256, 512):
    x = torch.randn(b, H, device="cuda").half()
    cfgs = {"qd z2/1 (pick)": dict(prod_tile_n=512, cons_tile_n=512, prod_splits=2, cluster_pairs=2),
            "512/512 z3/1": dict(prod_tile_n=512, cons_tile_n=512, prod_splits=3),
            "512/512 z4/2": dict(prod_tile_n=512, cons_tile_n=512, prod_splits=4, cons_splits=2)}
    for pw, cw in ((384, 384), (384, 512), (512, 384)):
        for z1, z2 in ((2, 1), (3, 1), (4, 1), (2, 2), (3, 2), (4, 2)):
            cfgs[f"{pw}/{cw} z{z1}/{z2}"] = dict(prod_tile_n=pw, cons_tile_n=cw, prod_splits=z1,
                                                   cons_splits=z2)
    chains = {}
    for k, kw in cfgs.items():
        try:
            ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, **kw)
            ch()
            chains[k] = ch
        except Exception as e:  # noqa: BLE001
            pass
    runs = {k: [] for k in chains}
    for _ in range(3):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    print(f"B={b}:", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k]))[:10]:
        assert not chains[k].cs.watchdog_fired(), k
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
