"""GeMM1 claimed column-band first (prod_order BandedColumnMajor(rows)) so each W1 column
block streams from HBM once, with TileSync consumers that start on the finished column
blocks, vs the RowMajor-producer plans; GPT-3 MLP shard B=1024."""
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
for b in (int(a) for a in (sys.argv[1:] or ["1024", "2048"])):
    x = torch.randn(b, H, device="cuda").half()
    rows = b // 256
    base = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)
    cfgs = {
        "row z2 band4 (fixed)": dict(base, policy=ts.RowSync(), prod_splits=2, cons_order=ts.BandedColumnMajor(4)),
        "row z1 rowmajor": dict(base, policy=ts.RowSync()),
    }
    for z in (1, 2, 3):
        for co in ("RowMajor", "band4"):
            o = ts.RowMajor() if co == "RowMajor" else ts.BandedColumnMajor(4)
            for pb in (rows, 2):
                cfgs[f"tile z{z} prodband{pb} cons {co}"] = dict(
                    base, policy=ts.TileSync(), prod_splits=z, cons_order=o,
                    prod_order=ts.BandedColumnMajor(pb))
    chains = {k: ts.MlpChain(x, w1, w2, **kw) for k, kw in cfgs.items()}
    runs = {k: [] for k in chains}
    for _ in range(3):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    cu = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(), iters=20)
    print(f"B={b}: cublas {cu:.1f} us", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k])):
        assert not chains[k].cs.watchdog_fired(), k
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
