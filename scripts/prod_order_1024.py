"""B=1024 RowSync fixed plan (GeMM1 in 2 slices, BandedColumnMajor(4) consumer) with
different GeMM1 claim orders; medians of interleaved rounds."""
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
x = torch.randn(1024, H, device="cuda").half()
base = dict(policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
            prod_splits=2, cons_order=ts.BandedColumnMajor(4))
cfgs = {"prod RowMajor (fixed)": dict(base), "prod Band2": dict(base, prod_order=ts.BandedColumnMajor(2)),
        "prod Band4": dict(base, prod_order=ts.BandedColumnMajor(4)),
        "prod Strided(2)": dict(base, prod_order=ts.StridedRowMajor(2)),
        "prod Strided(3)": dict(base, prod_order=ts.StridedRowMajor(3))}
chains = {k: ts.MlpChain(x, w1, w2, **kw) for k, kw in cfgs.items()}
runs = {k: [] for k in chains}
for _ in range(4):
    for k, ch in chains.items():
        runs[k].append(planner._time(ch, iters=20, warm=3))
for k in sorted(runs, key=lambda k: statistics.median(runs[k])):
    assert not chains[k].cs.watchdog_fired(), k
    print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
