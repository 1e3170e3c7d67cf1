"""L2 prefetch of a waiting consumer tile's weights (TS_FLAG_L2_PREFETCH) on vs off, GPT-3
MLP shard, the planner's usual plans per batch; medians of interleaved rounds."""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import _lib, planner

H, F = 12288, 6144
torch.manual_seed(0)
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
B = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512, mode="fused", policy=ts.RowSync())
PLANS = {
    64: [dict(B, prod_splits=6, cons_splits=3), dict(B, prod_splits=4, cons_splits=2)],
    256: [dict(B, prod_splits=2, cluster_pairs=2), dict(B, prod_splits=4, cons_splits=2),
          dict(B, prod_splits=4, cons_splits=3), dict(B, prod_splits=3)],
    512: [dict(B, prod_splits=3), dict(B, prod_splits=3, cons_order=ts.BandedColumnMajor(2)),
          dict(B, prod_splits=2)],
    1024: [dict(B, prod_splits=2, cons_order=ts.BandedColumnMajor(4)), dict(B, prod_splits=2),
           dict(B)],
    2048: [dict(B), dict(B, prod_splits=2, cons_order=ts.BandedColumnMajor(4))],
}
for b in (int(a) for a in (sys.argv[1:] or ["64", "256", "512", "1024", "2048"])):
    x = torch.randn(b, H, device="cuda").half()
    chains = {}
    for i, kw in enumerate(PLANS[b]):
        for pf in (0, _lib.TS_FLAG_L2_PREFETCH):
            chains[f"plan{i} {planner.describe(kw)['splits']} qd{kw.get('cluster_pairs', 1)}"
                   f"{' band' if 'cons_order' in kw else ''}{' +L2pf' if pf else ''}"] = \
                ts.MlpChain(x, w1, w2, extra_flags=pf, **kw)
    runs = {k: [] for k in chains}
    for _ in range(3):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    cu = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(), iters=20)
    print(f"B={b}: cublas {cu:.1f} us", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k])):
        assert not chains[k].cs.watchdog_fired(), k
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
