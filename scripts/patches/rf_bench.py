"""Ready-first k-step order (TS_FLAG_READY_FIRST) vs in-order TileSync vs RowSync on the
GPT-3 MLP shard: CUDA-event time of each configuration, interleaved round robin."""
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
for b in (int(a) for a in (sys.argv[1:] or ["256", "512", "1024", "2048"])):
    x = torch.randn(b, H, device="cuda").half()
    base = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)
    cfgs = {}
    for z in (1, 2, 3):
        for order in ("RowMajor", "BandedColumnMajor(4)"):
            o = ts.RowMajor() if order == "RowMajor" else ts.BandedColumnMajor(4)
            cfgs[f"row z{z} {order}"] = dict(base, policy=ts.RowSync(), prod_splits=z, cons_order=o)
            cfgs[f"tile z{z} {order}"] = dict(base, policy=ts.TileSync(), prod_splits=z, cons_order=o)
            cfgs[f"tile+rf z{z} {order}"] = dict(base, policy=ts.TileSync(), prod_splits=z,
                                                 cons_order=o, ready_first=True)
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
