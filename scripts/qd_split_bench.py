"""Two-pair-cluster (cluster_pairs=2) plans with split-K on both GeMMs, mid batch."""
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
for b in (int(a) for a in (sys.argv[1:] or ["256", "512"])):
    x = torch.randn(b, H, device="cuda").half()
    chains = {}
    for z1 in (1, 2, 3, 4):
        for z2 in (1, 2, 3):
            for qd in (1, 2):
                kw = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                          prod_splits=z1, cons_splits=z2, cluster_pairs=qd)
                try:
                    ch = ts.MlpChain(x, w1, w2, **kw)
                    ch()
                except Exception as e:  # noqa: BLE001
                    print("skip", kw, e)
                    continue
                chains[f"{'qd' if qd == 2 else 'pair'} z{z1}/{z2}"] = ch
    runs = {k: [] for k in chains}
    for _ in range(3):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    cu = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(), iters=20)
    print(f"B={b}: cublas {cu:.1f} us", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k])):
        assert not chains[k].cs.watchdog_fired(), k
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
