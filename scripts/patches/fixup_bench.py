"""Split-K fix-up shares (TS_FLAG_SPLIT_FIXUP) vs the default split reductions on the GPT-3
MLP shard: medians of interleaved rounds, CUDA events."""
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
PLANS = {
    256: [(2, 1), (3, 1), (4, 2), (6, 3), (6, 2), (8, 4), (4, 3), (6, 4)],
    512: [(2, 1), (3, 1), (3, 2), (4, 2), (6, 3)],
    1024: [(1, 1), (2, 1), (3, 1), (2, 2), (3, 2)],
    2048: [(1, 1), (2, 1), (2, 2)],
}
for b in (int(a) for a in (sys.argv[1:] or ["256", "512", "1024", "2048"])):
    x = torch.randn(b, H, device="cuda").half()
    chains = {}
    for pz, cz in PLANS[b]:
        for order in ("RowMajor", "band4"):
            o = ts.RowMajor() if order == "RowMajor" else ts.BandedColumnMajor(4 if b >= 1024 else 2)
            for fx in (False, True):
                if fx and pz == 1 and cz == 1:
                    continue
                kw = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                          prod_splits=pz, cons_splits=cz, cons_order=o, split_fixup=fx)
                chains[f"z{pz}/{cz} {order}{' fixup' if fx else ''}"] = ts.MlpChain(x, w1, w2, **kw)
    runs = {k: [] for k in chains}
    for _ in range(3):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    cu = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(), iters=20)
    print(f"B={b}: cublas {cu:.1f} us", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k]))[:12]:
        assert not chains[k].cs.watchdog_fired(), k
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
