"""B=1024 GPT-3 MLP plans under sustained load (the power cap settles over ~100 ms): each
plan runs N back-to-back chains per round, rounds interleaved, median per plan; plus the
clock the bench's sampler sees. Compares low-traffic (unsplit GeMM1) and split plans.
usage: python scripts/sustained_1024.py [N=200] [ROUNDS=4]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
H, F = 12288, 6144
torch.manual_seed(0)
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
x = torch.randn(1024, H, device="cuda").half()
base = dict(policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)
plans = {
    "fused z1 Band4": dict(base, cons_order=ts.BandedColumnMajor(4)),
    "fused z1 Band4 tail22x2": dict(base, cons_order=ts.BandedColumnMajor(4), cons_tail=(22, 2)),
    "fused z1 RowMajor": dict(base),
    "fused z2 Band4 (fixed)": dict(base, prod_splits=2, cons_order=ts.BandedColumnMajor(4)),
    "fused z2 Band2": dict(base, prod_splits=2, cons_order=ts.BandedColumnMajor(2)),
    "fused z3 Band2": dict(base, prod_splits=3, cons_order=ts.BandedColumnMajor(2)),
    "stream z1 RowMajor": dict(base, mode="stream"),
    "stream z2 Band4": dict(base, mode="stream", prod_splits=2,
                            cons_order=ts.BandedColumnMajor(4)),
    "stream z1 Band3 tail22x2": dict(base, mode="stream", cons_order=ts.BandedColumnMajor(3),
                                     cons_tail=(22, 2)),
    "stream z1 Band4 tail22x2": dict(base, mode="stream", cons_order=ts.BandedColumnMajor(4),
                                     cons_tail=(22, 2)),
}
chains = {k: ts.MlpChain(x, w1, w2, **kw) for k, kw in plans.items()}


def cublas():
    return torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t()


runs = {k: [] for k in list(chains) + ["cuBLAS"]}
for _ in range(rounds):
    for k in runs:
        fn = cublas if k == "cuBLAS" else chains[k]
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        runs[k].append(e0.elapsed_time(e1) * 1e3 / n)
for k, ch in chains.items():
    assert not ch.cs.watchdog_fired(), k
for k in sorted(runs, key=lambda k: statistics.median(runs[k])):
    print(f"   {statistics.median(runs[k]):7.1f} us  {k}  (rounds {[round(v, 1) for v in runs[k]]})",
          flush=True)
