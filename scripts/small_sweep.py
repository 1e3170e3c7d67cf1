"""Small-batch GPT-3 MLP shard (HBM-bound on weights): swapped tiles x split-K x policy."""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288


def main():
    batches = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1]
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for b in batches:
        x = torch.randn(b, H, device="cuda").half()
        us = time_fn(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t())
        print(f"B={b} cublas {us:.1f} us ({302e6 / us / 1e6:.2f} TB/s weights)", flush=True)
        tn = next(t for t in (32, 64, 128, 256) if t >= b)
        res = []
        for (z1, z2), (mode, pol) in itertools.product(
                ((3, 1), (3, 3), (6, 3)),
                (("fused", ts.RowSync()), ("fused", ts.TileSync()), ("stream", ts.RowSync()))):
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn, swap_ab=True,
                             prod_splits=z1, cons_splits=z2)
            us = time_fn(ch)
            res.append((us, f"B={b} swap{tn} z{z1}/{z2} {mode} {type(pol).__name__}: {us:.1f} us "
                            f"({302e6 / us / 1e6:.2f} TB/s) wd={ch.cs.watchdog_fired()}"))
        for (cg, tn), (z1, z2), (mode, pol) in itertools.product(
                ((1, 256), (1, 128), (2, 256)), ((6, 3), (3, 3), (3, 1), (6, 6), (12, 6)),
                (("fused", ts.RowSync()), ("fused", ts.TileSync()), ("stream", ts.RowSync()))):
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn, cta_group=cg,
                             prod_splits=z1, cons_splits=z2)
            us = time_fn(ch)
            res.append((us, f"B={b} normal cg{cg} {tn} z{z1}/{z2} {mode} {type(pol).__name__}: "
                            f"{us:.1f} us ({302e6 / us / 1e6:.2f} TB/s) wd={ch.cs.watchdog_fired()}"))
        for us, line in sorted(res)[:10]:
            print(line, flush=True)
        for us, line in sorted(r for r in res if "normal" in r[1])[:5]:
            print(line, flush=True)


if __name__ == "__main__":
    main()
