"""GPT-3 MLP shard: split-K (reference z) x tile-width configurations, fused and stream."""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288


def main():
    batches = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024]
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for b in batches:
        x = torch.randn(b, H, device="cuda").half()
        fl = 2 * b * H * (H // 2) * 2
        us = time_fn(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t())
        print(f"B={b} cublas {us:.1f} us", flush=True)
        res = []
        for (pt, ct), (z1, z2), (mode, pol) in itertools.product(
                ((512, 512), (256, 512)),
                ((1, 1), (2, 1), (3, 1), (3, 2), (2, 2), (4, 2), (1, 2), (3, 3)),
                (("fused", ts.RowSync()), ("fused", ts.TileSync()), ("stream", ts.RowSync()))):
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=256, cta_group=2,
                             prod_tile_n=pt, cons_tile_n=ct, prod_splits=z1, cons_splits=z2,
                             cons_order=ts.BandedColumnMajor(min(4, b // 256)))
            us = time_fn(ch)
            res.append((us, f"B={b} {pt}/{ct} z{z1}/{z2} {mode} {type(pol).__name__}: {us:.1f} us "
                            f"{fl / us / 1e6:.0f} TF/s wd={ch.cs.watchdog_fired()}"))
        for us, line in sorted(res)[:14]:
            print(line, flush=True)


if __name__ == "__main__":
    main()
