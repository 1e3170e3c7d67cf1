"""A/B timing of the current build vs old_build/pkg_old on the same box (same process
order: old, new, old, new). Configurations: small-batch MLP, conv pairs, B=1024 MLP."""
import importlib
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "old_build")
from scripts.sweep import time_fn  # noqa: E402

H = 12288


def run(ts, tag):
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    out = []
    for b, kw in ((1, dict(swap_ab=True, tile_n=32, prod_splits=3, cons_splits=3)),
                  (256, dict(swap_ab=True, tile_n=256, prod_splits=3)),
                  (1024, dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                              cons_order=ts.BandedColumnMajor(4)))):
        x = torch.randn(b, H, device="cuda").half()
        for mode, pol in (("fused", ts.RowSync()), ("fused", ts.TileSync()), ("stream", ts.RowSync())):
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, **kw)
            out.append((f"mlp B={b} {mode} {type(pol).__name__}", time_fn(ch, iters=50)))
    for n, hw, c, tn in ((32, 56, 64, 64), (8, 28, 128, 128)):
        x = torch.randn(n, hw, hw, c, device="cuda").half()
        wc = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        for mode in ("fused", "stream"):
            ch = ts.ConvChain(x, wc, wc.clone(), mode=mode, tile_n=tn, cta_group=1)
            out.append((f"conv {n}x{hw}x{c} {mode}", time_fn(ch, iters=50)))
    return out


if __name__ == "__main__":
    new = importlib.import_module("paper_2305_13450_b200")
    old = importlib.import_module("pkg_old")
    res = {}
    for rnd in range(2):
        for tag, mod in (("old", old), ("new", new)):
            for name, us in run(mod, tag):
                res.setdefault(name, {}).setdefault(tag, []).append(us)
    for name, d in res.items():
        o, n = min(d["old"]), min(d["new"])
        print(f"{name:28s} old {o:7.1f} us  new {n:7.1f} us  ({o / n:.3f}x)")
