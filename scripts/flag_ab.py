"""A/B timing of one diagnostic flag bit on the current build (same process, interleaved
rounds): `python scripts/flag_ab.py 23` times each chain with extra_flags 0 and 1 << 23.
Configurations: MLP B=1/256/1024, ResNet conv pairs at batch 32, attention S=512."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288


def chains():
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for b, kw in ((1, dict(swap_ab=True, tile_n=32, prod_splits=3, cons_splits=3)),
                  (256, dict(swap_ab=True, tile_n=256, prod_splits=3)),
                  (1024, dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                              cons_order=ts.BandedColumnMajor(4)))):
        x = torch.randn(b, H, device="cuda").half()
        for pol in (ts.RowSync(), ts.TileSync()):
            yield f"mlp B={b} {type(pol).__name__}", ts.MlpChain(x, w1, w2, policy=pol, **kw)
    for n, hw, c, tn, cg, z in ((32, 56, 64, 64, 1, 1), (32, 28, 128, 128, 1, 1),
                                (32, 14, 256, 256, 2, 1), (32, 7, 512, 256, 2, 1),
                                (1, 7, 512, 64, 1, 4), (8, 7, 512, 128, 1, 4),
                                (1, 14, 256, 64, 1, 4)):
        x = torch.randn(n, hw, hw, c, device="cuda").half()
        wc = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        yield f"conv {n}x{hw}x{c} z{z}", ts.ConvChain(x, wc, wc.clone(), tile_n=tn, cta_group=cg,
                                                      prod_splits=z, cons_splits=z)
    x = torch.randn(512, H, device="cuda").half()
    wq = (torch.randn(3 * 12 * 128, H, device="cuda") / H ** 0.5).half()
    wo = (torch.randn(H, 12 * 128, device="cuda") / (12 * 128) ** 0.5).half()
    yield "attn S=512", ts.AttentionChain(x, wq, wo, qkv_splits=2)


if __name__ == "__main__":
    bit = int(sys.argv[1]) if len(sys.argv) > 1 else 23
    res = {}
    for name, ch in chains():
        for rnd in range(2):
            for tag, fl in (("off", 0), ("on", 1 << bit)):
                ch.cs.extra_flags = fl
                ch.cs._desc = None
                res.setdefault(name, {}).setdefault(tag, []).append(time_fn(ch, iters=50))
        o, n = min(res[name]["off"]), min(res[name]["on"])
        print(f"{name:24s} flag off {o:7.1f} us  flag {bit} on {n:7.1f} us  ({o / n:.3f}x)",
              flush=True)
