"""Headline chain (GPT-3 MLP B=1024, 256x512 pair tiles, banded consumer, 22-tile GeMM2 tail)
under kernel knobs carried in flags: commit-group size (bits 17-18), weight / activation L2
hints (bits 8-9 / 10-11). Interleaved rounds, min of 3."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

H = 12288
torch.manual_seed(0)
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
x = torch.randn(1024, H, device="cuda").half()
knobs = {"default": 0, "G=1": 1 << 17, "G=3": 3 << 17, "B evict_first": 1 << 8,
         "B evict_normal": 2 << 8, "B evict_last": 3 << 8, "A evict_first": 1 << 10,
         "A evict_normal": 2 << 10}
chains = {k: ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512,
                         cons_order=ts.BandedColumnMajor(4), cons_tail=(22, 2), extra_flags=f)
          for k, f in knobs.items()}
res = {k: [] for k in knobs}
for _ in range(3):
    for k, ch in chains.items():
        res[k].append(time_fn(ch, iters=30))
for k, v in res.items():
    print(f"{k:16s} {min(v):7.1f} us  wd={chains[k].cs.watchdog_fired()}", flush=True)
