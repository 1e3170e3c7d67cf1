"""Halo conv pipeline diagnostics: timing with diagnostic flags (bit 13: no MMAs, bit 12:
no semaphore waits) to see which role paces a tile."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
hw, c = 56, 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for b in (128, 256):
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    for name, fl, mode in (("stream batch8", 1 << 6, "stream"), ("fused batch8", 1 << 6, "fused"),
                           ("stream nothing batch8", (1 << 13) | (1 << 24) | (1 << 25) | (1 << 15) | (1 << 6), "stream"),
                           ("stream", 0, "stream"), ("stream no-mma", 1 << 13, "stream"),
                           ("stream no-tmem-ld", 1 << 24, "stream"),
                           ("stream no-mma no-tmem-ld", (1 << 13) | (1 << 24), "stream"),
                           ("stream no-stores", 1 << 25, "stream"),
                           ("stream nothing", (1 << 13) | (1 << 24) | (1 << 25), "stream"),
                           ("stream nothing no-window", (1 << 13) | (1 << 24) | (1 << 25) | (1 << 15), "stream"),
                           ("stream no-window", 1 << 15, "stream")):
        ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True, extra_flags=fl)
        print(f"B={b} {name}: {planner._time(ch, iters=20):.1f} us", flush=True)
