"""Halo conv pair (56x56x64, B=256) vs the number of persistent CTAs: does the per-tile
cost scale with tiles per CTA (a per-CTA serial pipeline) or stay flat (a shared limit)?"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
hw, c = 56, 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for b in (64, 256):
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    for mode in ("stream", "fused"):
        for nc in (148, 111, 74, 37):
            ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True, num_ctas=nc)
            us = planner._time(ch, iters=10)
            tiles = 2 * b * ((hw + 2) * hw + 127) // 128
            print(f"B={b} {mode} ctas {nc}: {us:.1f} us, {us * nc / tiles:.2f} us per tile per CTA", flush=True)
