"""Halo conv 56x56x64 pair time vs rows per tile (TS_HRPT env in an experiment build):
does the per-tile cost scale with tiles (per-item overhead) or with positions?"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
hw, c = 56, 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for b in (32, 256):
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    for mode in ("stream", "fused"):
        ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True)
        print(f"B={b} {mode}: {planner._time(ch, iters=10):.1f} us", flush=True)
