"""Halo conv 56x56x64: time with each tile's MMAs issued twice (diagnostic flag bit 25 of an
experiment build; results invalid) vs once: the marginal cost of a second sub-tile."""
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
        for fl in (0, 1 << 25):
            ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True, extra_flags=fl)
            print(f"B={b} {mode} {'double MMAs' if fl else 'normal'}: {planner._time(ch, iters=10):.1f} us", flush=True)
