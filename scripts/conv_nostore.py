"""Halo conv pair with the epilogue's global stores skipped (diagnostic flag bit 25 of an
experiment build; results invalid) vs normal: the stores' share of the per-item time."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
c = 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for hw, b in ((56, 256), (224, 32)):
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    for mode in ("fused", "stream"):
        for fl in (0, 1 << 25):
            ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True, extra_flags=fl)
            print(f"{hw}x{hw} B={b} {mode} {'no stores' if fl else 'normal'}: {planner._time(ch, iters=10):.1f} us", flush=True)
