"""Halo conv pair timing for given (hw, batch) cases: python conv_halo_quick.py 224:8 56:256"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
c = 64
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
for case in sys.argv[1:]:
    hw, b = (int(v) for v in case.split(":"))
    x = torch.randn(b, hw, hw, c, device="cuda").half()
    out = []
    for mode in ("fused", "stream"):
        ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=True)
        out.append(f"{mode} {planner._time(ch, iters=20):.1f}")
        assert not ch.cs.watchdog_fired()
    print(f"{hw}x{hw}x{c} B={b}: " + ", ".join(out) + " us", flush=True)
