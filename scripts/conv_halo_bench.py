"""Halo-staged vs im2col-per-tap convolution pairs (Cin = Cout = 64) vs cuDNN."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
for hw, batches in ((56, (1, 8, 32, 128, 256)), (224, (1, 8, 32))):
    c = 64
    torch.manual_seed(0)
    w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
    wt1 = w1.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    wt2 = w2.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
    for b in batches:
        x = torch.randn(b, hw, hw, c, device="cuda").half()
        res = {}
        for mode in ("fused", "stream"):
            for halo in (False, True):
                ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode=mode, halo=halo)
                res[f"{mode}{'/halo' if halo else ''}"] = planner._time(ch, iters=20)
                assert not ch.cs.watchdog_fired()
        xt = x.permute(0, 3, 1, 2)
        cu = planner._time(lambda: torch.nn.functional.conv2d(
            torch.relu(torch.nn.functional.conv2d(xt, wt1, padding=1)), wt2, padding=1), iters=20)
        print(f"{hw}x{hw}x{c} B={b}: " + ", ".join(f"{k} {v:.1f}" for k, v in res.items())
              + f", cudnn {cu:.1f} us", flush=True)
