"""Per-role stall profile of the halo-conv pipeline (diagnostic flag bit 7): producer
(ring-slot wait, claim, window-buffer wait, total), MMA warp (tile take, TMEM slot wait,
window wait, total), epilogue (tile take, accumulator wait, total, items), in cycles."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
hw, c, b = 56, 64, 256
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
x = torch.randn(b, hw, hw, c, device="cuda").half()
NOTHING = (1 << 13) | (1 << 24) | (1 << 25) | (1 << 15)
names = ["P ring-slot", "P claim", "P win-buf", "P total", "M take", "M tmem-slot", "M window",
         "M total", "E take", "E acc-wait", "E total", "E items", "M stage/weights", "M taps+commit", "-"]
for label, fl in (("real", 0), ("nothing", NOTHING)):
    ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode="stream", halo=True, extra_flags=fl | 128)
    ch.cs.enable_trace(148 * 16 * 8 // 48 + 64)
    ch()
    torch.cuda.synchronize()
    a = ch.cs._trace[: 148 * 16 * 8].view(torch.int64).reshape(148, 16).cpu().numpy()
    m = a[:, :15].mean(axis=0)
    print(label + ": " + ", ".join(f"{n} {v / 1e3:.1f}k" for n, v in zip(names, m)), flush=True)
