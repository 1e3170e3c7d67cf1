import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
hw, c, b = 56, 64, 256
torch.manual_seed(0)
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
x = torch.randn(b, hw, hw, c, device="cuda").half()
NOTHING = (1 << 13) | (1 << 24) | (1 << 25) | (1 << 15)
for nc in (148, 74, 37):
    for name, fl in (("real", 0), ("nothing", NOTHING)):
        ch = ts.ConvChain(x, w1, w2, tile_n=64, cta_group=1, mode="stream", halo=True, extra_flags=fl, num_ctas=nc)
        print(f"ctas {nc} {name}: {planner._time(ch, iters=10):.1f} us", flush=True)
# also: one-stage (only conv1 launch) to check per-launch cost
