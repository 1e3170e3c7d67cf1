"""One fused im2col conv pair (28x28x128, B=256, tile_n=128, single CTA) for ncu: three
warm-up launches, then the profiled one (ncu -s 3 -c 1 -k regex:chain_kernel)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_13450_b200.chains import ConvChain  # noqa: E402

torch.manual_seed(11)
c = 128
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
x = torch.randn(256, 28, 28, c, device="cuda").half()
ch = ConvChain(x, w1, w2, tile_n=128, cta_group=1, mode=sys.argv[1] if len(sys.argv) > 1 else "fused")
for _ in range(4):
    ch()
torch.cuda.synchronize()
assert not ch.cs.watchdog_fired()
print("done")
