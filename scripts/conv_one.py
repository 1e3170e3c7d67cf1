"""One conv pair configuration timed (debug). argv: N HW C tile_n cg mode flags [z]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.sweep import time_fn  # noqa: E402

n, hw, c, tn, cg = (int(v) for v in sys.argv[1:6])
mode, flags = sys.argv[6], int(sys.argv[7], 0)
z = int(sys.argv[8]) if len(sys.argv) > 8 else 1
x = torch.randn(n, hw, hw, c, device="cuda").half()
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
ch = ts.ConvChain(x, w1, w2, mode=mode, tile_n=tn, cta_group=cg, extra_flags=flags,
                  prod_splits=z, cons_splits=z)
print(sys.argv[1:], f"{time_fn(ch):.1f} us", ch.cs.watchdog_fired())
