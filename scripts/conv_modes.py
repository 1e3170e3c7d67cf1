"""Conv pair: every planner candidate timed in fused and stream mode side by side (same
tile / split configuration), to see where a fused launch loses to its own stream form.
usage: python scripts/conv_modes.py 7:512:1,8 28:128:128"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402
from paper_2305_13450_b200.chains import ConvChain  # noqa: E402

if __name__ == "__main__":
    torch.manual_seed(11)
    for arg in sys.argv[1:]:
        hw, c, bs = arg.split(":")
        hw, c = int(hw), int(c)
        w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        for b in (int(v) for v in bs.split(",")):
            x = torch.randn(b, hw, hw, c, device="cuda").half()
            print(f"layer {hw}x{hw}x{c} B={b}", flush=True)
            for kw in planner.conv_candidates(c, "fused", b * hw * hw):
                row = []
                for mode in ("fused", "stream"):
                    ch = ConvChain(x, w1, w2, **{**kw, "mode": mode})
                    row.append(planner._time(ch, iters=20))
                    planner._check_watchdog(ch, kw)
                k = {a: v for a, v in kw.items() if a != "mode"}
                print(f"   fused {row[0]:7.1f}  stream {row[1]:7.1f}  {k}", flush=True)
