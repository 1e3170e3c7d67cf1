"""Planner candidate table for the GPT-3 MLP shard: `python scripts/plan_mlp.py 64,256,512`
prints the fastest fused and stream candidates per batch next to cuBLAS."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402

H = 12288
torch.manual_seed(0)
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
for b in (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256").split(",")):
    x = torch.randn(b, H, device="cuda").half()
    cu = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(),
                       iters=20)
    print(f"B={b} cublas {cu:.1f} us", flush=True)
    for mode in ("fused", "stream"):
        _, table = planner.pick_mlp(x, w1, w2, mode)
        for r in sorted(table, key=lambda r: r["us"])[:6]:
            print(f"  {mode:6s} {r['us']:7.1f} us {r['policy']:8s} {r['tile']:22s} cg{r['cta_group']} "
                  f"z{r['splits'][0]}/{r['splits'][1]} {r['consumer_order']} "
                  f"tail={r.get('consumer_tail', '-')}", flush=True)
