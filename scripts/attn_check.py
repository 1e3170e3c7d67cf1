"""Run each attention-chain configuration once; report watchdog / numerics (debug)."""
import itertools
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 512
hidden, heads = 12288, 12
torch.manual_seed(8)
wqkv = (torch.randn(3 * heads * 128, hidden, device="cuda") / hidden ** 0.5).half()
w2 = (torch.randn(hidden, heads * 128, device="cuda") / (heads * 128) ** 0.5).half()
x = torch.randn(s, hidden, device="cuda").half()
for mode, cg, z, pol in itertools.product(("fused", "stream"), (1, 2), (1, 2, 4),
                                          (ts.RowSync(), ts.TileSync())):
    t0 = time.time()
    ch = ts.AttentionChain(x, wqkv, w2, second_policy=pol, mode=mode, cta_group=cg, qkv_splits=z)
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
        ch()
    torch.cuda.synchronize()
    print(mode, cg, z, type(pol).__name__, "watchdog", ch.cs.watchdog_fired(),
          f"{time.time() - t0:.2f}s", flush=True)
