"""GPT-3 MLP shard at B: fused (one persistent launch) vs co-resident (the paper's
two-stream form, gate auto/on) vs stream-synchronized, same tiles. CUDA-event timing."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from paper_2305_13450_b200 import planner  # noqa: E402

H, FFN = 12288, 6144
for b in [int(a) for a in sys.argv[1:]] or [1024]:
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
    kw = dict(policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)
    res = {}
    for mode, gate in (("fused", None), ("stream", None), ("coresident", "auto"),
                       ("coresident", "on")):
        ch = ts.MlpChain(x, w1, w2, mode=mode, **kw)
        if gate:
            ch.cs.wait_kernel = gate
        res[f"{mode}{'/' + gate if gate else ''}"] = planner._time(ch, iters=20, warm=5)
        assert not ch.cs.watchdog_fired()
    print(f"B={b} 256x512 RowSync: " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()))
