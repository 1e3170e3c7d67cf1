"""Host-side cost of CuSync.launch() and the GPU time of the same chain via CUDA graph."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.small_batch import time_fn  # noqa: E402

H = 12288
torch.manual_seed(0)
x = torch.randn(1, H, device="cuda").half()
w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
for label, kw in (("normal N256 cg1", dict(tile_n=256, cta_group=1)),
                  ("swap N32 z3", dict(tile_n=32, swap_ab=True, prod_splits=3))):
    for mode in ("stream", "fused"):
        ch = ts.MlpChain(x, w1, w2, mode=mode, **kw)
        ch()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            ch()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        host_us = (t1 - t0) / 200 * 1e6
        ev_us = time_fn(ch)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ch(s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    ch(s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_us = e0.elapsed_time(e1) * 1e3 / 50
        print(f"{label} {mode}: host {host_us:.1f} us/launch, eager events {ev_us:.1f} us, "
              f"graph {graph_us:.1f} us/chain", flush=True)
