"""Small-batch chain: swapped tiles + split-K. Correctness vs torch and timing.
Usage: python scripts/small_batch.py [B,...] [z1,...] [z2,...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H = 12288


def time_fn(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    arg = lambda i, d: [int(v) for v in sys.argv[i].split(",")] if len(sys.argv) > i else d
    batches, z1s, z2s = arg(1, [1, 64, 128, 256]), arg(2, [1, 2, 3, 4]), arg(3, [1, 2, 3])
    for b in batches:
        x = torch.randn(b, H, device="cuda").half()
        h_ref = torch.nn.functional.gelu(x.float() @ w1.float().t()).half()
        y_ref = h_ref.float() @ w2.float().t()
        cu = time_fn(lambda: torch.nn.functional.gelu(x @ w1.t()) @ w2.t())
        print(f"B={b} cublas {cu:.1f} us", flush=True)
        tn = next(t for t in (32, 64, 128, 256) if t >= b)
        for z1 in z1s:
            for z2 in z2s:
                for mode, pol in (("stream", ts.RowSync()), ("fused", ts.RowSync()),
                                  ("fused", ts.TileSync())):
                    ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn, swap_ab=True,
                                     prod_splits=z1, cons_splits=z2)
                    y = ch()
                    torch.cuda.synchronize()
                    eh = (ch.h.float() - h_ref.float()).abs().max().item()
                    ey = (y.float() - y_ref).abs().max().item()
                    us = time_fn(ch)
                    print(f"  tn={tn} z1={z1} z2={z2} {mode:6s} {type(pol).__name__:8s} "
                          f"{us:7.1f} us err_h={eh:.4f} err_y={ey:.4f} "
                          f"wd={ch.cs.watchdog_fired()}", flush=True)


if __name__ == "__main__":
    main()
