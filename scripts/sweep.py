"""Timing sweep over chain options on the GPT-3 MLP shard (CTA-pair tiles, per-stage
widths 256 / 512). Prints one line per config, fastest first per batch.

    python scripts/sweep.py [B1,B2,...]
"""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H = 12288


def time_fn(fn, iters=20, warm=3):
    for _ in range(warm):
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
    batches = [int(b) for b in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024]
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for b in batches:
        x = torch.randn(b, H, device="cuda").half()
        fl = 2 * b * H * (H // 2) * 2
        us = time_fn(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t())
        print(f"B={b} cublas {us:.1f} us {fl / us / 1e6:.0f} TF/s", flush=True)
        gx = -(-b // 256)
        res = []
        for pt, ct, (mode, pol), band in itertools.product(
                (256, 512), (256, 512),
                (("stream", ts.RowSync()), ("fused", ts.RowSync()), ("fused", ts.TileSync())),
                sorted({1, min(gx, 4), gx})):
            order = ts.BandedColumnMajor(band) if band > 1 else ts.RowMajor()
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=256, cta_group=2,
                             prod_tile_n=pt, cons_tile_n=ct, cons_order=order)
            us = time_fn(ch)
            res.append((us, f"B={b} {pt}/{ct} {mode:6s} {type(pol).__name__:8s} band{band}: "
                            f"{us:.1f} us {fl / us / 1e6:.0f} TF/s wd={ch.cs.watchdog_fired()}"))
        for us, line in sorted(res):
            print(line, flush=True)


if __name__ == "__main__":
    main()
