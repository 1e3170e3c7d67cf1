"""Timing sweep over chain options on the GPT-3 MLP shard. Prints one line per config."""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H = 12288


def time_fn(fn, iters=10, warm=3):
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
    hints = [int(h) for h in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
    tns = [int(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [256]
    torch.manual_seed(0)
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for b in batches:
        x = torch.randn(b, H, device="cuda").half()
        fl = 2 * b * H * (H // 2) * 2

        def cub():
            return torch.nn.functional.gelu(x @ w1.t()) @ w2.t()
        us = time_fn(cub)
        print(f"B={b} cublas {us:.1f} us {fl / us / 1e6:.0f} TF/s", flush=True)
        for tn, hint in itertools.product(tns, hints):
            for mode, pol in (("stream", ts.RowSync()), ("fused", ts.RowSync()),
                              ("fused", ts.TileSync())):
                ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn,
                                 extra_flags=hint << 8)
                us = time_fn(ch)
                print(f"B={b} tn={tn} hint={hint} {mode:6s} {type(pol).__name__:8s} "
                      f"{us:.1f} us {fl / us / 1e6:.0f} TF/s wd={ch.cs.watchdog_fired()}",
                      flush=True)


if __name__ == "__main__":
    main()
