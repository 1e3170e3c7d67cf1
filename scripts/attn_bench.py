"""GPT-3 attention block (TP=8 shard): fused vs stream vs torch/cuBLAS, S in 512..2048."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.small_batch import time_fn  # noqa: E402

H, HEADS = 12288, 12


def torch_attn(x, wqkv, w2):
    qkv = x @ wqkv.t()
    m = x.shape[0]
    q, k, v = qkv.view(m, 3, HEADS, 128).unbind(1)
    dot = (torch.softmax((q * v).float(), dim=-1) * k.float()).to(x.dtype).reshape(m, -1)
    return dot @ w2.t()


def main():
    torch.manual_seed(0)
    wqkv = (torch.randn(3 * HEADS * 128, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, HEADS * 128, device="cuda") / (HEADS * 128) ** 0.5).half()
    for s in (512, 1024, 2048):
        x = torch.randn(s, H, device="cuda").half()
        cu = time_fn(lambda: torch_attn(x, wqkv, w2))
        fl = 2 * s * H * 3 * HEADS * 128 + 2 * s * HEADS * 128 * H
        print(f"S={s} torch {cu:.1f} us", flush=True)
        for cg, tn in ((2, 256), (1, 256), (2, 128)):
            for mode, pol in (("stream", ts.TileSync()), ("fused", ts.TileSync()),
                              ("fused", ts.RowSync())):
                ch = ts.AttentionChain(x, wqkv, w2, second_policy=pol, mode=mode, cta_group=cg,
                                       tile_n=tn)
                us = time_fn(ch)
                print(f"  cg={cg} tn={tn} {mode:6s} {type(pol).__name__:8s} {us:7.1f} us "
                      f"{fl / us / 1e6:.0f} TF/s wd={ch.cs.watchdog_fired()}", flush=True)


if __name__ == "__main__":
    main()
