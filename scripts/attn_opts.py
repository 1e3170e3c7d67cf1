"""GPT-3 attention shard S=512/1024: the planner's grid plus claimed dot items (flag bit 16:
dot tiles stay claimed work items instead of running on the last-arriving producer CTA) and
out-projection split-K; CUDA-event medians of interleaved rounds."""
import itertools
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import planner
from paper_2305_13450_b200.chains import AttentionChain

H, heads = 12288, 12
torch.manual_seed(8)
wqkv = (torch.randn(3 * heads * 128, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, heads * 128, device="cuda") / (heads * 128) ** 0.5).half()
for s in (int(a) for a in (sys.argv[1:] or ["512", "1024"])):
    x = torch.randn(s, H, device="cuda").half()
    chains = {}
    for mode, cg, z, ow, oz, fl in itertools.product(("fused", "stream"), (1, 2), (1, 2, 4), (0, 512), (1, 2),
                                                      (0, 1 << 16)):
        if (ow and cg == 1) or (mode == "stream" and fl):
            continue
        pol = ts.TileSync()
        try:
            ch = AttentionChain(x, wqkv, w2, second_policy=pol, mode=mode, cta_group=cg,
                                qkv_splits=z, out_tile_n=ow, out_splits=oz, extra_flags=fl)
            ch()
        except Exception as e:  # noqa: BLE001
            continue
        chains[f"{mode} cg{cg} z{z} ow{ow or 256} oz{oz}{' claimed-dot' if fl else ''}"] = ch
    runs = {k: [] for k in chains}
    for _ in range(2):
        for k, ch in chains.items():
            runs[k].append(planner._time(ch, iters=20, warm=3))
    print(f"S={s}:", flush=True)
    for k in sorted(runs, key=lambda k: statistics.median(runs[k]))[:14]:
        print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
