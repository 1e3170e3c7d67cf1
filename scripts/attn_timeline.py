"""Device-trace timeline of the GPT-3 attention chain. argv: S cg z policy [flags]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.timeline import summarize  # noqa: E402

s, cg, z = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pol = {"row": ts.RowSync(), "tile": ts.TileSync()}[sys.argv[4]]
flags = int(sys.argv[5], 0) if len(sys.argv) > 5 else 0
mode = sys.argv[6] if len(sys.argv) > 6 else "fused"
ow = int(sys.argv[7]) if len(sys.argv) > 7 else 0
hidden, heads = 12288, 12
torch.manual_seed(8)
wqkv = (torch.randn(3 * heads * 128, hidden, device="cuda") / hidden ** 0.5).half()
w2 = (torch.randn(hidden, heads * 128, device="cuda") / (heads * 128) ** 0.5).half()
x = torch.randn(s, hidden, device="cuda").half()
ch = ts.AttentionChain(x, wqkv, w2, second_policy=pol, cta_group=cg, qkv_splits=z,
                       extra_flags=flags, mode=mode, out_tile_n=ow)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for _ in range(3):
    ch()
e0.record()
for _ in range(10):
    ch()
e1.record()
torch.cuda.synchronize()
print(f"-- untraced {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
ch.cs.enable_trace()
for _ in range(2):
    ch()
torch.cuda.synchronize()
summarize(ch.cs, f"attention S={s} cg{cg} z{z} {sys.argv[4]} {mode}")
