"""One attention-chain configuration, N launches (debug). argv: seq cg z policy flags n"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

s, cg, z = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pol = {"row": ts.RowSync(), "tile": ts.TileSync()}[sys.argv[4]]
flags = int(sys.argv[5], 0)
n = int(sys.argv[6])
hidden, heads = 12288, 12
torch.manual_seed(8)
wqkv = (torch.randn(3 * heads * 128, hidden, device="cuda") / hidden ** 0.5).half()
w2 = (torch.randn(hidden, heads * 128, device="cuda") / (heads * 128) ** 0.5).half()
x = torch.randn(s, hidden, device="cuda").half()
ch = ts.AttentionChain(x, wqkv, w2, second_policy=pol, cta_group=cg, qkv_splits=z,
                       extra_flags=flags)
for i in range(n):
    ch()
    torch.cuda.synchronize()
print("ok", sys.argv[1:], ch.cs.watchdog_fired(), flush=True)
