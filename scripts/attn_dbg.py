"""Debug: one attention launch, keep semaphores, compare with the oracle's totals."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

s, cg, z = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pol = {"row": ts.RowSync(), "tile": ts.TileSync()}[sys.argv[4]]
flags = int(sys.argv[5], 0) if len(sys.argv) > 5 else 0
hidden, heads = 12288, 12
torch.manual_seed(8)
wqkv = (torch.randn(3 * heads * 128, hidden, device="cuda") / hidden ** 0.5).half()
w2 = (torch.randn(hidden, heads * 128, device="cuda") / (heads * 128) ** 0.5).half()
x = torch.randn(s, hidden, device="cuda").half()
ch = ts.AttentionChain(x, wqkv, w2, second_policy=pol, cta_group=cg, qkv_splits=z,
                       extra_flags=flags, keep_sems=len(sys.argv) > 6)
for i in range(3):
    t0 = time.time()
    ch()
    torch.cuda.synchronize()
    print(i, "time", time.time() - t0, "watchdog", ch.cs.watchdog_fired(),
          "scratch", ch.cs._scratch.cpu().tolist(), flush=True)
    for st in ch.cs.stages:
        if st.cnt is not None:
            print("   cnt nonzero", int((st.cnt != 0).sum()), flush=True)
for d in ch.cs.deps:
    v = d.sem.cpu().tolist()
    print(d.id, "min", min(v), "max", max(v), "n", len(v), v[:24])
print("scratch", ch.cs._scratch.cpu().tolist())
