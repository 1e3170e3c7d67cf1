import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
n, hw, c, tn, z = 1, 7, 512, 64, 4
x = torch.randn(n, hw, hw, c, device="cuda").half()
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
ch = ts.ConvChain(x, w1, w2, tile_n=tn, cta_group=1, prod_splits=z, cons_splits=z)
for _ in range(3): ch()
ch.cs.enable_trace()
ch(); torch.cuda.synchronize()
recs = ch.cs.trace_records()
t0 = min(r.t_ns for r in recs)
from collections import defaultdict
per = defaultdict(list)
for r in recs:
    per[(r.stage, r.tb)].append((r.t_ns - t0, r.kind, r.k, r.sem, r.value))
for key in sorted(per)[:6] + sorted(per)[32:40]:
    ev = sorted(per[key])
    waits = [e for e in ev if e[1] in (1, 2)]
    print(key, "sched %.1f" % (ev[0][0]/1e3), "nwait", len(waits)//2,
          "first_wait %.1f..%.1f" % (waits[0][0]/1e3, waits[1][0]/1e3) if waits else "",
          "last_wait_end %.1f" % (waits[-1][0]/1e3) if waits else "",
          " ".join("%s@%.1f" % ({5:"mma0",6:"mma1",7:"epi0",8:"epi1",9:"part",3:"post",4:"fin"}[k], t/1e3) for t,k,_,_,_ in ev if k in (3,4,5,6,7,8,9)))
