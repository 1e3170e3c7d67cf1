"""Device trace of one conv pair (ConvChain) -> gpurun_out/trace_<name>.json for
scripts/unit_timeline.py.   python scripts/dump_conv_trace.py B HW C NAME KW_JSON"""
import json
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts
b, hw, c, name, kw = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], json.loads(sys.argv[5])
torch.manual_seed(0)
x = torch.randn(b, hw, hw, c, device="cuda").half()
w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
ch = ts.ConvChain(x, w1, w2, **kw)
for _ in range(3):
    ch()
ch.cs.enable_trace(1 << 20)
ch()
torch.cuda.synchronize()
recs = ch.cs.trace_records()
out = [[r.t_ns, r.kind, r.stage, r.tb, r.k, r.dep, r.sem, r.value, r.x, r.y, r.z, r.smid, r.clk]
       for r in recs]
json.dump({"batch": b, "name": name, "stages": [s.id for s in ch.cs.stages], "recs": out},
          open(f"gpurun_out/trace_{name}.json", "w"))
print("dumped", len(out))
