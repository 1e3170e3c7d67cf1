"""Run one GPT-3 MLP chain configuration with the device trace on and save the raw
records (ts_trace_rec) to gpurun_out/trace_<name>.json for offline analysis
(scripts/unit_timeline.py).

    python scripts/dump_trace.py B NAME KW_JSON
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H, FFN = 12288, 6144
POL = {"row": ts.RowSync(), "tile": ts.TileSync()}


def order(s):
    return ts.BandedColumnMajor(int(s[4:])) if s.startswith("band") else ts.RowMajor()


b, name, spec = int(sys.argv[1]), sys.argv[2], json.loads(sys.argv[3])
spec["policy"] = POL[spec.get("policy", "row")]
for k in ("cons_order", "prod_order"):
    if k in spec:
        spec[k] = order(spec[k])
if "cons_tail" in spec:
    spec["cons_tail"] = tuple(spec["cons_tail"])
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
ch = ts.MlpChain(x, w1, w2, **spec)
for _ in range(3):
    ch()
ch.cs.enable_trace(1 << 17)
ch()
torch.cuda.synchronize()
recs = ch.cs.trace_records()
out = [[r.t_ns, r.kind, r.stage, r.tb, r.k, r.dep, r.sem, r.value, r.x, r.y, r.z, r.smid, r.clk]
       for r in recs]
json.dump({"batch": b, "name": name, "stages": [s.id for s in ch.cs.stages], "recs": out},
          open(f"gpurun_out/trace_{name}.json", "w"))
print("dumped", len(out), "records")
