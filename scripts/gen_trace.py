"""Measured side of the generations comparison: run the GPT-3 MLP
chain plans bench.py ships with the device trace on, and dump per-stage claim / finish
times and SMs, plus the chain's reference-scenario description, to
gpurun_out/gen_trace_B<b>_<name>.json. scripts/generations.py (run where /root/reference
is importable) adds the reference engine's prediction for the same B200 grids.

    python scripts/gen_trace.py B NAME=KW_JSON ...
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from paper_2305_13450_b200 import planner  # noqa: E402

H, FFN = 12288, 6144
POL = {"row": ts.RowSync(), "tile": ts.TileSync()}


def order(s):
    if s.startswith("band"):
        return ts.BandedColumnMajor(int(s[4:]))
    return ts.RowMajor()


def main():
    b = int(sys.argv[1])
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
    for arg in sys.argv[2:]:
        name, spec = arg.split("=", 1)
        if spec == "pick":
            kw, _ = planner.pick_mlp(x, w1, w2, mode="fused")
        else:
            kw = json.loads(spec)
            kw.setdefault("mode", "fused")
            kw["policy"] = POL[kw.get("policy", "row")]
            kw["cons_order"] = order(kw.get("cons_order", "row"))
            if "cons_tail" in kw:
                kw["cons_tail"] = tuple(kw["cons_tail"])
        ch = ts.MlpChain(x, w1, w2, **kw)
        for _ in range(3):
            ch()
        ch.cs.enable_trace(1 << 17)
        ch()
        torch.cuda.synchronize()
        recs = ch.cs.trace_records()
        t0 = min(r.t_ns for r in recs)
        out = {"batch": b, "name": name, "plan": planner.describe(kw), "stages": [], "deps": []}
        sc = ch.cs.scenario()
        for s_i, st in enumerate(sc.stages):
            sched = sorted(((r.t_ns - t0) / 1e3, r.tb, r.smid) for r in recs
                           if r.kind == 0 and r.stage == s_i)
            fin = sorted(((r.t_ns - t0) / 1e3, r.tb, r.smid) for r in recs
                         if r.kind == 4 and r.stage == s_i)
            out["stages"].append({"id": st.id, "grid": [st.grid.x, st.grid.y, st.grid.z],
                                  "k_steps": st.k_steps, "order": repr(st.order),
                                  "scheduled": sched, "finished": fin})
        for d in sc.deps:
            out["deps"].append({"producer": d.producer, "consumer": d.consumer,
                                "policy": repr(d.policy)})
        out["units"] = ch.cs.num_ctas or torch.cuda.get_device_properties(0).multi_processor_count // (
            ch.cs.cta_group * ch.cs.cluster_pairs)
        with open(f"gpurun_out/gen_trace_B{b}_{name}.json", "w") as f:
            json.dump(out, f)
        print(name, planner.describe(kw), "makespan",
              max(f[0] for s in out["stages"] for f in s["finished"]))


if __name__ == "__main__":
    main()
