"""DRAM bytes per launch for every CTA-pair B=1024 planner candidate, keyed the way bench.py
looks them up (planner.describe), into profiles/roofline_traffic.json.

  run:   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --print-units base --csv \
             -k regex:chain_kernel --log-file gpurun_out/traffic.csv \
             python scripts/traffic_table.py run gpurun_out/traffic_cfgs.json
  merge: python scripts/traffic_table.py merge gpurun_out/traffic_cfgs.json gpurun_out/traffic.csv

Each configuration launches twice (warm-up, then the counted launch); ncu's default cache
control flushes caches before each launch, so the counts are cold-cache per launch."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, ".")
B = 1024


def configs():
    from paper_2305_13450_b200 import planner
    units, qd = planner.chain_units(), planner.chain_units(cluster_pairs=2)
    out = []
    for kw in planner.with_reduce_variants(planner.candidates(B, "fused", n2=12288, units=units,
                                                             qd_units=qd)):
        if kw.get("cta_group") == 2 and not kw.get("swap_ab"):
            out.append(kw)
    return out


def run(cfg_path):
    import torch
    import paper_2305_13450_b200 as ts
    from paper_2305_13450_b200 import planner
    H, F = 12288, 6144
    torch.manual_seed(0)
    w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
    x = torch.randn(B, H, device="cuda").half()
    done = []
    for kw in configs():
        ch = ts.MlpChain(x, w1, w2, **kw)
        ch()
        ch()
        torch.cuda.synchronize()
        done.append(planner.describe(kw))
    Path(cfg_path).write_text(json.dumps(done))


def merge(cfg_path, csv_path):
    cfgs = json.loads(Path(cfg_path).read_text())
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    head = rows[0]
    iid, iname, ival = head.index("ID"), head.index("Metric Name"), head.index("Metric Value")
    per = defaultdict(float)
    for r in rows[1:]:
        if r[iname].startswith("dram__bytes_"):
            per[int(r[iid])] += float(r[ival].replace(",", ""))
    ids = sorted(per)
    assert len(ids) == 2 * len(cfgs), (len(ids), len(cfgs))
    prof = Path("profiles/roofline_traffic.json")
    table = json.loads(prof.read_text())
    for i, c in enumerate(cfgs):
        key = f"gpt3_mlp_b{B}_cfg{i:03d}"
        for k, rec in list(table.items()):
            if rec["config"] == c and rec["batch"] == B:
                key = k
        table[key] = {"batch": B, "bytes": int(per[ids[2 * i + 1]]), "config": c,
                      "source": "profiles/r02s3_traffic_table.txt (scripts/traffic_table.py: "
                                "ncu dram__bytes_read.sum + dram__bytes_write.sum, second of "
                                "two launches of this configuration)"}
        print(f"{per[ids[2 * i + 1]] / 1e6:8.1f} MB  {json.dumps(c)}")
    prof.write_text(json.dumps(table, indent=1) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        merge(sys.argv[2], sys.argv[3])
