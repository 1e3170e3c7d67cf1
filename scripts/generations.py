"""Predicted vs measured generations and the tail-wave occupancy of the shipped GPT-3 MLP
plans (VERDICT r01 "missing" #5).

Predicted: the reference engine (tilesync_sim.simulate, /root/reference/pkg/src; run here,
where the reference is importable) on the chain's own B200 tile grids, with one "SM" per
work unit of the persistent kernel (a CTA pair for 256-row tiles: GpuConfig(74)) and, as
SURVEY.md §8a asks, GpuConfig(148). Generations = distinct grant times (engine.py:585-611).
The reference knows RowMajor / StridedRowMajor only; a BandedColumnMajor consumer is
predicted in RowMajor order (noted).

Measured: gpurun_out/gen_trace_B<b>_<name>.json from scripts/gen_trace.py (device trace:
claim / finish time and SM of every tile). A unit's n-th claim belongs to measured
generation n; the table gives each generation's size and claim-time span. The occupancy
profile counts units holding a tile (claimed, not finished) per 5% of the makespan.

    python scripts/generations.py gpurun_out/gen_trace_B1024_*.json > profiles/r02_generations.txt
"""
import json
import sys
from collections import defaultdict

sys.path.insert(0, "/root/reference/pkg/src")
from tilesync_sim import (Dependency, Dim3, GpuConfig, RowMajor, RowSync, Scenario,  # noqa: E402
                          Stage, TileSync, simulate)


def predicted(rec, sms):
    stages = []
    for s in rec["stages"]:
        stages.append(Stage(id=s["id"], grid=Dim3(*s["grid"]), occupancy=1,
                            k_steps=s["k_steps"], order=RowMajor()))
    deps = tuple(Dependency(d["producer"], d["consumer"], "a",
                            RowSync() if d["policy"].startswith("RowSync") else TileSync())
                 for d in rec["deps"])
    _, m = simulate(Scenario(gpu=GpuConfig(sms), stages=tuple(stages), deps=deps))
    return m


def measured(rec):
    claims = []  # (time, stage, smid)
    spans = []   # (start, end, smid)
    for s in rec["stages"]:
        fin = {tb: (t, sm) for t, tb, sm in s["finished"]}
        for t, tb, sm in s["scheduled"]:
            claims.append((t, s["id"], sm))
            if tb in fin:
                spans.append((t, fin[tb][0], sm))
    claims.sort()
    nth = defaultdict(int)
    gens = defaultdict(list)
    for t, sid, sm in claims:
        gens[nth[sm]].append((t, sid))
        nth[sm] += 1
    make = max(e for _, e, _ in spans)
    occ = []
    for i in range(20):
        lo, hi = make * i / 20, make * (i + 1) / 20
        mid = (lo + hi) / 2
        occ.append(len({sm for s0, e, sm in spans if s0 <= mid < e}))
    return gens, make, occ


def main():
    for path in sys.argv[1:]:
        rec = json.load(open(path))
        print(f"==== B={rec['batch']} {rec['name']}: {rec['plan']}")
        print(f"  work units (persistent CTA pairs / CTAs): {rec['units']}")
        for s in rec["stages"]:
            print(f"  stage {s['id']}: grid {s['grid']} k_steps {s['k_steps']} order {s['order']}")
        for sms in (rec["units"], 148):
            m = predicted(rec, sms)
            waves = ", ".join(f"{p.stage} {float(p.waves_frac):.2f} ({p.waves_ceil})"
                              for p in m.per_stage)
            print(f"  reference simulate, GpuConfig({sms}): generations {m.generations} "
                  f"sizes {list(m.generation_sizes)}; waves {waves}; makespan "
                  f"{float(m.makespan):.0f} cost units")
        gens, make, occ = measured(rec)
        print(f"  measured: makespan {make:.1f} us, {len(gens)} generations (n-th claim per unit)")
        for n in sorted(gens):
            g = gens[n]
            by = defaultdict(int)
            for _, sid in g:
                by[sid] += 1
            ts_ = [t for t, _ in g]
            print(f"    gen {n}: {len(g)} claims {dict(by)}, claim times "
                  f"{min(ts_):.1f}..{max(ts_):.1f} us")
        print("  units holding a tile per 5% of the makespan: " + " ".join(map(str, occ)))
        tail = occ[-6:]
        print(f"  tail (last 30%): mean {sum(tail) / len(tail):.1f} of {rec['units']} units busy")


if __name__ == "__main__":
    main()
