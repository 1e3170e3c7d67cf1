"""Per-unit (CTA pair / CTA, keyed by the leader's SM) timeline of a dumped device trace:
the sequence of items each unit ran, with MMA span, epilogue and idle gaps, so balanced
(stream-K) segments — several per tile — are attributed correctly.

    python scripts/unit_timeline.py gpurun_out/trace_NAME.json [--units N]
"""
import json
import sys
from collections import defaultdict

KIND = {0: "sched", 1: "wait_b", 2: "wait_e", 3: "post", 4: "fin", 5: "mma_b", 6: "mma_e",
        7: "epi_b", 8: "epi_e", 9: "part"}


def main(path, show=4):
    d = json.load(open(path))
    recs = sorted(d["recs"])
    t0 = recs[0][0]
    by_sm = defaultdict(list)
    for r in recs:
        by_sm[r[11]].append(r)
    items = {}  # per unit: list of dicts
    stats = defaultdict(float)
    makespan = (recs[-1][0] - t0) / 1e3
    for sm, rs in by_sm.items():
        # each role (scheduler, MMA warp, epilogue) handles a unit's items in claim order,
        # so the i-th record of a once-per-item kind belongs to the unit's i-th item
        seq = defaultdict(list)
        for r in rs:
            seq[KIND.get(r[1], str(r[1]))].append(r)
        lst = []
        for i, r in enumerate(seq["sched"]):
            it = {"stage": d["stages"][r[2]], "tb": r[3], "sched": (r[0] - t0) / 1e3}
            for k in ("mma_b", "mma_e", "epi_b", "epi_e", "fin"):
                if i < len(seq[k]):
                    it[k] = (seq[k][i][0] - t0) / 1e3
            lst.append(it)
        # waits and partial-plane records carry their item's (stage, tb)
        for k in ("wait_b", "wait_e", "part"):
            for r in seq[k]:
                for it in lst:
                    if it["stage"] == d["stages"][r[2]] and it["tb"] == r[3] and k not in it:
                        it[k] = (r[0] - t0) / 1e3
                        break
        items[sm] = lst
    units = sorted(items)
    mma_busy, first_mma, last_end = [], [], []
    for sm in units:
        lst = items[sm]
        busy = sum(it.get("mma_e", 0) - it.get("mma_b", 0) for it in lst if "mma_b" in it)
        mma_busy.append(busy)
        fm = [it["mma_b"] for it in lst if "mma_b" in it]
        first_mma.append(min(fm) if fm else 0)
        le = [it.get("fin", it.get("epi_e", 0)) for it in lst]
        last_end.append(max(le) if le else 0)
    n = len(units)
    print(f"{path}: {n} units, makespan {makespan:.1f} us")
    print(f"  MMA busy per unit: mean {sum(mma_busy) / n:.1f} us (min {min(mma_busy):.1f}, "
          f"max {max(mma_busy):.1f}) = {sum(mma_busy) / n / makespan:.0%} of the makespan")
    print(f"  first MMA per unit: mean {sum(first_mma) / n:.1f} us (max {max(first_mma):.1f})")
    print(f"  unit end: min {min(last_end):.1f} mean {sum(last_end) / n:.1f} max {max(last_end):.1f} us")
    # per item-type averages
    agg = defaultdict(list)
    for sm in units:
        for it in items[sm]:
            key = it["stage"]
            if "mma_b" in it and "mma_e" in it:
                agg[key + " mma"].append(it["mma_e"] - it["mma_b"])
                agg[key + " sched->mma"].append(it["mma_b"] - it["sched"])
            if "epi_b" in it and "epi_e" in it:
                agg[key + " epi"].append(it["epi_e"] - it["epi_b"])
            if "wait_b" in it and "wait_e" in it:
                agg[key + " wait"].append(it["wait_e"] - it["wait_b"])
            if "mma_e" in it and "epi_b" in it:
                agg[key + " mma_e->epi_b"].append(it["epi_b"] - it["mma_e"])
    for k in sorted(agg):
        v = agg[k]
        print(f"  {k:24s} n {len(v):4d} mean {sum(v) / len(v):7.1f} us  max {max(v):7.1f}")
    for sm in units[:show]:
        print(f"  unit sm{sm}:")
        for it in items[sm]:
            print("    " + " ".join(f"{k}={v:.1f}" if isinstance(v, float) else f"{k}={v}"
                                    for k, v in it.items()))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4)
