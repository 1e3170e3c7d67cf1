"""Device-trace timeline of one chain launch: per-stage tile durations, waits, and the
SM-occupancy profile of the tail wave. Usage: python scripts/timeline.py B POLICY TILE_N"""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H = 12288


def summarize(cs, label):
    evs = cs.trace_events()
    sched, fin, wb, we = {}, {}, defaultdict(float), {}
    for e in evs:
        key = (e.stage, e.tb)
        if e.kind == "scheduled":
            sched[key] = e.time
        elif e.kind == "finished":
            fin[key] = e.time
        elif e.kind == "wait_begin":
            we[(key, e.k)] = e.time
        elif e.kind == "wait_end":
            wb[key] += e.time - we[(key, e.k)]
    makespan = max(fin.values())
    print(f"== {label}: makespan {makespan / 1e3:.1f} us, events {len(evs)}")
    # per-tile SM clock from (clock64, globaltimer) at claim and at finish (same CTA)
    recs = cs.trace_records()
    start = {(r.stage, r.tb): r for r in recs if r.kind == 0}
    for s_i, st in enumerate(cs.stages):
        mhz = []
        for r in recs:
            if r.kind == 4 and r.stage == s_i and (r.stage, r.tb) in start:
                a = start[(r.stage, r.tb)]
                if a.smid == r.smid and r.t_ns > a.t_ns:
                    mhz.append(((r.clk - a.clk) % (1 << 32)) / (r.t_ns - a.t_ns) * 1e3)
        if mhz:
            mhz.sort()
            print(f"  {st.id}: SM clock per tile median {mhz[len(mhz) // 2]:.0f} MHz "
                  f"min {mhz[0]:.0f} max {mhz[-1]:.0f}")
    for st in cs.stages:
        d = [fin[k] - sched[k] for k in sched if k[0] == st.id]
        w = [wb[k] for k in sched if k[0] == st.id]
        s0 = min(sched[k] for k in sched if k[0] == st.id)
        f1 = max(fin[k] for k in fin if k[0] == st.id)
        print(f"  {st.id}: tiles {len(d)} dur mean {sum(d) / len(d) / 1e3:.1f} us "
              f"min {min(d) / 1e3:.1f} max {max(d) / 1e3:.1f}; wait mean {sum(w) / len(w) / 1e3:.2f} us "
              f"max {max(w) / 1e3:.1f}; span {s0 / 1e3:.1f}..{f1 / 1e3:.1f} us")
    mbr = {(r.stage, r.tb): r for r in recs if r.kind == 5}
    mb = {k: r.t_ns for k, r in mbr.items()}
    me = {(r.stage, r.tb): r for r in recs if r.kind == 6}
    t0 = min(r.t_ns for r in recs)
    for s_i, st in enumerate(cs.stages):
        keys = [k for k in me if k[0] == s_i and k in mb and k in start]
        if keys:
            mma = [me[k].t_ns - mb[k] for k in keys]
            cyc = [(me[k].clk - mbr[k].clk) % (1 << 32) for k in keys if me[k].smid == mbr[k].smid]
            starve = [me[k].value for k in keys]
            lead = [mb[k] - start[k].t_ns for k in keys]
            # ideal tensor cycles of one tile: 4096 MAC/clk per SM (8192 per CTA pair)
            macs = cs.tile_m * st.width * st.k // max(1, st.splits)
            ideal = macs / (4096 * (2 if cs.cta_group == 2 else 1) * cs.cluster_pairs)
            eff = (f", {sum(cyc) / len(cyc):.0f} cycles = {ideal / (sum(cyc) / len(cyc)) * 100:.0f}%"
                   f" of the MMA floor") if cyc and st.kind == "gemm" else ""
            print(f"  {st.id}: MMA span mean {sum(mma) / len(mma) / 1e3:.1f} us{eff}, "
                  f"operand-starved {sum(starve) / len(starve) / 1e3:.1f} us, claim->first MMA "
                  f"{sum(lead) / len(lead) / 1e3:.1f} us")
    eb = {(r.stage, r.tb): r.t_ns for r in recs if r.kind == 7}
    ee = {(r.stage, r.tb): r.t_ns for r in recs if r.kind == 8}
    for s_i, st in enumerate(cs.stages):
        d = [ee[k] - eb[k] for k in eb if k[0] == s_i and k in ee]
        lag = [eb[k] - me[k].t_ns for k in eb if k[0] == s_i and k in me]
        if d and lag:
            print(f"  {st.id}: epilogue mean {sum(d) / len(d) / 1e3:.1f} us (last MMA issue -> "
                  f"accumulator ready {sum(lag) / len(lag) / 1e3:.1f} us)")
        elif d:
            print(f"  {st.id}: compute mean {sum(d) / len(d) / 1e3:.1f} us")
    pw = {(r.stage, r.tb): r.t_ns for r in recs if r.kind == 9}
    for s_i, st in enumerate(cs.stages):
        w = [pw[k] - eb[k] for k in pw if k[0] == s_i and k in eb]
        rest = [ee[k] - pw[k] for k in pw if k[0] == s_i and k in ee]
        if w:
            print(f"  {st.id}: split-K partial write mean {sum(w) / len(w) / 1e3:.1f} us, "
                  f"then count + reduce mean {sum(rest) / len(rest) / 1e3:.1f} us "
                  f"(max {max(rest) / 1e3:.1f})")
    # MMA idle per CTA(-pair leader): before its first tile, between tiles, after its last
    per_sm = defaultdict(list)
    for k, r in me.items():
        if k in mb:
            per_sm[r.smid].append((mb[k], r.t_ns))
    if per_sm:
        t_end = max(e for v in per_sm.values() for _, e in v)
        head = gaps = tail = 0.0
        for v in per_sm.values():
            v.sort()
            head += v[0][0] - t0
            gaps += sum(max(0, v[i + 1][0] - v[i][1]) for i in range(len(v) - 1))
            tail += t_end - v[-1][1]
        n = len(per_sm)
        print(f"  MMA idle per unit ({n} units): head {head / n / 1e3:.1f} us, between tiles "
              f"{gaps / n / 1e3:.1f} us, tail {tail / n / 1e3:.1f} us "
              f"(makespan {(t_end - t0) / 1e3:.1f} us)")
    if len(cs.stages) > 1:
        p_end = max(fin[k] for k in fin if k[0] == cs.stages[0].id)
        for name, sel in (("during producers", lambda k: sched[k] < p_end),
                          ("after producers", lambda k: sched[k] >= p_end)):
            ks = [k for k in sched if k[0] == cs.stages[1].id and sel(k)]
            if ks:
                d = sum(fin[k] - sched[k] - wb[k] for k in ks) / len(ks)
                print(f"  {cs.stages[1].id} {name}: {len(ks)} tiles, mean busy (dur-wait) "
                      f"{d / 1e3:.1f} us")
    # busy tiles over time (in 5% buckets)
    nb = 20
    busy = [0.0] * nb
    for k in sched:
        a, b = sched[k], fin[k]
        for i in range(nb):
            lo, hi = makespan * i / nb, makespan * (i + 1) / nb
            busy[i] += max(0.0, min(b, hi) - max(a, lo)) / (hi - lo)
    print("  tiles in flight per 5% bucket:", " ".join(f"{b:.0f}" for b in busy))


def order(s):
    if s == "row":
        return ts.RowMajor()
    return ts.BandedColumnMajor(int(s[4:]))  # "band<N>"


def main():
    """argv: B then variants MODE:POLICY:PROD_ORDER:CONS_ORDER[:FLAGS:SWAP_TN:Z1/Z2:W1/W2:TAIL],
    e.g. fused:row:row:band4 or fused:row:row:band4:0:0:1/1:512/512:22,3"""
    b = int(sys.argv[1])
    variants = sys.argv[2:] or ["stream:row:row:row", "fused:row:row:row"]
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    for v in variants:
        parts = v.split(":")
        mode, pol, po, co = parts[:4]
        flags = int(parts[4], 0) if len(parts) > 4 else 0
        swap_tn = int(parts[5]) if len(parts) > 5 else 0
        zs = [int(z) for z in parts[6].split("/")] if len(parts) > 6 else [1]
        z1, z2 = zs[0], (zs[1] if len(zs) > 1 else 1)
        widths = [int(w) for w in parts[7].split("/")] if len(parts) > 7 else [0, 0]
        tail = tuple(int(t) for t in parts[8].split(",")) if len(parts) > 8 else (0, 1)
        qd = int(parts[9]) if len(parts) > 9 else 1
        policy = {"row": ts.RowSync(), "tile": ts.TileSync()}[pol]
        kw = dict(prod_splits=z1, cons_splits=z2, cons_tail=tail, cluster_pairs=qd)
        kw.update(dict(swap_ab=True, tile_n=swap_tn) if swap_tn else
                  dict(prod_tile_n=widths[0], cons_tile_n=widths[1]))
        ch = ts.MlpChain(x, w1, w2, policy=policy, mode=mode, prod_order=order(po),
                         cons_order=order(co), extra_flags=flags, **kw)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for _ in range(3):
            ch()
        e0.record()
        for _ in range(10):
            ch()
        e1.record()
        torch.cuda.synchronize()
        print(f"-- {v}: untraced {e0.elapsed_time(e1) / 10 * 1e3:.1f} us/chain")
        ch.cs.enable_trace()
        for _ in range(3):
            ch()
        torch.cuda.synchronize()
        summarize(ch.cs, f"B={b} {v}")


if __name__ == "__main__":
    main()
