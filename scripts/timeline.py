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
    for st in cs.stages:
        d = [fin[k] - sched[k] for k in sched if k[0] == st.id]
        w = [wb[k] for k in sched if k[0] == st.id]
        s0 = min(sched[k] for k in sched if k[0] == st.id)
        f1 = max(fin[k] for k in fin if k[0] == st.id)
        print(f"  {st.id}: tiles {len(d)} dur mean {sum(d) / len(d) / 1e3:.1f} us "
              f"min {min(d) / 1e3:.1f} max {max(d) / 1e3:.1f}; wait mean {sum(w) / len(w) / 1e3:.2f} us "
              f"max {max(w) / 1e3:.1f}; span {s0 / 1e3:.1f}..{f1 / 1e3:.1f} us")
    # busy tiles over time (in 5% buckets)
    nb = 20
    busy = [0.0] * nb
    for k in sched:
        a, b = sched[k], fin[k]
        for i in range(nb):
            lo, hi = makespan * i / nb, makespan * (i + 1) / nb
            busy[i] += max(0.0, min(b, hi) - max(a, lo)) / (hi - lo)
    print("  tiles in flight per 5% bucket:", " ".join(f"{b:.0f}" for b in busy))


def main():
    b, pol, tn = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    policy = {"row": ts.RowSync(), "tile": ts.TileSync()}[pol]
    for mode in ("stream", "fused"):
        ch = ts.MlpChain(x, w1, w2, policy=policy, mode=mode, tile_n=tn)
        ch.cs.enable_trace()
        for _ in range(3):
            ch()
        torch.cuda.synchronize()
        summarize(ch.cs, f"B={b} {mode} {pol} tn={tn}")


if __name__ == "__main__":
    main()
