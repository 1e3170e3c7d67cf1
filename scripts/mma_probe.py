"""Per-tile MMA issue efficiency of one GeMM stage from the device trace: cycles between a
tile's first MMA issue and its last commit vs the tensor-pipe floor (128 cycles per
256x256x16 pair MMA), and the time the MMA warp waited for operands.

    python scripts/mma_probe.py M N K tile_n [flags]
"""
import statistics
import sys

import torch

import os  # noqa: E402

sys.path.insert(0, ".")
if os.environ.get("TS_OLD"):  # A/B against a previous build copied to old_build/pkg_old
    sys.path.insert(0, "old_build")
    import pkg_old as ts  # noqa: E402
else:
    import paper_2305_13450_b200 as ts  # noqa: E402


def main():
    m, n, k, tn = (int(v) for v in sys.argv[1:5])
    flags = int(sys.argv[5], 0) if len(sys.argv) > 5 else 0
    band = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    swap = int(sys.argv[7]) if len(sys.argv) > 7 else 0  # swapped tile_n (small batch)
    splits = int(sys.argv[8]) if len(sys.argv) > 8 else 1
    x = torch.randn(m, k, device="cuda").half()
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).half()
    c = torch.empty(m, n, device="cuda", dtype=torch.half)
    order = ts.BandedColumnMajor(band) if band > 1 else ts.RowMajor()
    if swap:
        cs = ts.CuSync(tile_n=swap, swap_ab=True, mode="stream", extra_flags=flags)
        cs.stage(x, w, c, order=order, splits=splits)
    else:
        cs = ts.CuSync(tile_n=min(tn, 256), cta_group=2, mode="stream", extra_flags=flags)
        if tn > 256:
            cs.stage(x, w, c, tile_n=tn, order=order, splits=splits)
        else:
            cs.stage(x, w, c, order=order, splits=splits)
    cs()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        cs()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    cs.enable_trace()
    cs()
    torch.cuda.synchronize()
    recs = cs.trace_records()
    mb = {(r.stage, r.tb): r for r in recs if r.kind == 5}
    me = {(r.stage, r.tb): r for r in recs if r.kind == 6}
    kb = k // 64 // splits
    floor = kb * 4 * 128 * (tn // 256)
    wbytes = (128 if swap else tn) * kb * 64 * 2  # weight bytes one tile streams
    cyc, starve, ns = [], [], []
    for key, e in me.items():
        b = mb.get(key)
        if b is None or b.smid != e.smid:
            continue
        cyc.append((e.clk - b.clk) % (1 << 32))
        ns.append(e.t_ns - b.t_ns)
        starve.append(e.value)
    mhz = [c_ / t * 1e3 for c_, t in zip(cyc, ns) if t > 0]
    print(f"M={m} N={n} K={k} tile_n={tn} flags={flags:#x} band={band}: tiles {len(cyc)} "
          f"MMA cycles median {statistics.median(cyc):.0f} (floor {floor}, "
          f"eff {floor / statistics.median(cyc):.1%}), span {statistics.median(ns) / 1e3:.1f} us "
          f"at {statistics.median(mhz):.0f} MHz, operand wait median "
          f"{statistics.median(starve) / 1e3:.2f} us max {max(starve) / 1e3:.2f} us; weights "
          f"{wbytes / statistics.median(ns):.1f} GB/s per tile; kernel {us:.1f} us")


if __name__ == "__main__":
    main()
