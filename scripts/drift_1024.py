"""Does a plan's time drift over many back-to-back launches, and do its outputs stay
bit-identical? (sustained_1024.py saw 'fused z1 Band4' at 310 then 366-382 us.)
Times blocks of 100 launches of the same chain and compares every block's output with the
first launch's (unsplit plans are deterministic).
usage: python scripts/drift_1024.py [BLOCKS=12]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 12
H, F = 12288, 6144
torch.manual_seed(0)
w1 = (torch.randn(F, H, device="cuda") / H ** 0.5).half()
w2 = (torch.randn(H, F, device="cuda") / F ** 0.5).half()
x = torch.randn(1024, H, device="cuda").half()
base = dict(policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)
for name, kw in (("z1 Band4", dict(base, cons_order=ts.BandedColumnMajor(4))),
                 ("z1 Band4 tail22x2", dict(base, cons_order=ts.BandedColumnMajor(4),
                                            cons_tail=(22, 2))),
                 ("z2 Band4 (fixed)", dict(base, prod_splits=2,
                                           cons_order=ts.BandedColumnMajor(4)))):
    ch = ts.MlpChain(x, w1, w2, **kw)
    ref = ch().clone()
    torch.cuda.synchronize()
    times, same = [], True
    for _ in range(blocks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            y = ch()
        e1.record()
        torch.cuda.synchronize()
        times.append(round(e0.elapsed_time(e1) * 10, 1))
        if "z2" not in name:
            same &= bool(torch.equal(y, ref))
        else:
            same &= bool(torch.allclose(y.float(), ref.float(), atol=2e-2, rtol=1e-2))
    assert not ch.cs.watchdog_fired(), name
    print(f"{name:20s} per-launch us by block of 100: {times}  outputs match first: {same}",
          flush=True)
