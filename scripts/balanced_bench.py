"""Balanced (stream-K) schedule vs the planner's pick vs cuBLAS on the GPT-3 MLP shard,
plus a device-trace summary of the balanced chain. CUDA-event timing (planner._time).

    python scripts/balanced_bench.py B [B ...]
"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_2305_13450_b200 as ts  # noqa: E402
from paper_2305_13450_b200 import planner  # noqa: E402
from timeline import summarize  # noqa: E402

H, FFN = 12288, 6144
for b in [int(a) for a in sys.argv[1:]] or [1024]:
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(FFN, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device="cuda") / FFN ** 0.5).half()
    ref = torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t()
    res = {}
    cub = planner._time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(),
                        iters=20, warm=5)
    for name, kw in [
        ("bal row 512/512 band4", dict(policy=ts.RowSync(), prod_tile_n=512, cons_tile_n=512,
                                       cons_order=ts.BandedColumnMajor(4))),
        ("bal row 512/512 rowmajor", dict(policy=ts.RowSync(), prod_tile_n=512, cons_tile_n=512)),
        ("bal tile 512/512 band4", dict(policy=ts.TileSync(), prod_tile_n=512, cons_tile_n=512,
                                        cons_order=ts.BandedColumnMajor(4))),
        ("bal row 512/512 colmajor", dict(policy=ts.RowSync(), prod_tile_n=512, cons_tile_n=512,
                                          prod_order=ts.BandedColumnMajor(64),
                                          cons_order=ts.BandedColumnMajor(64))),
        ("bal row 256/512", dict(policy=ts.RowSync(), cons_tile_n=512)),
    ]:
        ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, balanced=True, **kw)
        res[name] = planner._time(ch, iters=20, warm=5)
        assert not ch.cs.watchdog_fired()
        err = (ch.y.float() - ref.float()).abs().max().item()
        assert err < 0.05, err
    pick, _ = planner.pick_mlp(x, w1, w2, mode="fused")
    chp = ts.MlpChain(x, w1, w2, **pick)
    res["pick " + str(planner.describe(pick))] = planner._time(chp, iters=20, warm=5)
    print(f"B={b}: cublas {cub:.1f} us")
    for k, v in res.items():
        print(f"   {v:7.1f} us  {k}")
    best = min((k for k in res if k.startswith("bal")), key=res.get)
    print("   trace of", best)
    kw = {"bal row 512/512 band4": dict(policy=ts.RowSync(), prod_tile_n=512, cons_tile_n=512,
                                        cons_order=ts.BandedColumnMajor(4))}.get(best)
    if kw:
        ch = ts.MlpChain(x, w1, w2, tile_n=256, cta_group=2, balanced=True, **kw)
        ch()
        ch.cs.enable_trace(1 << 17)
        ch()
        torch.cuda.synchronize()
        try:
            summarize(ch.cs, best)
        except Exception as e:  # trace summaries assume one claim per tile
            print("   (summary failed:", e, ")")
