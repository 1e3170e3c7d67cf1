"""Diagnostic: GEMM1 alone (stream mode) at B=1 — MMA on/off (bit 13), activation
loads on/off (bit 15), for the normal N=64 tile (96 CTAs) and swapped N=32 split 3."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.small_batch import time_fn  # noqa: E402

H = 12288
torch.manual_seed(0)
for b in (1, 128):
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    h = torch.empty(b, H // 2, device="cuda").half()
    for label, kw, z in (("normal N64", dict(tile_n=64, cta_group=1), 1),
                         ("swap N32 z3", dict(tile_n=32, swap_ab=True), 3)):
        for flags, f in ((0, "mma+act"), (1 << 13, "act only"), (1 << 15, "mma no-act"),
                         ((1 << 13) | (1 << 15), "weights only")):
            cs = ts.CuSync(mode="stream", extra_flags=flags, **kw)
            st = cs.stage(x, w1, h, epilogue="gelu", splits=z)
            us = time_fn(cs.launch)
            print(f"B={b} {label:12s} {f:12s}: {st.grid.total():3d} units {us:6.1f} us  "
                  f"{151e6 / us / 1e6:.2f} TB/s", flush=True)
