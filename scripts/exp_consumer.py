"""Why are consumer tiles slower in a fused launch? Compare GeMM2 tile durations when
(A) launched alone after GeMM1, (B) fused with GeMM1 without a dependency, (C) fused
with RowSync, (D) fused with RowSync but the wait skipped (diagnostic flag)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from scripts.timeline import summarize  # noqa: E402

H = 12288


def build(x, w1, w2, h, y, mode, dep, flags, band):
    cs = ts.CuSync(mode=mode, extra_flags=flags)
    p = cs.stage(x, w1, h, epilogue="gelu", id="gemm1")
    c = cs.stage(h, w2, y, id="gemm2", order=ts.BandedColumnMajor(band) if band else ts.RowMajor())
    if dep:
        cs.dependency(ts.RowSync(), p, c)
    return cs


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    band = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    h = torch.empty(b, H // 2, device="cuda").half()
    y = torch.empty(b, H, device="cuda").half()
    for label, mode, dep, flags in (("A stream", "stream", False, 0),
                                    ("B fused-nodep", "fused", False, 0),
                                    ("C fused-row", "fused", True, 0),
                                    ("D fused-row-nowait", "fused", True, 0x1000),
                                    ("E fused-row-noreorder", "fused", True, 0x2)):
        cs = build(x, w1, w2, h, y, mode, dep, flags, band)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for _ in range(3):
            cs.launch()
        e0.record()
        for _ in range(10):
            cs.launch()
        e1.record()
        torch.cuda.synchronize()
        print(f"-- {label}: untraced {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
        cs.enable_trace()
        for _ in range(2):
            cs.launch()
        torch.cuda.synchronize()
        summarize(cs, f"B={b} {label}")


if __name__ == "__main__":
    main()
