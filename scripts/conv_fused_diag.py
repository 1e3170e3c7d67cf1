"""Where a fused conv pair loses to its stream form: the same configuration with diagnostic
flag bits (12: no semaphore waits, 22: no release fence before posts, 23: no producer-done
watermark) and CTA counts. Results of the diagnostic variants are not checked.
usage: python scripts/conv_fused_diag.py 28:128:256:128:1 7:512:1:256:1:4"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402
from paper_2305_13450_b200.chains import ConvChain  # noqa: E402

if __name__ == "__main__":
    torch.manual_seed(11)
    for arg in sys.argv[1:]:
        f = [int(v) for v in arg.split(":")]
        hw, c, b, tn, cg = f[:5]
        z = f[5] if len(f) > 5 else 1
        w1 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        w2 = (torch.randn(c, 3, 3, c, device="cuda") / (9 * c) ** 0.5).half()
        x = torch.randn(b, hw, hw, c, device="cuda").half()
        base = dict(tile_n=tn, cta_group=cg, prod_splits=z, cons_splits=z)
        cfgs = {"stream": dict(base, mode="stream"), "fused": dict(base, mode="fused"),
                "fused no-wait(12)": dict(base, mode="fused", extra_flags=1 << 12),
                "fused no-fence(22)": dict(base, mode="fused", extra_flags=1 << 22),
                "fused no-watermark(23)": dict(base, mode="fused", extra_flags=1 << 23),
                "fused ctas=74": dict(base, mode="fused", num_ctas=74),
                "stream ctas=74": dict(base, mode="stream", num_ctas=74)}
        chains = {k: ConvChain(x, w1, w2, **kw) for k, kw in cfgs.items()}
        runs = {k: [] for k in chains}
        for _ in range(3):
            for k, ch in chains.items():
                runs[k].append(planner._time(ch, iters=20))
        print(f"layer {hw}x{hw}x{c} B={b} {base}", flush=True)
        for k in runs:
            print(f"   {statistics.median(runs[k]):7.1f} us  {k}", flush=True)
