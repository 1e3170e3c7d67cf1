"""Mainloop probe: one GeMM stage of the chain kernel (stream mode) under diagnostic flag
variants, timed (CUDA events, NVML clock) and then traced once for per-tile MMA span,
operand starvation and epilogue time (scripts/timeline.summarize).

    python scripts/mainloop_probe.py M N K TILE_N CG VARIANT...
VARIANT = name=flags (decimal), e.g. base=0 nowait=524288 (bit 19: MMA without operand
waits) ahint=2048 (A evict_first) ...
"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import paper_2305_13450_b200 as ts  # noqa: E402
from gemm_eff import report, time_fn  # noqa: E402
from timeline import summarize  # noqa: E402


def main():
    m, n, k, tn, cg = (int(v) for v in sys.argv[1:6])
    variants = [v.split("=") for v in sys.argv[6:]] or [["base", "0"]]
    dev = torch.device("cuda")
    torch.manual_seed(0)
    x = torch.randn(m, k, device=dev).half()
    w = (torch.randn(n, k, device=dev) / k ** 0.5).half()
    c = torch.empty(m, n, device=dev, dtype=torch.half)
    print(f"M={m} N={n} K={k} tile {128 * cg}x{tn}", flush=True)
    report("cublas", m, n, k, *time_fn(lambda: torch.matmul(x, w.t(), out=c)))
    for name, fl in variants:
        cs = ts.CuSync(tile_n=min(tn, 256), cta_group=cg, mode="stream", extra_flags=int(fl))
        cs.stage(x, w, c, tile_n=tn if tn > 256 else 0)
        report(f"ours {name}", m, n, k, *time_fn(cs))
        cs.enable_trace(1 << 16)
        cs()
        torch.cuda.synchronize()
        summarize(cs, name)


if __name__ == "__main__":
    main()
