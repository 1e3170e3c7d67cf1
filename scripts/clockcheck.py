"""Run each chain variant back to back for ~3 s while sampling SM clocks and power."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

H = 12288


def sample_during(fn, seconds=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
            n += 1
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    clk = sorted(int(l.split(",")[0]) for l in out if l.strip())
    pw = sorted(float(l.split(",")[1]) for l in out if l.strip())
    return e0.elapsed_time(e1) / n * 1e3, clk[len(clk) // 2], pw[len(pw) // 2], out[len(out) // 2]


def main():
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    torch.manual_seed(0)
    x = torch.randn(b, H, device="cuda").half()
    w1 = (torch.randn(H // 2, H, device="cuda") / H ** 0.5).half()
    w2 = (torch.randn(H, H // 2, device="cuda") / (H // 2) ** 0.5).half()
    variants = {
        "cublas": lambda: torch.nn.functional.gelu(x @ w1.t()) @ w2.t(),
        "stream": ts.MlpChain(x, w1, w2, mode="stream"),
        "fused_row": ts.MlpChain(x, w1, w2, policy=ts.RowSync()),
        "fused_tile": ts.MlpChain(x, w1, w2, policy=ts.TileSync()),
    }
    for name, fn in variants.items():
        us, clk, pw, raw = sample_during(fn)
        print(f"B={b} {name:10s} {us:8.1f} us/chain  sm_clk_median={clk} MHz power={pw:.0f} W  [{raw}]",
              flush=True)


if __name__ == "__main__":
    main()
