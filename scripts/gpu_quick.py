"""Quick device check: the MLP chain in stream and fused modes for both CTA-group
variants against torch fp32 on the same fp16 inputs; then timings."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402


def ref_mlp(x, w1, w2):
    h = torch.nn.functional.gelu(x.float() @ w1.float().t()).to(x.dtype)
    return h, (h.float() @ w2.float().t())


def time_fn(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    timing = len(sys.argv) > 1 and sys.argv[1] == "time"
    cases = [(256, 1024, 1024, 1024, 256, ts.RowSync()),
             (200, 512, 512, 768, 128, ts.TileSync()),
             (300, 1024, 512, 512, 128, ts.TileSync()),
             (64, 1024, 512, 512, 256, ts.TileSync())]
    if timing:
        cases = [(b, 12288, 6144, 12288, 256, pol) for b in (256, 1024, 2048)
                 for pol in (ts.RowSync(), ts.TileSync())]
    for (m, k, n1, n2, tn, pol) in cases:
        x = torch.randn(m, k, device=dev).half()
        w1 = (torch.randn(n1, k, device=dev) / k ** 0.5).half()
        w2 = (torch.randn(n2, n1, device=dev) / n1 ** 0.5).half()
        h_ref, y_ref = ref_mlp(x, w1, w2)
        fl = 2 * m * k * n1 + 2 * m * n1 * n2
        for cg in (1, 2):
            for mode in ("stream", "fused"):
                ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn, cta_group=cg)
                y = ch()
                torch.cuda.synchronize()
                eh = (ch.h.float() - h_ref.float()).abs().max().item()
                ey = (y.float() - y_ref).abs().max().item()
                wd = ch.cs.watchdog_fired()
                us = time_fn(ch) if timing else 0.0
                print(f"m={m} k={k} n1={n1} n2={n2} tn={tn} cg={cg} {type(pol).__name__} {mode}: "
                      f"err_h={eh:.4f} err_y={ey:.4f} watchdog={wd} {us:.1f} us "
                      f"{fl / max(us, 1e-9) / 1e6:.0f} TF/s", flush=True)
        if timing:
            us = time_fn(lambda: torch.nn.functional.gelu(x @ w1.t()) @ w2.t())
            print(f"   cublas: {us:.1f} us {fl / us / 1e6:.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
