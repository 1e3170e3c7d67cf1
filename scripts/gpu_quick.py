"""Quick device check: one GeMM, then the MLP chain in stream and fused modes, against
torch fp32 on the same fp16 inputs. Prints max errors and timings."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402


def ref_mlp(x, w1, w2):
    h = torch.nn.functional.gelu(x.float() @ w1.float().t()).to(x.dtype)
    return h, (h.float() @ w2.float().t())


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    for (m, k, n1, n2, tn, pol) in [(256, 1024, 1024, 1024, 256, ts.RowSync()),
                                    (200, 512, 512, 768, 128, ts.TileSync()),
                                    (64, 1024, 512, 512, 64, ts.TileSync()),
                                    (1024, 12288, 6144, 12288, 256, ts.RowSync())]:
        x = torch.randn(m, k, device=dev).half()
        w1 = (torch.randn(n1, k, device=dev) / k ** 0.5).half()
        w2 = (torch.randn(n2, n1, device=dev) / n1 ** 0.5).half()
        h_ref, y_ref = ref_mlp(x, w1, w2)
        for mode in ("stream", "fused"):
            ch = ts.MlpChain(x, w1, w2, policy=pol, mode=mode, tile_n=tn)
            y = ch()
            torch.cuda.synchronize()
            eh = (ch.h.float() - h_ref.float()).abs().max().item()
            ey = (y.float() - y_ref).abs().max().item()
            wd = ch.cs.watchdog_fired()
            # timing
            for _ in range(3):
                ch()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(10):
                ch()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 10 * 1e3
            tf = 2 * m * k * n1 + 2 * m * n1 * n2
            print(f"m={m} k={k} n1={n1} n2={n2} tn={tn} {type(pol).__name__} {mode}: "
                  f"err_h={eh:.4f} err_y={ey:.4f} watchdog={wd} {us:.1f} us "
                  f"{tf / us / 1e6:.1f} TFLOP/s", flush=True)
        # cuBLAS reference timing
        def cub():
            h = torch.nn.functional.gelu(x @ w1.t())
            return h @ w2.t()
        for _ in range(3):
            cub()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            cub()
        e1.record()
        torch.cuda.synchronize()
        print(f"   cublas: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
