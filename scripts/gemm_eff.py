"""Single-GeMM efficiency probe: one stage of the chain kernel (no dependencies) vs
cuBLAS on the same shape, with the SM clock and board power sampled (NVML) during each
timed loop, so efficiency can be compared per clock (MAC/clk/SM) as well as per second.

    python scripts/gemm_eff.py [M N K ...]
    python scripts/gemm_eff.py prof M N K [tile_n cta_group iters band]   # ours only (ncu)
"""
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402

SMS = 148


class Sampler:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.clk, self.pw = [], []

    def __enter__(self):
        self.stop = False
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def run(self):
        while not self.stop:
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000)
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop = True
        self.t.join()


def time_fn(fn, ms=300):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    iters = max(5, int(ms / max(e0.elapsed_time(e1), 1e-3)))
    s = Sampler()
    with s:
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    clk = statistics.median(s.clk[len(s.clk) // 4:]) if s.clk else float("nan")
    pw = statistics.median(s.pw[len(s.pw) // 4:]) if s.pw else float("nan")
    return us, clk, pw


def report(name, m, n, k, us, clk, pw, err=None):
    mac = m * n * k
    per_clk = mac / (us * 1e-6) / (clk * 1e6) / SMS
    e = f" err {err:.3g}" if err is not None else ""
    print(f"   {name:28s} {us:8.1f} us {2 * mac / us / 1e6:6.0f} TF/s  {clk:5.0f} MHz "
          f"{pw:4.0f} W  {per_clk:5.0f} MAC/clk/SM ({per_clk / 4096:.1%}){e}", flush=True)


def make_stage(x, w, c, tn, cg, band, flags=0, qd=1):
    """tn = 512: a double-width CTA-pair stage of a tile_n = 256 chain (qd = 2: on a
    two-pair cluster)."""
    cs = ts.CuSync(tile_n=min(tn, 256), cta_group=cg, mode="stream", extra_flags=flags,
                   cluster_pairs=qd)
    order = ts.BandedColumnMajor(band) if band > 1 else ts.RowMajor()
    cs.stage(x, w, c, order=order, tile_n=tn if tn > 256 else 0)
    return cs


def prof(m, n, k, tn=256, cg=2, iters=3, band=1):
    """Our kernel only (for ncu)."""
    dev = torch.device("cuda")
    x = torch.randn(m, k, device=dev).half()
    w = (torch.randn(n, k, device=dev) / k ** 0.5).half()
    c = torch.empty(m, n, device=dev, dtype=torch.half)
    cs = make_stage(x, w, c, tn, cg, band)
    for _ in range(iters):
        cs()
    torch.cuda.synchronize()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "prof":
        return prof(*[int(v) for v in sys.argv[2:]])
    shapes = [(8192, 8192, 8192), (1024, 6144, 12288), (1024, 12288, 6144), (2048, 6144, 12288)]
    if len(sys.argv) > 3:
        a = [int(v) for v in sys.argv[1:]]
        shapes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
    dev = torch.device("cuda")
    torch.manual_seed(0)
    for (m, n, k) in shapes:
        x = torch.randn(m, k, device=dev).half()
        w = (torch.randn(n, k, device=dev) / k ** 0.5).half()
        c = torch.empty(m, n, device=dev, dtype=torch.half)
        ref = (x.float() @ w.float().t())
        print(f"M={m} N={n} K={k}", flush=True)
        report("cublas", m, n, k, *time_fn(lambda: torch.matmul(x, w.t(), out=c)))
        for (tn, cg, qd) in ((512, 2, 1), (512, 2, 2), (256, 2, 1), (256, 1, 1)):
            for band in (1, 4):
                for gbits in ((1,) if band == 1 else (0,)):
                    if band * 128 * cg > m and band > 1:
                        continue
                    cs = make_stage(x, w, c, tn, cg, band, flags=gbits << 17, qd=qd)
                    cs()
                    torch.cuda.synchronize()
                    err = (c.float() - ref).abs().max().item()
                    grp = {0: 2, 1: 1, 2: 2, 3: 4}[gbits]
                    report(f"ours {128 * cg}x{tn} qd{qd} band{band} G{grp}", m, n, k, *time_fn(cs),
                           err=err)


if __name__ == "__main__":
    main()
