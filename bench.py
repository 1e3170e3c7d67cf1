"""Benchmark: GPT-3 145B MLP tensor-parallel shard, GeMM -> GeLU -> GeMM, fp16, on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Metric (BASELINE.json): dependent-GeMM chain latency in microseconds (lower is better),
with the speed-up over the stream-synchronized baseline reported beside it.

Workload (BASELINE.json configs[1]): X[B, 12288] x W1[12288, 6144] -> GeLU -> x W2[6144,
12288] — the per-GPU shard of GPT-3 145B's MLP at TP=8. Weights
are random-init with that architecture, inputs synthetic (no network). One step = one
chain; with N > 1 ranks each rank runs its TP shard chain and the row-parallel output is
all-reduced over NCCL (N = 8 is exactly the TP=8 layer; per-GPU work is fixed, so
scaling is "weak"). The weights (302 MB) are larger than L2 (126 MB), so no L2 flush is
needed between steps.

Arms
  ours       one persistent tcgen05 launch per chain with tile semaphores (CuSync fused).
             Also measured, on the same box: the same kernel in stream mode (the
             stream-synchronized baseline) and torch/cuBLAS.
  reference  the CPU restatement of the chain under the paper's protocol
             (oracle/tilesync_oracle.run_chain_cpu, all host threads), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

H = 12288
FFN = 6144  # 4H / 8: the TP=8 shard of the MLP's inner dimension


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--fused-allreduce", action="store_true",
                    help="also time the chain with the tensor-parallel all-reduce fused into "
                         "it (FusedTPMlp over torch symmetric memory) beside chain + NCCL")
    ap.add_argument("--plan", choices=["auto", "fixed"], default="auto",
                    help="auto: time the planner's candidates; fixed: the B=1024 headline "
                         "configuration without the search (for profiling runs)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """NVML polling (SM clock, throttle reasons) in a thread during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.0005)  # the timed region can be a few ms (20 chains)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._sample()  # the end of the timed region (the GPU just went idle)
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": names, "samples": len(self.samples)}


# idle seconds before each device-timed arm (see main()): the power-capped clock recovers
# its burst level at rest, so every arm is timed from the same rested state with the
# paper's protocol (W warm-up chains, then K timed)
REST_S = 1.0


def time_steps(fn, steps, warmup, torch, dist=None, poll=None):
    """Device time per step (us): W untimed steps, then exactly K steps bracketed by a
    barrier and synchronize, timed with CUDA events on the launching stream; max over
    ranks."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    if poll is not None:
        # clock samples while the enqueued steps run (the launches return at once, so the
        # timed region on the device is mostly ahead of the host here)
        while not e1.query():
            poll()
            time.sleep(0.0002)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    if dist is not None:
        t = torch.tensor([us], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t.item())
        dist.barrier()
    return us


def cpu_baseline_sample(b, budget_s=20.0):
    """The oracle's CPU chain (run_chain_cpu, all host threads) on the same workload,
    timed for a bounded ~20 s sample on rank 0 — a reported baseline, not the target."""
    import numpy as np

    from oracle import tilesync_oracle as O
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    x = O.round_to(rng.standard_normal((b, H), dtype=np.float32), "fp16")
    w1 = O.round_to(rng.standard_normal((FFN, H), dtype=np.float32) / H ** 0.5, "fp16")
    w2 = O.round_to(rng.standard_normal((H, FFN), dtype=np.float32) / FFN ** 0.5, "fp16")
    O.run_chain_cpu(x, w1, w2, threads=cores)
    times, t_start = [], time.perf_counter()
    while not times or time.perf_counter() - t_start < budget_s:
        t0 = time.perf_counter()
        O.run_chain_cpu(x, w1, w2, threads=cores)
        times.append(time.perf_counter() - t0)
        if len(times) >= 20:
            break
    return {"value": statistics.mean(times) * 1e6, "unit": "us", "cores": cores, "kind": "port",
            "sample": f"{len(times)} full chains B={b} (fp32 numpy, RowSync, 256x256 tiles, "
                      f"{cores}-thread pool) after 1 warm-up"}


def run_reference(args):
    """The reference arm: the CPU restatement of the chain, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from oracle import tilesync_oracle as O
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    x = O.round_to(rng.standard_normal((args.batch, H), dtype=np.float32), "fp16")
    w1 = O.round_to(rng.standard_normal((FFN, H), dtype=np.float32) / H ** 0.5, "fp16")
    w2 = O.round_to(rng.standard_normal((H, FFN), dtype=np.float32) / FFN ** 0.5, "fp16")
    budget_s = 90.0
    for _ in range(min(args.warmup, 1)):
        O.run_chain_cpu(x, w1, w2, threads=cores)
    times = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.run_chain_cpu(x, w1, w2, threads=cores)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    us = statistics.mean(times) * 1e6
    sample = (f"full GPT-3 MLP shard chain B={args.batch} in fp32 numpy, RowSync over "
              f"256x256 tiles on a {cores}-thread pool; {len(times)} of {args.steps} "
              f"requested steps timed (90 s budget)")
    out = {
        "impl": "reference", "metric": "GPT-3 MLP/attn dependent-GeMM latency (µs), "
        "speedup vs stream-sync baseline", "value": us, "unit": "us", "n_gpus": args.gpus,
        "steps": len(times), "warmup": min(args.warmup, 1), "ms_per_step": us / 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic",
        "config": {"workload": "gpt3_mlp_tp8_shard", "batch": args.batch, "hidden": H,
                   "ffn_shard": FFN, "policy": "RowSync", "parallelism": f"tp{args.gpus}"},
        "cpu_baseline": {"value": us, "unit": "us", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2305_13450_b200 as ts
    from paper_2305_13450_b200 import planner

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    use_dist = world > 1
    if use_dist:
        # NCCL's INIT lines (rank/nranks, NVLS/P2P transport) go to stderr-side logs; the
        # JSON headline is printed last, after the process group is destroyed
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    b = args.batch
    dev = torch.device("cuda", local)
    # tensor parallelism: every rank sees the same activations X (replicated), and holds
    # its own W1 column shard / W2 row shard (seeded per rank)
    torch.manual_seed(1234)
    x = torch.randn(b, H, device=dev).half()
    torch.manual_seed(1234 + 7919 * rank)
    w1 = (torch.randn(FFN, H, device=dev) / H ** 0.5).half()
    w2 = (torch.randn(H, FFN, device=dev) / FFN ** 0.5).half()
    flops = 2 * b * H * FFN * 2

    # co-scheduling choice (policy, tile order, CTA group) from measured candidates; the
    # fixed plan is the B=1024 configuration that led every A/B of round 2
    # (profiles/r02ff_ready_first_and_ring.txt): GeMM1 in two split-K slices, GeMM2
    # claimed in bands of four row tiles
    fixed = dict(policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512,
                 cons_tile_n=512, prod_splits=2, cons_order=ts.BandedColumnMajor(4))
    if args.plan == "auto":
        best, cands = planner.pick_mlp(x, w1, w2, mode="fused")
        base, bcands = planner.pick_mlp(x, w1, w2, mode="stream")
        if b == 1024:
            # guard against a noisy pick: the planner's choice and the fixed plan are
            # re-timed round robin under sustained load (4 x 200 chains each: the power cap
            # settles over ~100 ms, and short bursts favour the split plans whose extra
            # DRAM traffic costs clock later; profiles/r02s3e_sustained.txt) and the faster
            # median is kept, the fixed plan on ties
            # (with the lowest-traffic plan, unsplit GeMM1 + a 2-slice GeMM2 tail: 354 MB
            # per launch vs 613 for the fixed plan; sustained, DRAM traffic costs clock)
            lean = dict(fixed, mode="fused", prod_splits=1, cons_tail=(22, 2))
            best = planner.pick_between(x, w1, w2, [dict(fixed, mode="fused"), best, lean],
                                        rounds=4, iters=200)
    else:
        best, cands = dict(fixed, mode="fused"), []
        base, bcands = dict(fixed, mode="stream"), []
    chain = ts.MlpChain(x, w1, w2, **best)
    stream_chain = ts.MlpChain(x, w1, w2, **base)

    kernel_events = []  # (start, end) CUDA events around each chain launch, timed region

    def step():
        if record_kernel[0]:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            y = chain()
            e1.record()
            kernel_events.append((e0, e1))
        else:
            y = chain()
        if use_dist:
            dist.all_reduce(y)

    record_kernel = [False]

    def step_stream():
        y = stream_chain()
        if use_dist:
            dist.all_reduce(y)

    def step_cublas():
        y = torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t()
        if use_dist:
            dist.all_reduce(y)

    sampler = ClockSampler(local)
    # Each device-timed arm (fused, stream, cuBLAS) starts from rest (REST_S idle), then
    # runs its W warm-up steps and its K timed steps. Without the rest the arm timed first
    # inherits the clock the planner's timings left under sw_power_cap (the cap settles
    # over ~300 chains, scripts/drift_1024.py), and 20-step bursts swung the fused/stream
    # ratio between 0.89 and 1.09 on one plan (profiles/r02s3e_sustained.txt).
    torch.cuda.synchronize()
    time.sleep(REST_S)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    with sampler:
        record_kernel[0] = True
        us = time_steps(step, args.steps, 0, torch, dist if use_dist else None,
                        poll=sampler._sample if sampler.ok else None)
        record_kernel[0] = False
    time.sleep(REST_S)
    us_stream = time_steps(step_stream, args.steps, args.warmup, torch, dist if use_dist else None)
    time.sleep(REST_S)
    us_cublas = time_steps(step_cublas, args.steps, args.warmup, torch, dist if use_dist else None)
    us_fused_ar = None
    if args.fused_allreduce:
        # the all-reduce inside the chain: tile t summed by rank t % world over NVLink peer
        # memory as soon as every rank posted it (tp.FusedTPMlp, symmetric-memory pointers)
        from paper_2305_13450_b200.tp import FusedTPMlp
        if not use_dist:
            import socket
            so = socket.socket()
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
            so.close()
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev,
                                    init_method=f"tcp://127.0.0.1:{port}")
        # (a stage that feeds the all-reduce cannot carry last-wave tail slices)
        far = FusedTPMlp.from_group(x, w1, w2, **dict(best, cons_tail=(0, 1)))
        us_fused_ar = time_steps(far, args.steps, args.warmup, torch, dist if use_dist else None)
        assert not far.chain.cs.watchdog_fired(), "semaphore watchdog fired (fused all-reduce)"

    # kernel-only duration of the chain launch (roofline denominator): the average of the
    # per-launch CUDA-event durations recorded inside the timed region, on the launch stream
    us_kernel = statistics.mean(a.elapsed_time(b) for a, b in kernel_events) * 1e3
    assert not chain.cs.watchdog_fired(), "semaphore watchdog fired"

    # end to end through the public API with host buffers: pinned X -> device, chain,
    # Y -> pinned host, every step, inside the timed region
    xh = x.cpu().pin_memory()
    yh = torch.empty(b, H, dtype=torch.float16).pin_memory()
    # the end-to-end chain completes rows in order (RowMajor consumer) so finished row
    # units can leave over PCIe while later rows compute
    # (split-K slices finish the last row sooner on the device but gated by PCIe the
    # unsplit chain was measured faster end to end: both are timed, the faster kept)
    # (the row-tile copy gates count whole tiles per row: no last-wave tail slices here)
    e2e_opts = [dict(best, cons_order=ts.RowMajor(), cons_tail=(0, 1))]
    if best.get("prod_splits", 1) > 1 or best.get("cons_splits", 1) > 1:
        e2e_opts.append(dict(best, cons_order=ts.RowMajor(), prod_splits=1, cons_splits=1,
                             cons_tail=(0, 1)))
    e2e_cands = [ts.MlpChain(x.clone(), w1, w2, **kw) for kw in e2e_opts]
    e2e_chain = min(e2e_cands, key=lambda c: planner._time(lambda: c.run_host(xh, yh)))

    def step_e2e():
        if use_dist:
            chain.x.copy_(xh, non_blocking=True)
            y = chain()
            dist.all_reduce(y)
            yh.copy_(y, non_blocking=True)
        else:
            # row-chunked H2D / D2H overlapped with the chain through row semaphores
            e2e_chain.run_host(xh, yh)

    us_e2e = time_steps(step_e2e, args.steps, args.warmup, torch, dist if use_dist else None)

    def step_e2e_stream():
        # the same end-to-end step synchronized by stream order: H2D, chain, D2H
        e2e_chain.x.copy_(xh, non_blocking=True)
        y = e2e_chain()
        if use_dist:
            dist.all_reduce(y)
        yh.copy_(y, non_blocking=True)

    us_e2e_stream = time_steps(step_e2e_stream, args.steps, args.warmup, torch,
                               dist if use_dist else None)

    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        sweep = {"gpt3_mlp": planner.sweep_mlp(batches=(1, 64, 256, 512, 1024, 2048), device=dev),
                 "gpt3_attention": planner.sweep_attention(device=dev),
                 "resnet38_conv_pairs": planner.sweep_conv(batches=(1, 8, 32, 128, 256),
                                                           device=dev),
                 "vgg19_conv_pairs": planner.sweep_conv(batches=(1, 8, 32),
                                                        layers=planner.VGG19_LAYERS, device=dev),
                 "llama8b_swiglu": planner.sweep_swiglu(device=dev)}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return
    burst, sustained, hbm, which = peaks()
    achieved = flops / (us_kernel * 1e-6) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "roofline_traffic.json"
    if prof.exists():
        # the ncu capture counts only for the configuration it was taken on
        for rec in json.loads(prof.read_text()).values():
            if rec["config"] == planner.describe(best) and rec["batch"] == b:
                traffic = rec["bytes"]
    # the CPU baseline (reference's algorithm restated in numpy, all host threads) is a
    # bounded ~20 s sample on rank 0 at every N
    cpu_baseline = cpu_baseline_sample(b)
    # Detail (candidate timings, the per-config sweep) goes to an earlier stdout line and
    # to gpurun_out/ when present; the LAST line is the compact headline the driver parses.
    detail = {"candidates": {"fused": cands, "stream": bcands}, "sweep": sweep}
    out_dir = ROOT / "gpurun_out"
    if out_dir.is_dir():
        (out_dir / "bench_detail.json").write_text(json.dumps(detail, indent=1))
    print(json.dumps({"detail": "sweep + candidates", "sweep_rows": {
        k: [{kk: vv for kk, vv in r.items() if kk.endswith("_us") or kk in ("batch", "seq",
            "layer", "tp")} for r in v] for k, v in (sweep or {}).items()}}))
    d = planner.describe(best)
    chain_s = (f"{d['mode']} {d['policy']} {d['tile']} cg{d['cta_group']} "
               f"splits{d['splits'][0]}/{d['splits'][1]} {d['consumer_order']}"
               + (f" tail{d['consumer_tail']}" if "consumer_tail" in d else "")
               + (f" reduce:{d['reduce']}" if "reduce" in d else ""))
    out = {
        "metric": "GPT-3 MLP/attn dependent-GeMM latency (µs), speedup vs stream-sync baseline",
        "value": round(us, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(us / 1e3, 5), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic (random-init GPT-3 shard)",
        "config": {"workload": "gpt3_mlp_tp8_shard", "batch": b, "hidden": H,
                   "ffn_shard": FFN, "global_batch": b, "parallelism": f"tp{world}",
                   "chain": chain_s, "l2": "inputs larger than L2 (weights 302 MB)"},
        "stream_sync_us": round(us_stream, 2), "speedup_vs_stream": round(us_stream / us, 4),
        "cublas_us": round(us_cublas, 2), "speedup_vs_cublas": round(us_cublas / us, 4),
        **({"fused_allreduce_us": round(us_fused_ar, 2)} if us_fused_ar is not None else {}),
        "kernel_us": round(us_kernel, 2),
        # the kernel is timed in a short burst from rest (REST_S), so the denominator is
        # the burst bf16 figure; the fraction of the sustained figure rides along
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": burst,
                     "unit": "TFLOP/s", "frac": round(achieved / burst, 4), "traffic": traffic,
                     "algorithmic_flops": flops, "peak_source": f"{which} bf16 burst",
                     "frac_of_sustained": round(achieved / sustained, 4)},
        "cpu_baseline": cpu_baseline,
        "e2e": {"value": round(us_e2e, 2), "unit": "us", "h2d_bytes_per_step": b * H * 2,
                "d2h_bytes_per_step": b * H * 2, "stream_sync_us": round(us_e2e_stream, 2)},
        "gpu_launches": args.steps,
        "clocks": sampler.summary(),
    }
    if dist.is_initialized():
        dist.destroy_process_group()
    sys.stdout.flush()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
