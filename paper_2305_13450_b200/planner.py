"""Co-scheduling planner: pick the tile shape, CTA group, policy and tile orders of a
chain from measured candidates on the device it will run on.

The paper observes that no single policy wins everywhere; which one wins
on B200 depends on wave quantization over 148 SMs, on HBM reuse of
the weight panels and on the power cap. Rather than model all of that, the planner times
a small candidate set with CUDA events (3 warm-up + 10 timed launches each) and keeps
the fastest. ``wave_table`` gives the closed-form wave arithmetic the candidates come
from (reference gpu.waves at GpuConfig(148)).
"""

from __future__ import annotations

import itertools
import statistics

import torch

from .chains import MlpChain
from .gpu import GpuConfig, waves
from .policies import BandedColumnMajor, RowMajor, RowSync, TileSync


def _time(fn, iters=10, warm=3) -> float:
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def _check_watchdog(ch, kw) -> None:
    """A fired semaphore watchdog is a deadlock or a protocol bug, never a slow
    candidate: fail loudly (the device analogue of detect_deadlock, engine.py:614-637)."""
    if ch.cs.watchdog_fired():
        raise RuntimeError(f"semaphore watchdog fired while timing candidate {kw}")


def chain_units(tile_n: int = 256, cta_group: int = 2, cluster_pairs: int = 1,
                swap_ab: bool = False, dtype: torch.dtype = torch.float16) -> int:
    """Work items the current device runs at once for this chain geometry (CTAs, CTA
    pairs or two-pair clusters; co-resident cluster count from the driver)."""
    import ctypes

    from . import _lib
    out = ctypes.c_int(0)
    _lib.check(_lib.load().ts_chain_units(tile_n, cta_group, cluster_pairs, int(swap_ab),
                                          _lib.TS_DTYPE_BF16 if dtype == torch.bfloat16
                                          else _lib.TS_DTYPE_F16, ctypes.byref(out)))
    return out.value


def candidates(m: int, mode: str, n2: int | None = None, units: int = 74,
               qd_units: int | None = None):
    """Candidate chain configurations for `m` activation rows.

    Large batch: normal tiles (activations on the UMMA M side), CTA pairs or single CTAs,
    RowMajor or band-ordered consumers. Small batch (m <= 256, HBM-bound on weights):
    swapped tiles (weights on the UMMA M side, activations as UMMA N = the smallest tile
    width >= m) with split-K slices so every SM streams weights.
    """
    out = []
    pols = [RowSync(), TileSync()] if mode == "fused" else [RowSync()]
    if m <= 256:
        tn = next(t for t in (32, 64, 128, 256) if t >= m)
        for z1, z2 in ((3, 3), (3, 1), (6, 3), (3, 2), (2, 2), (1, 1)):
            for pol in pols:
                out.append(dict(policy=pol, mode=mode, tile_n=tn, cta_group=1, swap_ab=True,
                                prod_splits=z1, cons_splits=z2))
        # normal layout with split-K: weights on the UMMA N side (256 rows per MMA, 2.6x
        # the weight bytes per MMA of the swapped layout); the activation rows pad a
        # 128-row tile and split-K slices fill the SMs
        for tn_n, zs in ((256, ((6, 3), (6, 6), (3, 3), (4, 2))) if m <= 128 else (256, ()),
                         (128, ((3, 3), (3, 1), (6, 3), (2, 2)))):
            for (z1, z2), pol in itertools.product(zs, pols):
                out.append(dict(policy=pol, mode=mode, tile_n=tn_n, cta_group=1,
                                prod_splits=z1, cons_splits=z2))
    for cg, tn in ((2, 256), (1, 256), (2, 128), (1, 128)):
        gx = -(-m // (128 * cg))
        # consumer orders: RowMajor, and bands of 2 / 3 / 4 row tiles (a band shares each
        # weight column block in L2; a narrower band puts the last producer row's tiles
        # later in the claim order, where they wait less)
        orders = [RowMajor()] + [BandedColumnMajor(b) for b in sorted({2, 3, min(gx, 4)})
                                 if 1 < b <= gx]
        # per-stage widths: CTA-pair 256-wide chains may give either stage double-width
        # (256 x 512) tiles — fewer operand bytes per MAC, coarser wave quantization
        # (256 x 384 = two N = 192 MMAs: B=1024's GeMM1 as 64 tiles keeps 64 of 74 pairs
        # busy instead of 48)
        widths = ([(0, 0), (0, 512), (512, 512), (512, 0), (384, 512), (384, 384)]
                  if (cg, tn) == (2, 256) else [(0, 0)])
        for pol, co, (pw, cw) in itertools.product(pols, orders, widths):
            out.append(dict(policy=pol, mode=mode, tile_n=tn, cta_group=cg, cons_order=co,
                            prod_tile_n=pw, cons_tile_n=cw))
        if (cg, tn) == (2, 256) and m <= 512:
            # Mid batch: a handful of 256 x 512 CTA-pair tiles per stage, split-K slices
            # (weights on the UMMA N side, 256 rows per MMA) to occupy every pair
            for (z1, z2), pol in itertools.product(((6, 3), (4, 2), (6, 2), (3, 3), (4, 4)), pols):
                out.append(dict(policy=pol, mode=mode, tile_n=tn, cta_group=cg,
                                prod_tile_n=512, cons_tile_n=512, prod_splits=z1, cons_splits=z2))
        if (cg, tn) == (2, 256) and m >= 512:
            # Large batch: GeMM1 has fewer double-width tiles than CTA pairs (B=1024: 48
            # for 74), so its split-K slices fill the idle pairs and finish rows sooner
            for pol, co, z1 in itertools.product(pols, orders, (2, 3)):
                out.append(dict(policy=pol, mode=mode, tile_n=tn, cta_group=cg, cons_order=co,
                                prod_tile_n=512, cons_tile_n=512, prod_splits=z1))
            if n2 and n2 % 512 == 0:
                # last-wave balancing: GeMM2's final partial wave as split-K slices
                tiles2 = -(-m // 256) * (n2 // 512)
                rem = tiles2 % units
                if rem:
                    # GeMM1 in 3 slices finishes in ~2 waves of short items (B=1024: 144 on
                    # 74 pairs) instead of a full second wave gating its last row; the tail
                    # sizes bracket GeMM2's partial last wave
                    tails = sorted({rem, min(tiles2, rem + units // 2)})
                    for co, z1, zt, tt in itertools.product(orders, (1, 2, 3), (2, 3), tails):
                        out.append(dict(policy=RowSync(), mode=mode, tile_n=tn, cta_group=cg,
                                        cons_order=co, prod_tile_n=512, cons_tile_n=512,
                                        prod_splits=z1, cons_tail=(tt, zt)))
                    for co, zt in itertools.product(orders, (2, 3)):
                        out.append(dict(policy=RowSync(), mode=mode, tile_n=tn, cta_group=cg,
                                        cons_order=co, prod_tile_n=384, cons_tile_n=512,
                                        cons_tail=(rem, zt)))
        if (cg, tn) == (2, 256) and m >= 256:
            # two-pair clusters: the 256 x 512 tile on two CTA pairs sharing the activation
            # rows by multicast (24 KB of operands per SM and K-block, double-buffered
            # accumulators): half the tile time of one pair, so GeMM1 at B=1024 is 1.3
            # waves of 37 clusters instead of 0.65 of 74 pairs
            qd = dict(tile_n=tn, cta_group=cg, cluster_pairs=2, prod_tile_n=512,
                      cons_tile_n=512)
            qu = qd_units or max(1, units // 2)
            for pol, co, z1 in itertools.product(pols, orders, (1, 2, 3)):
                out.append(dict(qd, policy=pol, mode=mode, cons_order=co, prod_splits=z1))
            if n2 and n2 % 512 == 0:
                rem = (-(-m // 256) * (n2 // 512)) % qu
                if rem:
                    for co, z1, zt in itertools.product(orders, (1, 2, 3), (2, 3)):
                        out.append(dict(qd, policy=RowSync(), mode=mode, cons_order=co,
                                        prod_splits=z1, cons_tail=(rem, zt)))
    return out


# split-K reduction variants (chain flags): the owner slice's tensor-core reduction
# (D += P x I over TMA-streamed partial planes, bit 27) and every slice publishing a plane
# for the last arriver to sum (bit 29); neither wins everywhere (profiles/r02x_reduce_ab.txt)
REDUCE_TC, REDUCE_ALL_PLANES = 1 << 27, 1 << 29


def with_reduce_variants(cands):
    """Each split-K candidate of a CTA-pair 256-wide chain also with the two alternative
    reduction paths."""
    out = []
    for kw in cands:
        out.append(kw)
        split = kw.get("prod_splits", 1) > 1 or kw.get("cons_splits", 1) > 1 or \
            kw.get("cons_tail", (0, 1))[0] > 0
        if split and kw.get("cta_group") == 2 and kw.get("tile_n") == 256 and \
                kw.get("cluster_pairs", 1) == 1 and not kw.get("swap_ab"):
            for fl in (REDUCE_TC, REDUCE_ALL_PLANES):
                out.append(dict(kw, extra_flags=kw.get("extra_flags", 0) | fl))
    return out


def describe(kw) -> dict:
    co = kw.get("cons_order", RowMajor())
    swap = kw.get("swap_ab", False)
    tile = f"128x{kw['tile_n']}" if not swap else f"{kw['tile_n']}x128 (swapped)"
    if not swap:
        m = 128 * kw["cta_group"]
        pw = kw.get("prod_tile_n") or kw["tile_n"]
        cw = kw.get("cons_tile_n") or kw["tile_n"]
        tile = f"{m}x{pw}" if pw == cw else f"{m}x{pw}/{m}x{cw}"
    d = {"mode": kw["mode"], "policy": type(kw["policy"]).__name__, "tile": tile,
         "cta_group": kw["cta_group"], "swap_ab": swap,
         "splits": [kw.get("prod_splits", 1), kw.get("cons_splits", 1)],
         "consumer_order": type(co).__name__ + (f"({co.band})" if hasattr(co, "band") else "")}
    if kw.get("cons_tail", (0, 1))[0]:
        d["consumer_tail"] = list(kw["cons_tail"])  # (tiles, split-K slices) of the last wave
    if kw.get("cluster_pairs", 1) == 2:
        d["cluster_pairs"] = 2  # the 256 x 512 tile on two multicast-sharing CTA pairs
    fl = kw.get("extra_flags", 0)
    if fl & (REDUCE_TC | REDUCE_ALL_PLANES):
        d["reduce"] = "tensor-core" if fl & REDUCE_TC else "all-planes"
    return d


def pick_mlp(x, w1, w2, mode="fused", tie=0.015):
    """Time every candidate; return (best kwargs for MlpChain, [(desc, us), ...]).

    Large batch: a configuration without GeMM1 split-K slices within `tie` (timing noise)
    of the fastest is preferred — the slices' second wave re-streams the weights and the
    partial planes add traffic (ncu: 626 vs 348-359 MB per B=1024 launch,
    profiles/r01k_traffic.txt), which costs power under the cap for no measured gain."""
    table = []
    best, best_us = None, float("inf")
    timed = []
    with torch.cuda.device(x.device):
        units, qd_units = chain_units(), chain_units(cluster_pairs=2)
    for kw in with_reduce_variants(candidates(x.shape[0], mode, n2=w2.shape[0], units=units,
                                              qd_units=qd_units)):
        ch = MlpChain(x, w1, w2, **kw)
        us = _time(ch)
        _check_watchdog(ch, kw)
        table.append({**describe(kw), "us": us})
        timed.append((us, kw))
        if us < best_us:
            best, best_us = kw, us
    # Candidates within a few percent of each other are separated by box noise (the power
    # cap moves the SM clock between measurements): re-time the fastest four round-robin,
    # three rounds of 20 chains, and keep the best median.
    top = sorted(timed, key=lambda t: t[0])[:4]
    # the fastest unsplit-GeMM1 candidate joins the re-timing: the preference below must
    # compare re-timed medians, not one first-pass sample
    lean0 = [(us, kw) for us, kw in sorted(timed, key=lambda t: t[0])
             if kw.get("prod_splits", 1) == 1 and not kw.get("swap_ab", False)]
    if x.shape[0] >= 512 and lean0 and all(kw is not lean0[0][1] for _, kw in top):
        top.append(lean0[0])
    retimed = set()
    if len(top) > 1:
        chains = [(kw, MlpChain(x, w1, w2, **kw)) for _, kw in top]
        runs = {id(kw): [] for kw, _ in chains}
        for _ in range(3):
            for kw, ch in chains:
                runs[id(kw)].append(_time(ch, iters=20, warm=3))
        for kw, ch in chains:
            _check_watchdog(ch, kw)
        scored = [(statistics.median(runs[id(kw)]), i, kw) for i, (kw, _) in enumerate(chains)]
        best_us, _, best = min(scored, key=lambda t: (t[0], t[1]))
        timed = [(statistics.median(runs[id(kw)]) if id(kw) in runs else us, kw)
                 for us, kw in timed]
        retimed = set(runs)
    if x.shape[0] >= 512 and best is not None and best.get("prod_splits", 1) > 1:
        lean = [(us, kw) for us, kw in timed
                if kw.get("prod_splits", 1) == 1 and not kw.get("swap_ab", False)
                and id(kw) in retimed and us <= best_us * (1 + tie)]
        if lean:
            best = min(lean, key=lambda t: t[0])[1]
    return best, table


def pick_between(x, w1, w2, plans, rounds=3, iters=20):
    """The plan (MlpChain kwargs) with the lowest median over `rounds` round-robin timings
    of `iters` chains each (ties: the first listed)."""
    chains = [MlpChain(x, w1, w2, **kw) for kw in plans]
    runs = [[] for _ in plans]
    for _ in range(rounds):
        for i, ch in enumerate(chains):
            runs[i].append(_time(ch, iters=iters, warm=3))
    for kw, ch in zip(plans, chains):
        _check_watchdog(ch, kw)
    med = [statistics.median(r) for r in runs]
    return plans[min(range(len(plans)), key=lambda i: (med[i], i))]


def sweep_mlp(batches=(1, 64, 256, 512, 1024, 2048), hidden=12288, ffn=6144, device=None):
    """GPT-3 MLP shard latency per batch: best fused, best stream-synced, cuBLAS."""
    torch.manual_seed(7)
    w1 = (torch.randn(ffn, hidden, device=device) / hidden ** 0.5).half()
    w2 = (torch.randn(hidden, ffn, device=device) / ffn ** 0.5).half()
    rows = []
    for b in batches:
        x = torch.randn(b, hidden, device=device).half()
        fk, _ = pick_mlp(x, w1, w2, "fused")
        sk, _ = pick_mlp(x, w1, w2, "stream")
        fu = _time(MlpChain(x, w1, w2, **fk), iters=20)
        su = _time(MlpChain(x, w1, w2, **sk), iters=20)
        cu = _time(lambda: torch.nn.functional.gelu(x @ w1.t(), approximate="tanh") @ w2.t(), iters=20)
        flops = 2 * b * hidden * ffn * 2
        rows.append({"batch": b, "fused_us": fu, "stream_us": su, "cublas_us": cu,
                     "speedup_vs_stream": su / fu, "speedup_vs_cublas": cu / fu,
                     "fused_tflops": flops / fu / 1e6, "fused": describe(fk),
                     "stream": describe(sk)})
    return rows


def _torch_attention(x, wqkv, w2, heads):
    m = x.shape[0]
    qkv = x @ wqkv.t()
    q, k, v = qkv.view(m, 3, heads, 128).unbind(1)
    dot = (torch.softmax((q * v).float(), dim=-1) * k.float()).to(x.dtype).reshape(m, -1)
    return dot @ w2.t()


def sweep_attention(seqs=(512, 1024, 2048), hidden=12288, heads=12, device=None):
    """GPT-3 attention block (TP=8 shard): QKV -> fused dot -> out, fused vs stream vs a
    torch/cuBLAS implementation of the same math."""
    from .chains import AttentionChain
    torch.manual_seed(8)
    wqkv = (torch.randn(3 * heads * 128, hidden, device=device) / hidden ** 0.5).half()
    w2 = (torch.randn(hidden, heads * 128, device=device) / (heads * 128) ** 0.5).half()
    rows = []
    for s in seqs:
        x = torch.randn(s, hidden, device=device).half()
        best = {}
        for mode in ("fused", "stream"):
            timed = []
            for cg, z, ow in itertools.product((1, 2), (1, 2, 4), (0, 512)):
                if ow and cg == 1:
                    continue  # double-width output tiles are CTA-pair tiles
                for pol in ([RowSync(), TileSync()] if mode == "fused" else [TileSync()]):
                    kw = dict(second_policy=pol, mode=mode, cta_group=cg, qkv_splits=z,
                              out_tile_n=ow)
                    ch = AttentionChain(x, wqkv, w2, **kw)
                    timed.append((_time(ch, iters=20), kw))
            # the fastest three re-timed round robin (3 x 20 chains), best median kept
            top = sorted(timed, key=lambda t: t[0])[:3]
            chains = [AttentionChain(x, wqkv, w2, **kw) for _, kw in top]
            runs = [[_time(ch, iters=20, warm=3) for ch in chains] for _ in range(3)]
            med = [statistics.median(r[i] for r in runs) for i in range(len(chains))]
            i = min(range(len(chains)), key=lambda j: med[j])
            kw = top[i][1]
            best[mode] = (med[i], {"cta_group": kw["cta_group"],
                                   "policy": type(kw["second_policy"]).__name__,
                                   "qkv_splits": kw["qkv_splits"],
                                   "out_tile_n": kw["out_tile_n"] or 256})
        cu = _time(lambda: _torch_attention(x, wqkv, w2, heads), iters=20)
        flops = 2 * s * hidden * 3 * heads * 128 + 2 * s * heads * 128 * hidden
        rows.append({"seq": s, "fused_us": best["fused"][0], "stream_us": best["stream"][0],
                     "torch_us": cu, "speedup_vs_stream": best["stream"][0] / best["fused"][0],
                     "fused_tflops": flops / best["fused"][0] / 1e6,
                     "fused": best["fused"][1], "stream": best["stream"][1]})
    return rows


def wave_table(m: int, n1: int, n2: int, tile_m: int, tile_n: int, sms: int = 148):
    """Stream vs fused whole-wave counts for the two GeMMs."""
    units = sms // (tile_m // 128)
    g = GpuConfig(units)
    t1 = -(-m // tile_m) * (n1 // tile_n)
    t2 = -(-m // tile_m) * (n2 // tile_n)
    stream = waves(t1, g, 1).ceil + waves(t2, g, 1).ceil
    fine = waves(t1 + t2, g, 1).ceil
    return {"tiles": (t1, t2), "stream_waves": stream, "fine_waves": fine,
            "bound": stream / fine}


RESNET38_LAYERS = ((56, 64), (28, 128), (14, 256), (7, 512))
# VGG-19's 3x3 "same" conv pairs with equal in/out channels, one per resolution stage
# (Simonyan & Zisserman 2015, config E: 2x64 @224, 2x128 @112, 4x256 @56, 4x512 @28,
# 4x512 @14); BASELINE.json configs[4] names VGG-19 beside ResNet-38 (no reference text)
VGG19_LAYERS = ((224, 64), (112, 128), (56, 256), (28, 512), (14, 512))


def conv_candidates(c: int, mode: str, m: int = 1 << 30):
    """Tile configurations for a conv pair with `c` channels and `m` output pixels (output
    channels = tile columns: a tile no wider than the layer). Few pixels (deep layers at
    small batch) leave most SMs idle, so those also try split-K (reference z slices)."""
    out = []
    for cg, tn in ((1, 64), (1, 128), (2, 128), (1, 256), (2, 256)):
        if tn > c:
            continue
        tiles = -(-m // (128 * cg)) * (c // tn)
        for z in (1, 2, 4, 8):
            if z > 1 and (tiles * z > 2 * 148 or (9 * c // 64) % z):
                continue
            out.append(dict(mode=mode, tile_n=tn, cta_group=cg, prod_splits=z, cons_splits=z))
    if c == 64:
        # 64-channel layers: each tile's input rows + halo staged once, taps as shifted views
        # (TS_FLAG_CONV_HALO; 1.8-1.9x the im2col-per-tap tiles at B >= 32, r02y)
        out.append(dict(mode=mode, tile_n=64, cta_group=1, prod_splits=1, cons_splits=1,
                        halo=True))
    return out


def sweep_conv(batches=(1, 8, 32, 128, 256), layers=RESNET38_LAYERS, device=None,
               dtype=torch.float16):
    """ResNet-38 conv pairs (3x3, same padding): best fused (Conv2DTileSync(9)) vs best
    stream-synchronized launch of the same kernels vs cuDNN (channels-last conv2d)."""
    from .chains import ConvChain
    torch.manual_seed(11)
    rows = []
    for hw, c in layers:
        w1 = (torch.randn(c, 3, 3, c, device=device) / (9 * c) ** 0.5).to(dtype)
        w2 = (torch.randn(c, 3, 3, c, device=device) / (9 * c) ** 0.5).to(dtype)
        wt1 = w1.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
        wt2 = w2.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
        for b in batches:
            x = torch.randn(b, hw, hw, c, device=device).to(dtype)
            best = {}
            for mode in ("fused", "stream"):
                for kw in conv_candidates(c, mode, b * hw * hw):
                    ch = ConvChain(x, w1, w2, **kw)
                    us = _time(ch, iters=20)
                    _check_watchdog(ch, kw)
                    if mode not in best or us < best[mode][0]:
                        best[mode] = (us, kw)
            xt = x.permute(0, 3, 1, 2)  # NCHW view of NHWC memory = channels_last

            def cudnn():
                h = torch.relu(torch.nn.functional.conv2d(xt, wt1, padding=1))
                return torch.nn.functional.conv2d(h, wt2, padding=1)
            cu = _time(cudnn, iters=20)
            flops = 2 * 2 * b * hw * hw * c * 9 * c
            fu, su = best["fused"][0], best["stream"][0]
            rows.append({"layer": f"{hw}x{hw}x{c}", "batch": b, "fused_us": fu, "stream_us": su,
                         "cudnn_us": cu, "speedup_vs_stream": su / fu, "speedup_vs_cudnn": cu / fu,
                         "fused_tflops": flops / fu / 1e6,
                         "fused": {k: v for k, v in best["fused"][1].items() if k != "mode"},
                         "stream": {k: v for k, v in best["stream"][1].items() if k != "mode"}})
    return rows


def sweep_swiglu(batches=(256, 1024, 2048), tps=(8, 1), hidden=4096, ffn=14336, device=None):
    """LLaMA-style 8B SwiGLU MLP (BASELINE.json configs[3]), bf16, the per-rank chain of a
    TP=tp shard: H = SiLU(X Wg^T) * (X Wu^T) (gate/up interleaved per tile), Y = H Wd^T.
    Best fused vs best stream-synchronized configuration vs torch/cuBLAS."""
    from .chains import SwigluChain, interleave_gate_up
    torch.manual_seed(9)
    rows = []
    for tp in tps:
        f = ffn // tp
        wg = (torch.randn(f, hidden, device=device) / hidden ** 0.5).bfloat16()
        wu = (torch.randn(f, hidden, device=device) / hidden ** 0.5).bfloat16()
        wd = (torch.randn(hidden, f, device=device) / f ** 0.5).bfloat16()
        packed = {w: interleave_gate_up(wg, wu, w) for w in (256, 512)}
        for b in batches:
            x = torch.randn(b, hidden, device=device).bfloat16()
            best = {}
            for mode in ("fused", "stream"):
                pols = [RowSync(), TileSync()] if mode == "fused" else [RowSync()]
                for pw, cw, pol in itertools.product((256, 512), (0, 512), pols):
                    if (f // 2) % (pw // 2) or f % pw // 2:
                        continue
                    try:
                        ch = SwigluChain(x, packed[pw], wd, policy=pol, mode=mode, tile_n=256,
                                         cta_group=2, prod_tile_n=pw if pw == 512 else 0,
                                         cons_tile_n=cw)
                    except Exception:  # shapes a width does not divide
                        continue
                    us = _time(ch, iters=20)
                    _check_watchdog(ch, {"tile": (pw, cw), "policy": pol, "mode": mode})
                    if us < best.get(mode, (float("inf"),))[0]:
                        best[mode] = (us, {"policy": type(pol).__name__,
                                           "tile": f"256x{pw}/256x{cw or 256}"})
                # few row tiles (B <= 1024): split-K slices to fill the CTA pairs, reduced on
                # the tensor cores (the only split path under SwiGLU)
                for (z1, z2), pol in itertools.product(
                        ((2, 1), (4, 1), (4, 2), (8, 2)) if b <= 1024 else (), pols):
                    pw = 512
                    try:
                        ch = SwigluChain(x, packed[pw], wd, policy=pol, mode=mode, tile_n=256,
                                         cta_group=2, prod_tile_n=pw, cons_tile_n=512,
                                         prod_splits=z1, cons_splits=z2,
                                         extra_flags=REDUCE_TC)
                    except Exception:  # K not divisible into the slices
                        continue
                    us = _time(ch, iters=20)
                    _check_watchdog(ch, {"splits": (z1, z2), "policy": pol, "mode": mode})
                    if us < best.get(mode, (float("inf"),))[0]:
                        best[mode] = (us, {"policy": type(pol).__name__,
                                           "tile": "256x512/256x512", "splits": [z1, z2],
                                           "reduce": "tensor-core"})

            def torch_mlp():
                return (torch.nn.functional.silu(x @ wg.t()) * (x @ wu.t())) @ wd.t()
            cu = _time(torch_mlp, iters=20)
            flops = 2 * b * hidden * f * 3
            fu, su = best["fused"][0], best["stream"][0]
            rows.append({"tp": tp, "batch": b, "ffn_shard": f, "fused_us": fu, "stream_us": su,
                         "cublas_us": cu, "speedup_vs_stream": su / fu,
                         "speedup_vs_cublas": cu / fu, "fused_tflops": flops / fu / 1e6,
                         "fused": best["fused"][1], "stream": best["stream"][1]})
    return rows
