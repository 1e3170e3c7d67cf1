"""Reference fixtures for the BENCHMARKED chain configurations (B200 grids).

Run in the build container, where /root/reference exists (it does not on the GPU box):

    python tests/golden/make_bench_golden.py

For every chain configuration bench.py / planner.py can pick at the BASELINE.json sizes —
the GPT-3 MLP shard (H=12288, FFN=6144) at B in {1, 64, 256, 512, 1024, 2048} over every
planner candidate (tile shape, CTA group, split-K slices), the GPT-3 attention block (12
heads, S in {512, 1024, 2048}), the LLaMA-8B SwiGLU TP shards and the ResNet-38 conv pairs —
it builds the reference Scenario with that configuration's tile grids
(/root/reference/pkg/src/tilesync_sim/engine.py:71-131, workloads.py:55-69,112-153,180-200),
runs the reference simulator (engine.py:644-646) and records its final semaphores and
post / wait_end counts. tests/test_gpu_bench_parity.py matches the device's semaphores
for the same configurations against these records bit for bit.

Consumer tile orders are not part of the key: final semaphores and post/wait counts do
not depend on the consumer's claim order, and the BandedColumnMajor extension order has
no reference counterpart (the reference simulates RowMajor for it).
"""

from __future__ import annotations

import itertools
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
ROOT = OUT.parents[1]


def mlp_grids(kw, m, n1=6144, n2=12288):
    """(producer grid, consumer grid, consumer k_steps, producer k_steps) of an MlpChain
    built with the planner kwargs `kw` (mirrors CuStage.grid / CuSync.scenario: a stage
    without an incoming dependency has k / out_tile_cols k-steps)."""
    swap = kw.get("swap_ab", False)
    tn, cg = kw["tile_n"], kw.get("cta_group", 2)
    tile_m = tn if swap else 128 * cg
    w1 = 128 if swap else (kw.get("prod_tile_n") or tn)
    w2 = 128 if swap else (kw.get("cons_tile_n") or tn)
    gx = -(-m // tile_m)
    return ((gx, n1 // w1, kw.get("prod_splits", 1)), (gx, n2 // w2, kw.get("cons_splits", 1)),
            n1 // w1, 12288 // w1)


def key(stages, deps):
    """Order-free identity of a scenario: stage grids and k-steps, dependency policies."""
    return json.dumps([[list(s["grid"]), s["k_steps"]] for s in stages]
                      + [[d["producer"], d["consumer"], list(d["policy"])] for d in deps])


def main() -> None:
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import tilesync_sim as r  # noqa: PLC0415  (the reference, read-only)

    from paper_2305_13450_b200 import planner  # candidate enumeration (no GPU needed)

    pol = {"tile": r.TileSync(), "row": r.RowSync()}
    recs, seen = [], set()

    def add(name, stages, deps):
        """stages: [(id, grid, k_steps, order)], deps: [(prod, cons, operand, (kind, p))]."""
        sd = [{"id": i, "grid": list(g), "k_steps": k} for i, g, k, _ in stages]
        dd = [{"producer": p, "consumer": c, "operand": o, "policy": list(pk)}
              for p, c, o, pk in deps]
        kk = key(sd, dd)
        if kk in seen:
            return
        seen.add(kk)
        mk = {"tile": lambda p: r.TileSync(), "row": lambda p: r.RowSync(),
              "strided": lambda p: r.StridedSync(p), "conv2d": lambda p: r.Conv2DTileSync(p)}
        sc = r.Scenario(
            gpu=r.GpuConfig(148),
            stages=tuple(r.Stage(i, r.Dim3(*g), k_steps=k, order=o,
                                 operands=("qkv",) if i == "dot" else ("a", "b"))
                         for i, g, k, o in stages),
            deps=tuple(r.Dependency(p, c, o, mk[pk[0]](pk[1])) for p, c, o, pk in deps))
        trace, metrics = r.simulate(sc)
        assert not metrics.deadlock, name
        recs.append({"name": name, "key": kk, "stages": sd, "deps": dd,
                     "final_semaphores": {k: list(v) for k, v in trace.final_semaphores.items()},
                     "posts": sum(1 for e in trace.events if e.kind == "post"),
                     "wait_ends": sum(1 for e in trace.events if e.kind == "wait_end")})

    rm = r.RowMajor()
    # GPT-3 MLP shard: every fused candidate the planner times (planner.candidates)
    for b in (1, 64, 256, 512, 1024, 2048):
        for kw in planner.candidates(b, "fused", n2=12288, units=74):
            g1, g2, ks, ks1 = mlp_grids(kw, b)
            pk = ("row", 0) if type(kw["policy"]).__name__ == "RowSync" else ("tile", 0)
            add(f"gpt3_mlp_b{b}", [("gemm1", g1, ks1, rm), ("gemm2", g2, ks, rm)],
                [("gemm1", "gemm2", "a", pk)])
    # GPT-3 attention (TP=8: 12 heads of 128; QKV 4608 columns, out 12288): the sweep's
    # configurations (cta_group, qkv z-slices, out tile width; Row/Tile second policy)
    for s, cg, z, ow in itertools.product((512, 1024, 2048), (1, 2), (1, 2, 4), (0, 512)):
        if ow and cg == 1:
            continue
        tm, tn = 128 * cg, 256
        gx = -(-s // tm)
        stride = 4608 // (3 * tn)
        g_qkv, g_dot = (gx, 4608 // tn, z), (gx, 1536 // tn, 1)
        g_out = (gx, 12288 // (ow or tn), 1)
        for second in ("row", "tile"):
            add(f"gpt3_attn_s{s}",
                [("qkv", g_qkv, 12288 // tn, r.StridedRowMajor(stride)), ("dot", g_dot, 1, rm),
                 ("out", g_out, g_dot[1], rm)],
                [("qkv", "dot", "qkv", ("strided", stride)), ("dot", "out", "a", (second, 0))])
    # LLaMA-8B SwiGLU TP shards (H=4096, F=14336/tp): gate|up accumulator tiles of 256 or
    # 512 columns write 128 / 256 output columns
    for tp, b, pw, cw in itertools.product((8, 1), (256, 1024, 2048), (256, 512), (0, 512)):
        f = 14336 // tp
        if (2 * f) % pw:
            continue
        gx = -(-b // 256)
        g1, g2 = (gx, 2 * f // pw, 1), (gx, 4096 // (cw or 256), 1)
        for p in ("row", "tile"):
            add(f"llama_swiglu_tp{tp}_b{b}", [("gate_up", g1, 4096 // (pw // 2), rm),
                                             ("down", g2, f // (pw // 2), rm)],
                [("gate_up", "down", "a", (p, 0))])
    # ResNet-38 / VGG-19 conv pairs (Conv2DTileSync(9)): the sweeps' configurations
    conv_cases = [("resnet38", L, b) for L, b in
                  itertools.product(planner.RESNET38_LAYERS, (1, 8, 32, 128, 256))]
    conv_cases += [("vgg19", L, b) for L, b in
                   itertools.product(planner.VGG19_LAYERS, (1, 8, 32))]
    for net, (hw, c), b in conv_cases:
        for kw in planner.conv_candidates(c, "fused", b * hw * hw):
            tm = 128 * kw["cta_group"]
            gx = -(-(b * hw * hw) // tm)
            if kw.get("halo"):  # halo-staged tiles: per-image re-tiling
                from paper_2305_13450_b200.cusync import halo_tiles_per_image
                gx = b * halo_tiles_per_image(hw, hw, b, 148)  # B200: 148 SMs
            z = kw["prod_splits"]
            g = (gx, c // kw["tile_n"], z)
            add(f"{net}_conv_{hw}x{c}_b{b}", [("conv1", g, 9 * c // kw["tile_n"], rm),
                                                ("conv2", g, 9 * (c // kw["tile_n"]), rm)],
                [("conv1", "conv2", "a", ("conv2d", 9))])
    (OUT / "bench_scenarios.json").write_text(json.dumps(recs, separators=(",", ":")))
    print(f"wrote bench_scenarios.json: {len(recs)} scenarios")


if __name__ == "__main__":
    main()
