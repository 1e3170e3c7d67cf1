"""Generate the golden fixtures from the reference package itself.

Run in the build container, where /root/reference exists (it does not on the GPU box):

    python tests/golden/make_golden.py

It imports the reference simulator (/root/reference/pkg/src/tilesync_sim) read-only and
writes small JSON fixtures next to this script:

* ``policy_tables.json`` — sem_count / post_target / consumer_wait / wait_steps /
  order_tile over exhaustive small grids and every policy, plus the reference tests'
  explicit golden values (test_policies.py:23-194) and expected exceptions.
* ``scenarios.json`` — for the paper's chains at B200 grids (GpuConfig(148)) and for the
  reference's own presets and random scenarios: final semaphores, post/wait counts and
  a digest of the brute-force dependency DAG (oracle.py:45-76).
* ``traces.json`` — reference traces (fig2, toy attention) with the violations
  validate_trace reports for clean and corrupted copies (test_oracle.py:58-107).
"""

from __future__ import annotations

import dataclasses
import hashlib
import itertools
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF))
    import tilesync_sim as r  # noqa: PLC0415  (the reference, read-only)

    pol = {"tile": lambda p: r.TileSync(), "row": lambda p: r.RowSync(),
           "strided": lambda p: r.StridedSync(p), "conv2d": lambda p: r.Conv2DTileSync(p)}

    # ---------------- policy tables ----------------
    tables = []
    for gx, gy, gz in itertools.product((1, 2, 3), (1, 2, 3, 4, 6), (1, 2)):
        grid = r.Dim3(gx, gy, gz)
        for kind, params in (("tile", [0]), ("row", [0]), ("strided", [1, 2, 3, 4]),
                             ("conv2d", [1, 2, 3])):
            for p in params:
                policy = pol[kind](p)
                case = {"policy": [kind, p], "grid": [gx, gy, gz]}
                try:
                    case["sem_count"] = r.sem_count(policy, grid)
                except r.ConfigError:
                    case["sem_count"] = "ConfigError"
                    tables.append(case)
                    continue
                case["post_target"] = [
                    [x, y, z, r.post_target(policy, r.TileCoord(x, y, z), grid)]
                    for x in range(gx) for y in range(gy) for z in range(gz)]
                k_steps = gy * (p if kind == "conv2d" else 1)
                waits = []
                for x, y in itertools.product(range(gx), range(gy)):
                    for k in range(k_steps):
                        w = r.consumer_wait(policy, r.TileCoord(x, y, 0), k, grid, gz)
                        waits.append([x, y, k, None if w is None else [w.sem_index, w.expected]])
                case["consumer_wait"] = waits
                case["wait_steps"] = {str(n): list(r.wait_steps(policy, n)) for n in range(0, 7)}
                tables.append(case)
    orders = []
    for gx, gy, gz in itertools.product((1, 2, 3), (1, 2, 4, 6, 12), (1, 2)):
        grid = r.Dim3(gx, gy, gz)
        for kind, s in [("row_major", 1)] + [("strided_row_major", s) for s in (1, 2, 3, 4)]:
            order = r.RowMajor() if kind == "row_major" else r.StridedRowMajor(s)
            try:
                tiles = [list(dataclasses.astuple(r.order_tile(order, grid, n)))
                         for n in range(grid.total())]
            except r.ConfigError:
                tiles = "ConfigError"
            orders.append({"order": [kind, s], "grid": [gx, gy, gz], "tiles": tiles})
    explicit = {
        # test_policies.py:23-92, 152-167
        "sem_count": [[["tile", 0], [3, 2, 1], 6], [["row", 0], [3, 2, 1], 3],
                      [["strided", 2], [1, 6, 1], 2], [["strided", 4], [1, 6, 1], "ConfigError"]],
        "post_target": [[["tile", 0], [1, 1, 0], [3, 2, 1], 3], [["row", 0], [2, 0, 0], [3, 2, 1], 2],
                        [["strided", 2], [0, 4, 0], [1, 6, 1], 0]],
        "consumer_wait": [[["row", 0], [1, 0, 0], 0, [3, 2, 1], 1, [1, 2]],
                          [["row", 0], [1, 0, 0], 1, [3, 2, 1], 1, None],
                          [["tile", 0], [0, 3, 0], 1, [1, 6, 1], 1, [1, 1]],
                          [["conv2d", 9], [0, 5, 0], 10, [1, 6, 1], 1, None],
                          [["strided", 2], [0, 1, 0], 0, [1, 6, 1], 1, [1, 3]],
                          [["row", 0], [0, 0, 0], 0, [1, 96, 2], 2, [0, 192]]],
        "order_tile": [[["row_major", 1], [3, 2, 1], 3, [1, 1, 0]]],
    }
    # recompute the explicit expectations with the reference so the fixture is its output
    for e in explicit["consumer_wait"]:
        (kind, p), t, k, g, z, _ = e
        w = r.consumer_wait(pol[kind](p), r.TileCoord(*t), k, r.Dim3(*g), z)
        e[5] = None if w is None else [w.sem_index, w.expected]
    (OUT / "policy_tables.json").write_text(json.dumps(
        {"tables": tables, "orders": orders, "explicit": explicit}, separators=(",", ":")))

    # ---------------- scenarios ----------------
    def stage_dict(s):
        order = ["row_major", 1] if isinstance(s.order, r.RowMajor) else \
            ["strided_row_major", s.order.stride]
        return {"id": s.id, "grid": [s.grid.x, s.grid.y, s.grid.z], "k_steps": s.k_steps,
                "order": order, "occupancy": s.occupancy, "operands": list(s.operands)}

    def dep_dict(d):
        p = d.policy
        kind = {r.TileSync: "tile", r.RowSync: "row", r.StridedSync: "strided",
                r.Conv2DTileSync: "conv2d"}[type(p)]
        param = getattr(p, "stride", getattr(p, "kk", 0))
        return {"producer": d.producer, "consumer": d.consumer, "operand": d.operand,
                "policy": [kind, param]}

    def digest(dag):
        rows = sorted([list(k), sorted(list(t) for t in v[0]), v[1]]
                      for k, v in dag.requires.items())
        return hashlib.sha256(json.dumps(rows).encode()).hexdigest()

    scen = []

    def add(name, sc, run=True):
        dag = r.build_dep_dag(sc)
        rec = {"name": name, "mode": sc.mode.value, "num_sms": sc.gpu.num_sms,
               "stages": [stage_dict(s) for s in sc.stages],
               "deps": [dep_dict(d) for d in sc.deps],
               "dag_digest": digest(dag), "dag_entries": len(dag.requires)}
        if run:
            trace, metrics = r.simulate(sc)
            rec["final_semaphores"] = {k: list(v) for k, v in trace.final_semaphores.items()}
            rec["posts"] = sum(1 for e in trace.events if e.kind == "post")
            rec["wait_ends"] = sum(1 for e in trace.events if e.kind == "wait_end")
            rec["deadlock"] = metrics.deadlock
            rec["makespan"] = metrics.makespan
            rec["violations"] = len(r.validate_trace(trace, dag))
        scen.append(rec)

    # The paper's chains at B200 grids: 256x256 CTA-pair tiles (cta_group::2) and
    # 128x256 single-CTA tiles, GPT-3 MLP TP=8 shard.
    for tile_m in (128, 256):
        for b in (1, 64, 256, 512, 1024, 2048):
            gx = -(-b // tile_m)
            for pname in ("row", "tile"):
                params = r.MlpParams(f"b200-{b}", r.Dim3(gx, 6144 // 256, 1),
                                     r.Dim3(gx, 12288 // 256, 1), 1, num_sms=148 // (tile_m // 128))
                sc = r.mlp_scenario(params, pol[pname](0))
                add(f"gpt3_mlp_tm{tile_m}_b{b}_{pname}", sc, run=(b <= 1024))
    # SURVEY §7.2 config 1 (M=256, K=N=1024), 128x128 and 128x256 tiles.
    add("cfg1_row_128x128", r.mlp_scenario(
        r.MlpParams("cfg1", r.Dim3(2, 8, 1), r.Dim3(2, 8, 1), 1, num_sms=148), r.RowSync()))
    add("cfg1_row_128x256", r.mlp_scenario(
        r.MlpParams("cfg1", r.Dim3(2, 4, 1), r.Dim3(2, 4, 1), 1, num_sms=148), r.RowSync()))
    for name in ("fig2", "mlp:1-64", "mlp:256", "mlp:1024", "attn:toy", "attn:1024",
                 "conv128:1", "conv128:8"):
        info = r.PRESETS[name]
        for p in info.policies:
            for mode in (r.Mode.FINE, r.Mode.STREAM):
                add(f"{name}/{p}/{mode.value}", r.build_preset(name, p, mode))
    for seed in range(40):
        add(f"random:{seed}", r.random_scenario(seed))
    (OUT / "scenarios.json").write_text(json.dumps(scen, indent=0))

    # ---------------- traces ----------------
    traces = []
    for name, sc in (("fig2_fine_row", r.fig2_scenario(r.RowSync())),
                     ("fig2_fine_tile", r.fig2_scenario(r.TileSync())),
                     ("fig2_stream", r.fig2_scenario(r.RowSync(), r.Mode.STREAM)),
                     ("attn_toy_fine", r.build_preset("attn:toy", "tile"))):
        trace, _ = r.simulate(sc)
        dag = r.build_dep_dag(sc)
        evs = [json.loads(e.to_json()) for e in trace.events]
        cases = [{"what": "clean", "events": evs,
                  "violations": [v.kind for v in r.validate_trace(trace, dag)]}]
        if sc.mode is r.Mode.FINE:
            posts = [i for i, e in enumerate(trace.events) if e.kind == "post"]
            cut = trace.events[:posts[0]] + trace.events[posts[0] + 1:]
            cases.append({"what": "first_post_deleted",
                          "events": [json.loads(e.to_json()) for e in cut],
                          "violations": sorted(v.kind for v in r.validate_trace(cut, dag, sc.mode))})
        traces.append({"name": name, "scenario": [stage_dict(s) for s in sc.stages],
                       "deps": [dep_dict(d) for d in sc.deps], "mode": sc.mode.value,
                       "cases": cases})
    (OUT / "traces.json").write_text(json.dumps(traces, separators=(",", ":")))

    # ---------------- engine layer (engine.py:134-217) ----------------
    eng = {"gates": [], "kstep": [], "errors": []}
    gate_scen = [("fig2", lambda o: r.fig2_scenario(r.RowSync(), r.Mode.FINE, o))]
    for name in ("mlp:1-64", "mlp:1024", "attn:toy", "conv128:1"):
        gate_scen.append((name, lambda o, n=name: dataclasses.replace(
            r.build_preset(n, r.PRESETS[n].policies[0]), options=o)))
    for seed in range(20):
        gate_scen.append((f"random:{seed}", lambda o, sd=seed: dataclasses.replace(
            r.random_scenario(sd), options=o)))
    for name, mk in gate_scen:
        for wk in ("on", "off", "auto"):
            sc = mk(r.SimOptions(wait_kernel=wk))
            eng["gates"].append({
                "name": name, "wait_kernel": wk, "mode": sc.mode.value,
                "num_sms": sc.gpu.num_sms,
                "stages": [stage_dict(st) | {"occupancy": st.occupancy} for st in sc.stages],
                "deps": [dep_dict(d) for d in sc.deps],
                "gated": {st.id: list(r.gated_producers(sc, st)) for st in sc.stages},
                "avoid": [r.avoid_wait_kernel(sc.stage_by_id(d.producer),
                                              sc.stage_by_id(d.consumer), sc.gpu)
                          for d in sc.deps]})
    for vals in itertools.product((0.0, 1.5, 4.0), (1.0, 2.0), (0.5, 3.0), (1.0, 2.5)):
        for reorder in (False, True):
            eng["kstep"].append({"args": list(vals), "reorder": reorder,
                                 "value": r.kstep_duration(*vals, reorder=reorder)})
    D, S = r.Dim3, r.Stage
    bad = {
        "duplicate": ((S("a", D(2, 2, 1)), S("a", D(2, 2, 1))), ()),
        "unknown": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1))), (r.Dependency("a", "c"),)),
        "cycle": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1))), (r.Dependency("b", "a"),)),
        "operand": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1))), (r.Dependency("a", "b", "q"),)),
        "rows": ((S("a", D(2, 2, 1)), S("b", D(3, 2, 1))), (r.Dependency("a", "b"),)),
        "tile_ksteps": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1), k_steps=3)),
                        (r.Dependency("a", "b", policy=r.TileSync()),)),
        "conv_kk": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1), k_steps=10)),
                    (r.Dependency("a", "b", policy=r.Conv2DTileSync(9)),)),
        "conv_cols": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1), k_steps=27)),
                      (r.Dependency("a", "b", policy=r.Conv2DTileSync(9)),)),
        "strided": ((S("a", D(2, 6, 1)), S("b", D(2, 2, 1))),
                    (r.Dependency("a", "b", policy=r.StridedSync(4)),)),
        "ok": ((S("a", D(2, 2, 1)), S("b", D(2, 2, 1), k_steps=2)),
               (r.Dependency("a", "b", policy=r.TileSync()),)),
    }
    for name, (stages, deps) in bad.items():
        try:
            r.Scenario(gpu=r.GpuConfig(4), stages=stages, deps=deps)
            err = None
        except Exception as e:  # noqa: BLE001 - recorded as the golden outcome
            err = [type(e).__name__, str(e)]
        eng["errors"].append({"name": name, "stages": [stage_dict(st) for st in stages],
                              "deps": [dep_dict(d) for d in deps], "error": err})
    (OUT / "engine_layer.json").write_text(json.dumps(eng, indent=0))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()
