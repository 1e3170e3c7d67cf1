"""Pin the CPU oracle (oracle/tilesync_oracle.py) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the reference package
(/root/reference/pkg/src/tilesync_sim) — see tests/golden/make_golden.py. An oracle
that disagrees with them is wrong, whatever the device says.
"""

import json

import pytest

from conftest import GOLDEN
from oracle import tilesync_oracle as O

TABLES = json.loads((GOLDEN / "policy_tables.json").read_text())
SCEN = json.loads((GOLDEN / "scenarios.json").read_text())
TRACES = json.loads((GOLDEN / "traces.json").read_text())


def _pol(p):
    return (p[0], p[1])


@pytest.mark.parametrize("case", TABLES["tables"], ids=lambda c: f"{c['policy']}-{c['grid']}")
def test_policy_table(case):
    policy, grid = _pol(case["policy"]), tuple(case["grid"])
    if case["sem_count"] == "ConfigError":
        with pytest.raises(O.OracleConfigError):
            O.sem_count(policy, grid)
        return
    assert O.sem_count(policy, grid) == case["sem_count"]
    for x, y, z, idx in case["post_target"]:
        assert O.post_target(policy, (x, y, z), grid) == idx
    for x, y, k, w in case["consumer_wait"]:
        got = O.consumer_wait(policy, (x, y, 0), k, grid, grid[2])
        assert (None if got is None else list(got)) == w
    for n, steps in case["wait_steps"].items():
        assert list(O.wait_steps(policy, int(n))) == steps


@pytest.mark.parametrize("case", TABLES["orders"], ids=lambda c: f"{c['order']}-{c['grid']}")
def test_order_table(case):
    order, grid = tuple(case["order"]), tuple(case["grid"])
    if case["tiles"] == "ConfigError":
        with pytest.raises(O.OracleConfigError):
            O.order_tile(order, grid, 0)
        return
    got = [list(O.order_tile(order, grid, n)) for n in range(len(case["tiles"]))]
    assert got == case["tiles"]


def test_explicit_reference_test_values():
    ex = TABLES["explicit"]
    for pol, grid, want in ex["sem_count"]:
        if want == "ConfigError":
            with pytest.raises(O.OracleConfigError):
                O.sem_count(_pol(pol), tuple(grid))
        else:
            assert O.sem_count(_pol(pol), tuple(grid)) == want
    for pol, tile, grid, want in ex["post_target"]:
        assert O.post_target(_pol(pol), tuple(tile), tuple(grid)) == want
    for pol, tile, k, grid, z, want in ex["consumer_wait"]:
        got = O.consumer_wait(_pol(pol), tuple(tile), k, tuple(grid), z)
        assert (None if got is None else list(got)) == want
    for order, grid, n, want in ex["order_tile"]:
        assert list(O.order_tile(tuple(order), tuple(grid), n)) == want


def _stages(rec):
    return [{"id": s["id"], "grid": tuple(s["grid"]), "k_steps": s["k_steps"],
             "order": tuple(s["order"])} for s in rec["stages"]]


def _deps(rec):
    return [dict(d, policy=_pol(d["policy"])) for d in rec["deps"]]


@pytest.mark.parametrize("rec", SCEN, ids=lambda r: r["name"])
def test_scenario_dag_and_final_semaphores(rec):
    stages, deps = _stages(rec), _deps(rec)
    dag = O.build_dep_dag(stages, deps)
    assert len(dag) == rec["dag_entries"]
    assert O.dag_digest(dag) == rec["dag_digest"]
    if "final_semaphores" in rec and not rec["deadlock"]:
        assert {k: list(v) for k, v in O.final_semaphores(stages, deps).items()} == \
            rec["final_semaphores"]
        by_id = {s["id"]: s for s in stages}
        assert rec["posts"] == sum(
            by_id[d["producer"]]["grid"][0] * by_id[d["producer"]]["grid"][1]
            * by_id[d["producer"]]["grid"][2] for d in deps)


@pytest.mark.parametrize("rec", TRACES, ids=lambda r: r["name"])
def test_trace_validation_matches_reference(rec):
    stages = [{"id": s["id"], "grid": tuple(s["grid"]), "k_steps": s["k_steps"],
               "order": tuple(s["order"])} for s in rec["scenario"]]
    deps = [dict(d, policy=_pol(d["policy"])) for d in rec["deps"]]
    for case in rec["cases"]:
        got = O.validate_trace(case["events"], stages, deps, fine=rec["mode"] == "fine")
        assert sorted(v[0] for v in got) == sorted(case["violations"]), case["what"]
