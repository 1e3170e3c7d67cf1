"""The host engine layer (Stage / Dependency / Scenario, the wait-kernel gate "+W", the
"+R" k-step formula, structural validation) against fixtures generated from the
reference itself (tests/golden/make_golden.py -> engine_layer.json; engine.py:134-217).

`avoid_wait_kernel` runs through the C ABI (the same function the launcher uses)."""

import json

import pytest

import paper_2305_13450_b200 as ts
from conftest import GOLDEN
from paper_2305_13450_b200 import engine as E

ENG = json.loads((GOLDEN / "engine_layer.json").read_text())
POL = {"tile": lambda p: ts.TileSync(), "row": lambda p: ts.RowSync(),
       "strided": lambda p: ts.StridedSync(p), "conv2d": lambda p: ts.Conv2DTileSync(p)}


def order(o):
    kind, s = o
    return ts.RowMajor() if kind == "row_major" else ts.StridedRowMajor(s)


def stages(rec):
    return tuple(E.Stage(id=s["id"], grid=ts.Dim3(*s["grid"]), k_steps=s["k_steps"],
                         order=order(s["order"]), occupancy=s.get("occupancy", 1),
                         operands=tuple(s.get("operands", ("a", "b"))))
                 for s in rec["stages"])


def deps(rec):
    return tuple(E.Dependency(d["producer"], d["consumer"], d["operand"],
                              POL[d["policy"][0]](d["policy"][1])) for d in rec["deps"])


@pytest.mark.parametrize("rec", ENG["gates"], ids=lambda r: f"{r['name']}-{r['wait_kernel']}")
def test_wait_kernel_gate_matches_reference(rec):
    sc = E.Scenario(gpu=ts.GpuConfig(rec["num_sms"]), stages=stages(rec), deps=deps(rec),
                    mode=E.Mode(rec["mode"]), options=E.SimOptions(wait_kernel=rec["wait_kernel"]))
    for st in sc.stages:
        assert list(E.gated_producers(sc, st)) == rec["gated"][st.id]
    for d, avoid in zip(sc.deps, rec["avoid"]):
        assert E.avoid_wait_kernel(sc.stage_by_id(d.producer), sc.stage_by_id(d.consumer),
                                   sc.gpu) == avoid


@pytest.mark.parametrize("rec", ENG["kstep"], ids=lambda r: f"{r['args']}-{r['reorder']}")
def test_kstep_duration_matches_reference(rec):
    assert E.kstep_duration(*rec["args"], reorder=rec["reorder"]) == rec["value"]


@pytest.mark.parametrize("rec", ENG["errors"], ids=lambda r: r["name"])
def test_scenario_validation_matches_reference(rec):
    st, dp = stages(rec), deps(rec) if rec["deps"] else ()
    if rec["error"] is None:
        E.Scenario(gpu=ts.GpuConfig(4), stages=st, deps=dp)
        return
    kind, msg = rec["error"]
    with pytest.raises(getattr(ts, kind)) as ei:
        E.Scenario(gpu=ts.GpuConfig(4), stages=st, deps=dp)
    assert str(ei.value) == msg
