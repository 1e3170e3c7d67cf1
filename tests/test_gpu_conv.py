"""Device parity for the ResNet conv pair (implicit-GeMM Conv2D stages with the im2col TMA
operand) under Conv2DTileSync(9): numerics against the oracle's conv restatement
(oracle.conv_chain, itself pinned to torch's direct conv2d in float64 by
tests/test_oracle_numeric.py) and synchronization parity (device trace dependency-safe
under the reference DAG, final semaphores and wait counts exact)."""

import numpy as np
import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O

pytestmark = pytest.mark.gpu

TOL = {torch.float16: (2e-2, 1e-2), torch.bfloat16: (6e-2, 3e-2)}
DT = {torch.float16: "fp16", torch.bfloat16: "bf16"}


def make(n, h, w, c, dtype, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, h, w, c, generator=g).to(dtype)
    w1 = (torch.randn(c, 3, 3, c, generator=g) / (9 * c) ** 0.5).to(dtype)
    w2 = (torch.randn(c, 3, 3, c, generator=g) / (9 * c) ** 0.5).to(dtype)
    return x, w1, w2


def check_close(dev, ref, dtype):
    atol, rtol = TOL[dtype]
    d = dev.float().cpu().numpy()
    err = np.abs(d - ref)
    bad = err > atol + rtol * np.abs(ref)
    assert not bad.any(), f"max err {err.max():.4g}, {bad.sum()} elements out of tolerance"


CASES = [
    # n, h, w, c, tile_n, cta_group, mode[, splits]
    (1, 56, 56, 64, 64, 1, "fused"),     # ResNet-38 layer 1
    (1, 7, 7, 512, 128, 1, "fused", 4),  # layer 4 at batch 1: split-K slices
    (2, 14, 14, 256, 256, 2, "fused", 2),
    (2, 28, 28, 128, 128, 1, "fused"),   # layer 2
    (4, 14, 14, 256, 128, 2, "fused"),   # layer 3
    (8, 7, 7, 512, 256, 2, "fused"),     # layer 4
    (1, 9, 11, 128, 128, 2, "stream"),
    (3, 5, 13, 64, 64, 1, "fused"),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_conv_pair_numerics(case, dtype):
    n, h, w, c, tn, cg, mode = case[:7]
    z = case[7] if len(case) > 7 else 1
    x, w1, w2 = make(n, h, w, c, dtype)
    ch = ts.ConvChain(x.cuda(), w1.cuda(), w2.cuda(), mode=mode, tile_n=tn, cta_group=cg,
                      prod_splits=z, cons_splits=z)
    for _ in range(3):
        y = ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = O.conv_chain(x.float().numpy(), w1.float().numpy(), w2.float().numpy(),
                                DT[dtype])
    check_close(ch.h, h_ref, dtype)
    check_close(y, y_ref, dtype)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())


@pytest.mark.parametrize("tn,cg,c", [(64, 1, 64), (128, 2, 256), (256, 2, 512)])
def test_conv_pair_trace_parity(tn, cg, c):
    """The device trace of the fused conv pair passes the oracle's validate_trace under the
    reference DAG (conv_pair_scenario semantics: consumer k_steps = 9 x producer columns,
    Conv2DTileSync(9)); final semaphores and wait counts are exact."""
    x, w1, w2 = make(2, 14, 14, c, torch.float16, seed=5)
    ch = ts.ConvChain(x.cuda(), w1.cuda(), w2.cuda(), tile_n=tn, cta_group=cg, keep_sems=True)
    ch.cs.enable_trace()
    ch()
    torch.cuda.synchronize()
    sc = ch.cs.scenario()
    assert sc.stages[1].k_steps == 9 * sc.stages[0].grid.y
    stages = [{"id": s.id, "grid": (s.grid.x, s.grid.y, s.grid.z), "k_steps": s.k_steps,
               "order": ("row_major", 1)} for s in sc.stages]
    deps = [{"producer": d.producer, "consumer": d.consumer, "operand": d.operand,
             "policy": ("conv2d", d.policy.kk)} for d in sc.deps]
    evs = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind, "tile": list(e.tile),
            "k": e.k, "dep": e.dep, "sem": e.sem, "expected": e.expected}
           for e in ch.cs.trace_events()]
    assert O.validate_trace(evs, stages, deps, fine=True) == []
    assert {k: tuple(v) for k, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    dag = O.build_dep_dag(stages, deps)
    assert sum(1 for e in evs if e["kind"] == "wait_end") == sum(n for (_, n) in dag.values())
    _, y_ref = O.conv_chain(x.float().numpy(), w1.float().numpy(), w2.float().numpy(), "fp16")
    check_close(ch.y, y_ref, torch.float16)
