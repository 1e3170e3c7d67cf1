"""Device parity of two-pair clusters (``cluster_pairs=2``): a 256 x 512 tile computed by
two CTA pairs that share the activation rows by TMA multicast.

The reference semantics are those of the 256 x 512 tile (grids, post targets, waits), so
the checks are the same as for the one-pair kernel: outputs against the CPU oracle within
the fp16/bf16 tolerance, the device trace dependency-safe under the reference DAG, and
final semaphores / post and wait counts equal to the oracle's closed form (pinned to the
reference's goldens by tests/test_oracle_golden.py).
"""

import numpy as np
import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O

pytestmark = pytest.mark.gpu

TOL = {torch.float16: (2e-2, 1e-2), torch.bfloat16: (6e-2, 3e-2)}
DT = {torch.float16: "fp16", torch.bfloat16: "bf16"}


def make(m, k, n1, n2, dtype=torch.float16, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(m, k, generator=g).to(dtype)
    w1 = (torch.randn(n1, k, generator=g) / k ** 0.5).to(dtype)
    w2 = (torch.randn(n2, n1, generator=g) / n1 ** 0.5).to(dtype)
    return x, w1, w2


def check_close(dev, ref, dtype):
    atol, rtol = TOL[dtype]
    err = np.abs(dev.float().cpu().numpy() - ref)
    bad = err > atol + rtol * np.abs(ref)
    assert not bad.any(), f"max err {err.max():.4g}, {bad.sum()} elements out of tolerance"


QD = dict(tile_n=256, cta_group=2, cluster_pairs=2, prod_tile_n=512, cons_tile_n=512)

CASES = [
    # m, k, n1, n2, policy, mode, extra
    (256, 1024, 1024, 1024, ts.RowSync(), "fused", {}),
    (512, 1024, 2048, 1024, ts.TileSync(), "fused", {}),
    (520, 768, 1024, 1536, ts.RowSync(), "fused", {"cons_order": ts.BandedColumnMajor(2)}),
    (300, 512, 1024, 512, ts.TileSync(), "stream", {}),
    (1024, 1024, 1024, 2048, ts.RowSync(), "fused", {"prod_splits": 2}),
    (512, 1024, 1024, 1024, ts.TileSync(), "fused", {"prod_splits": 2, "cons_splits": 2}),
    (768, 512, 1024, 2048, ts.RowSync(), "fused", {"cons_tail": (5, 2)}),
    (77, 1024, 1024, 512, ts.RowSync(), "fused", {"prod_splits": 4, "cons_splits": 2}),
]


@pytest.mark.parametrize("m,k,n1,n2,pol,mode,extra", CASES)
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_mlp_two_pair_clusters(m, k, n1, n2, pol, mode, extra, dtype):
    x, w1, w2 = make(m, k, n1, n2, dtype)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=pol, mode=mode, **QD, **extra)
    for _ in range(3):  # relaunches: semaphores and split counters restored
        y = ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = O.mlp_chain(x.float().numpy(), w1.float().numpy(), w2.float().numpy(),
                               DT[dtype])
    check_close(ch.h, h_ref, dtype)
    check_close(y, y_ref, dtype)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())
    for st in ch.cs.stages:
        if st.cnt is not None:
            assert int(st.cnt.abs().sum()) == 0


def test_two_pair_matches_one_pair_bitwise():
    """Same tile, same K order, same fp32 accumulation per output element: the two-pair
    kernel's result equals the one-pair 256 x 512 kernel's bit for bit."""
    x, w1, w2 = make(512, 2048, 2048, 1024, seed=4)
    xd, w1d, w2d = x.cuda(), w1.cuda(), w2.cuda()
    one = ts.MlpChain(xd, w1d, w2d, policy=ts.RowSync(), tile_n=256, cta_group=2,
                      prod_tile_n=512, cons_tile_n=512)().clone()
    two = ts.MlpChain(xd, w1d, w2d, policy=ts.RowSync(), **QD)()
    torch.cuda.synchronize()
    assert torch.equal(one, two)


@pytest.mark.parametrize("pol", [ts.RowSync(), ts.TileSync()])
def test_two_pair_trace_and_semaphores(pol):
    x, w1, w2 = make(600, 512, 1024, 1024, seed=2)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=pol, keep_sems=True, **QD)
    ch.cs.enable_trace()
    ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    sc = ch.cs.scenario()
    kinds = {ts.TileSync: "tile", ts.RowSync: "row"}
    stages = [{"id": s.id, "grid": (s.grid.x, s.grid.y, s.grid.z), "k_steps": s.k_steps,
               "order": ("row_major", 1)} for s in sc.stages]
    deps = [{"producer": d.producer, "consumer": d.consumer, "operand": d.operand,
             "policy": (kinds[type(d.policy)], 0)} for d in sc.deps]
    evs = ch.cs.trace_events()
    ev = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind, "tile": list(e.tile),
           "k": e.k, "dep": e.dep, "sem": e.sem, "expected": e.expected} for e in evs]
    assert O.validate_trace(ev, stages, deps, fine=True) == []
    assert {k: tuple(v) for k, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    dag = O.build_dep_dag(stages, deps)
    assert sum(1 for e in evs if e.kind == "wait_end") == sum(n for (_, n) in dag.values())
    g1 = stages[0]["grid"]
    assert sum(1 for e in evs if e.kind == "post") == g1[0] * g1[1]
    for st in ch.cs.stages:  # one scheduled event per tile, in order_tile order
        sched = [e for e in evs if e.stage == st.id and e.kind == "scheduled"]
        assert sorted(e.tb for e in sched) == list(range(st.grid.total()))


def test_swiglu_two_pair_bf16():
    g = torch.Generator().manual_seed(1)
    m, k, f, n = 300, 512, 1024, 1024
    x = torch.randn(m, k, generator=g).bfloat16()
    wg = (torch.randn(f, k, generator=g) / k ** 0.5).bfloat16()
    wu = (torch.randn(f, k, generator=g) / k ** 0.5).bfloat16()
    wd = (torch.randn(n, f, generator=g) / f ** 0.5).bfloat16()
    wgu = ts.interleave_gate_up(wg, wu, 256)  # each pair: 128 gate + 128 up accumulators
    ch = ts.SwigluChain(x.cuda(), wgu.cuda(), wd.cuda(), policy=ts.TileSync(), tile_n=256,
                        cta_group=2, prod_tile_n=512, cons_tile_n=512, cluster_pairs=2)
    y = ch()
    torch.cuda.synchronize()
    h_ref, y_ref = O.swiglu_chain(x.float().numpy(), wg.float().numpy(), wu.float().numpy(),
                                  wd.float().numpy(), "bf16")
    check_close(ch.h, h_ref, torch.bfloat16)
    check_close(y, y_ref, torch.bfloat16)


def test_two_pair_config_errors():
    x, w1, w2 = make(256, 512, 1024, 512)
    with pytest.raises(ts.ConfigError):  # every GeMM stage must be 256 x 512
        ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), tile_n=256, cta_group=2, cluster_pairs=2)
    with pytest.raises(ts.ConfigError):
        ts.CuSync(tile_n=128, cta_group=2, cluster_pairs=2)
