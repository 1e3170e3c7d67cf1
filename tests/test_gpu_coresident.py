"""The paper's co-resident form on B200 (reference engine Mode.FINE with
the wait-kernel gate, engine.py:173-204, tests/test_engine.py:50-86): one launch per stage
on its own stream, live semaphores, the consumer stream gated by the one-thread wait kernel
on its producers' started flags.

* numerics against the CPU oracle, final semaphores / post and wait counts against the
  oracle (pinned to the reference), the device trace dependency-safe;
* gate "on" with an adversarial launch order (consumers enqueued first) completes
  correctly; gate "off" with the same order and a consumer grid that fills every SM
  deadlocks exactly as the reference predicts, and the semaphore watchdog aborts it;
* "auto" gates only when the two grids do not fit one wave (avoid_wait_kernel).
"""

import numpy as np
import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O
from test_gpu_chain import _scenario_dicts, check_close, make, oracle_mlp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pol", [ts.RowSync(), ts.TileSync()])
@pytest.mark.parametrize("gate,adv", [("on", False), ("auto", False), ("on", True)])
@pytest.mark.parametrize("tn,cg", [(128, 1), (256, 2)])
def test_coresident_mlp(pol, gate, adv, tn, cg):
    x, w1, w2 = make(1000, 1024, 2048, 1024)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=pol, mode="coresident", tile_n=tn,
                     cta_group=cg, keep_sems=True)
    ch.cs.wait_kernel, ch.cs.adversarial = gate, adv
    ch.cs.enable_trace()
    y = ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(ch.h, h_ref, torch.float16)
    check_close(y, y_ref, torch.float16)
    stages, deps = _scenario_dicts(ch.cs)
    assert {k: tuple(v) for k, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    evs = ch.cs.trace_events()
    ev_dicts = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind,
                 "tile": list(e.tile), "k": e.k, "dep": e.dep, "sem": e.sem,
                 "expected": e.expected} for e in evs]
    assert O.validate_trace(ev_dicts, stages, deps, fine=True) == []
    dag = O.build_dep_dag(stages, deps)
    assert sum(1 for e in evs if e.kind == "wait_end") == sum(n for (_, n) in dag.values())
    # relaunch without keep_sems: semaphores, counters and started flags come back to zero
    ch.cs.keep_sems = False
    ch.cs._desc = None
    ch.cs.reset_semaphores()
    for _ in range(3):
        ch()
    torch.cuda.synchronize()
    check_close(ch.y, y_ref, torch.float16)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())
    assert int(ch.cs._scratch[16:].abs().sum()) == 0
    assert not ch.cs.watchdog_fired()


def test_coresident_attention():
    g = torch.Generator().manual_seed(3)
    heads, h = 4, 512
    x = torch.randn(700, h, generator=g).half()
    wqkv = (torch.randn(3 * heads * 128, h, generator=g) / h ** 0.5).half()
    w2 = (torch.randn(h, heads * 128, generator=g) / (heads * 128) ** 0.5).half()
    ch = ts.AttentionChain(x.cuda(), wqkv.cuda(), w2.cuda(), mode="coresident", cta_group=1,
                           tile_n=128, keep_sems=True)
    ch.cs.wait_kernel = "on"
    ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    _, dot_ref, y_ref = O.attention_chain(x.float().numpy(), wqkv.float().numpy(),
                                          w2.float().numpy(), "fp16")
    check_close(ch.dot, dot_ref, torch.float16)
    check_close(ch.y, y_ref, torch.float16)
    stages, deps = _scenario_dicts(ch.cs)
    assert {k: tuple(v) for k, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()


def test_gate_off_adversarial_order_deadlocks_and_watchdog_aborts():
    """reference test_engine.py:51-60: with the gate off and consumers scheduled first,
    every SM holds a consumer block spinning on a semaphore no producer can post. Here the
    consumer grid (160 single-CTA tiles) covers all 148 SMs; the watchdog (~4 s) aborts."""
    x, w1, w2 = make(1024, 512, 512, 2560)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=ts.RowSync(), mode="coresident",
                     tile_n=128, cta_group=1)
    assert ch.cons.grid.total() >= torch.cuda.get_device_properties(0).multi_processor_count
    ch.cs.wait_kernel, ch.cs.adversarial = "off", True
    ch()
    torch.cuda.synchronize()
    assert ch.cs.watchdog_fired()
    # the same launch order with the gate on is safe (test_engine.py:62-67)
    ch2 = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=ts.RowSync(), mode="coresident",
                      tile_n=128, cta_group=1)
    ch2.cs.wait_kernel, ch2.cs.adversarial = "on", True
    y = ch2()
    torch.cuda.synchronize()
    assert not ch2.cs.watchdog_fired()
    _, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(y, y_ref, torch.float16)


def test_cuda_graph_replay_coresident():
    x, w1, w2 = make(512, 1024, 1024, 1024)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=ts.TileSync(), mode="coresident")
    ch()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            ch(s)
    for _ in range(4):
        graph.replay()
    torch.cuda.synchronize()
    _, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(ch.y, y_ref, torch.float16)
    assert not ch.cs.watchdog_fired()
