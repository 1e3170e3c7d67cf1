"""Ready-first k-step order, TS_FLAG_READY_FIRST: a TileSync GeMM consumer takes its k-steps
in the order its producer tiles complete. Every k-step still waits on the reference's
semaphore and count (policies.py:145-166), so the device trace must validate against the
reference-pinned oracle and the final semaphores must equal the oracle's; the numerics
change only by fp32 accumulation order (same tolerance as every fp16 chain test)."""

import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O
from test_gpu_bench_parity import check_sync, mlp_inputs
from test_gpu_chain import _scenario_dicts, check_close, make, oracle_mlp

pytestmark = pytest.mark.gpu

TOY = [
    # m, k, n1, n2, tile_n, cta_group, prod_tile_n, cons_tile_n, cons_splits
    (600, 512, 1024, 512, 128, 1, 0, 0, 1),
    (600, 512, 1024, 512, 128, 2, 0, 0, 1),
    (1000, 1024, 2048, 1536, 256, 2, 512, 512, 1),
    (1000, 1024, 2048, 1536, 256, 2, 256, 512, 1),
    (777, 2048, 4096, 1024, 256, 2, 512, 0, 2),     # split consumer: slices of the k-steps
    (256, 1024, 8192, 1024, 256, 2, 256, 0, 1),     # 32 k-steps per consumer tile
]


def _trace_ok(cs):
    stages, deps = _scenario_dicts(cs)
    evs = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind, "tile": list(e.tile),
            "k": e.k, "dep": e.dep, "sem": e.sem, "expected": e.expected}
           for e in cs.trace_events()]
    assert O.validate_trace(evs, stages, deps, fine=True) == []
    return stages, deps


@pytest.mark.parametrize("m,k,n1,n2,tn,cg,pw,cw,cz", TOY)
def test_ready_first_toy(m, k, n1, n2, tn, cg, pw, cw, cz):
    x, w1, w2 = make(m, k, n1, n2)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=ts.TileSync(), tile_n=tn,
                     cta_group=cg, prod_tile_n=pw, cons_tile_n=cw, cons_splits=cz,
                     ready_first=True, keep_sems=True)
    ch.cs.enable_trace()
    y = ch().clone()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(ch.h, h_ref, torch.float16)
    check_close(y, y_ref, torch.float16)
    stages, deps = _trace_ok(ch.cs)
    assert {k_: tuple(v) for k_, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    # relaunches restore every semaphore; results stay within tolerance (the k order may
    # differ from launch to launch)
    ch.cs.keep_sems = False
    ch.cs._desc = None
    ch.cs.reset_semaphores()
    for _ in range(3):
        ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    check_close(ch.y, y_ref, torch.float16)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())


@pytest.mark.parametrize("b", [256, 1024, 2048])
@pytest.mark.parametrize("prod_splits", [1, 2])
def test_ready_first_gpt3_mlp(b, prod_splits):
    """GPT-3 MLP shard (H=12288, FFN=6144) at the bench sizes, 256x512 pair tiles."""
    x, w1, w2, y_ref = mlp_inputs(b)
    ch = ts.MlpChain(x, w1, w2, policy=ts.TileSync(), tile_n=256, cta_group=2,
                     prod_tile_n=512, cons_tile_n=512, prod_splits=prod_splits,
                     cons_order=ts.BandedColumnMajor(4), ready_first=True, keep_sems=True)
    ch()
    torch.cuda.synchronize()
    check_sync(ch.cs)
    check_close(ch.y, y_ref, torch.float16)


def test_ready_first_is_inert_for_row_sync():
    """RowSync consumers wait once per tile: the flag changes nothing, bit for bit."""
    x, w1, w2 = make(600, 512, 1024, 512)
    ys = []
    for rf in (False, True):
        ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=ts.RowSync(), tile_n=128,
                         cta_group=2, ready_first=rf)
        ys.append(ch().clone())
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1])
