"""Split-K fix-up shares, TS_FLAG_SPLIT_FIXUP: every slice of a split CTA-pair tile writes
its fp32 plane; z later items per tile (any free pair) each sum 1/z of the tile's columns
over all planes in slice order, apply the epilogue, store and post once.

The consumer still sees the reference's z posts per producer tile (engine.py:469-514): the
final semaphores must equal the reference-pinned oracle's and the device trace must
validate; results are compared with the CPU oracle (fp16 tolerance) and are bit-identical
across relaunches (static reduction order)."""

import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O
from test_gpu_bench_parity import mlp_inputs
from test_gpu_chain import _scenario_dicts, check_close, make, oracle_mlp

pytestmark = pytest.mark.gpu

TOY = [
    # m, k, n1, n2, prod_tile_n, cons_tile_n, prod_splits, cons_splits, policy, mode
    (1000, 2048, 2048, 1536, 512, 512, 2, 1, ts.RowSync(), "fused"),
    (1000, 3072, 2048, 1536, 512, 256, 3, 2, ts.TileSync(), "fused"),
    (777, 6144, 1024, 1024, 256, 512, 6, 3, ts.RowSync(), "fused"),
    (256, 4096, 1024, 2048, 512, 512, 4, 4, ts.RowSync(), "fused"),
    (300, 8192, 512, 512, 512, 512, 8, 2, ts.TileSync(), "fused"),
    (1000, 2048, 2048, 1536, 512, 512, 2, 2, ts.RowSync(), "stream"),
]


@pytest.mark.parametrize("m,k,n1,n2,pw,cw,pz,cz,pol,mode", TOY)
def test_split_fixup_toy(m, k, n1, n2, pw, cw, pz, cz, pol, mode):
    x, w1, w2 = make(m, k, n1, n2)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=pol, mode=mode, tile_n=256,
                     cta_group=2, prod_tile_n=pw if pw == 512 else 0,
                     cons_tile_n=cw if cw == 512 else 0, prod_splits=pz, cons_splits=cz,
                     split_fixup=True, keep_sems=True)
    if mode == "fused":
        ch.cs.enable_trace()
    y = ch().clone()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(ch.h, h_ref, torch.float16)
    check_close(y, y_ref, torch.float16)
    if mode == "fused":
        stages, deps = _scenario_dicts(ch.cs)
        evs = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind, "tile": list(e.tile),
                "k": e.k, "dep": e.dep, "sem": e.sem, "expected": e.expected}
               for e in ch.cs.trace_events()]
        assert O.validate_trace(evs, stages, deps, fine=True) == []
        assert {k_: tuple(v) for k_, v in O.final_semaphores(stages, deps).items()} == \
            ch.cs.final_semaphores()
    # every counter back to zero; relaunches reproduce the result bit for bit
    assert all(int(v) == 0 for st in ch.cs.stages if st.cnt is not None for v in st.cnt.cpu())
    ch.cs.keep_sems = False
    ch.cs._desc = None
    ch.cs.reset_semaphores()
    for _ in range(3):
        ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    assert torch.equal(ch.y, y)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())
    assert all(int(v) == 0 for st in ch.cs.stages if st.cnt is not None for v in st.cnt.cpu())


@pytest.mark.parametrize("b,pz,cz", [(256, 6, 3), (256, 4, 2), (512, 3, 1), (1024, 2, 1),
                                     (2048, 2, 2)])
def test_split_fixup_gpt3_mlp(b, pz, cz):
    """GPT-3 MLP shard (H=12288, FFN=6144) at the bench sizes, 256x512 pair tiles."""
    x, w1, w2, y_ref = mlp_inputs(b)
    ch = ts.MlpChain(x, w1, w2, policy=ts.RowSync(), tile_n=256, cta_group=2, prod_tile_n=512,
                     cons_tile_n=512, prod_splits=pz, cons_splits=cz, split_fixup=True,
                     keep_sems=True)
    ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    stages, deps = _scenario_dicts(ch.cs)
    assert {k_: tuple(v) for k_, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    check_close(ch.y, y_ref, torch.float16)


def test_split_fixup_ignored_where_it_does_not_apply():
    """Unsplit stages and single-CTA kernels run exactly as without the flag."""
    x, w1, w2 = make(600, 512, 1024, 512)
    ys = []
    for fx in (False, True):
        ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), tile_n=128, cta_group=1,
                         prod_splits=2, split_fixup=fx)
        ys.append(ch().clone())
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1])
