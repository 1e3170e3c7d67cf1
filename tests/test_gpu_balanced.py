"""The balanced (static stream-K) schedule, TS_FLAG_BALANCED: every CTA pair runs an equal
K-block range of each GeMM stage; tiles cut between pairs are reduced into the head
segment's TMEM accumulator, which posts once (the reference's unsplit-tile semantics).

Checked against the CPU oracle (numerics) and the reference-pinned oracle / golden final
semaphores (synchronization), at toy sizes with ragged rows and at the GPT-3 MLP shard
sizes bench.py runs; relaunches must restore every counter and reproduce the result
bit for bit (the reduction order is static)."""

import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O
from test_gpu_bench_parity import check_sync, mlp_inputs
from test_gpu_chain import _scenario_dicts, check_close, make, oracle_mlp

pytestmark = pytest.mark.gpu

TOY = [
    # m, k, n1, n2, prod_tile_n, cons_tile_n, policy, num_ctas
    (1000, 1024, 2048, 1536, 512, 512, ts.RowSync(), 0),
    (1000, 1024, 2048, 1536, 512, 256, ts.TileSync(), 0),
    (777, 2048, 1024, 1024, 256, 512, ts.RowSync(), 0),
    (256, 4096, 1024, 2048, 512, 512, ts.TileSync(), 0),
    (512, 1024, 1024, 1024, 512, 512, ts.RowSync(), 20),   # few units: several tiles per unit
    (300, 8192, 512, 512, 512, 512, ts.RowSync(), 0),      # more units than tiles
]


@pytest.mark.parametrize("m,k,n1,n2,pw,cw,pol,nc", TOY)
def test_balanced_toy(m, k, n1, n2, pw, cw, pol, nc):
    x, w1, w2 = make(m, k, n1, n2)
    ch = ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), policy=pol, tile_n=256, cta_group=2,
                     prod_tile_n=pw if pw == 512 else 0, cons_tile_n=cw if cw == 512 else 0,
                     balanced=True, keep_sems=True, num_ctas=nc)
    y = ch().clone()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = oracle_mlp(x, w1, w2, torch.float16)
    check_close(ch.h, h_ref, torch.float16)
    check_close(y, y_ref, torch.float16)
    stages, deps = _scenario_dicts(ch.cs)
    assert {k_: tuple(v) for k_, v in O.final_semaphores(stages, deps).items()} == \
        ch.cs.final_semaphores()
    assert all(int(v) == 0 for st in ch.cs.stages for v in st.cnt.cpu())
    ch.cs.keep_sems = False
    ch.cs._desc = None
    ch.cs.reset_semaphores()
    for _ in range(3):
        ch()
    torch.cuda.synchronize()
    assert torch.equal(ch.y, y)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())
    assert all(int(v) == 0 for st in ch.cs.stages for v in st.cnt.cpu())


@pytest.mark.parametrize("b", [256, 512, 1024, 2048])
@pytest.mark.parametrize("pol", [ts.RowSync(), ts.TileSync()])
def test_balanced_gpt3_mlp(b, pol):
    """GPT-3 MLP shard (H=12288, FFN=6144) at the bench sizes, 256x512 pair tiles."""
    x, w1, w2, y_ref = mlp_inputs(b)
    ch = ts.MlpChain(x, w1, w2, policy=pol, tile_n=256, cta_group=2, prod_tile_n=512,
                     cons_tile_n=512, cons_order=ts.BandedColumnMajor(4), balanced=True,
                     keep_sems=True)
    ch()
    torch.cuda.synchronize()
    check_sync(ch.cs)
    check_close(ch.y, y_ref, torch.float16)


def test_balanced_rejects_unsupported():
    x, w1, w2 = make(256, 1024, 1024, 1024)
    with pytest.raises(ts.ConfigError):
        ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), cta_group=1, tile_n=128, balanced=True)()
    with pytest.raises(ts.ConfigError):
        ts.MlpChain(x.cuda(), w1.cuda(), w2.cuda(), prod_splits=2, balanced=True)()
