"""Device tests of the fused tensor-parallel all-reduce stage (CuSync.stage_allreduce,
tp.FusedTPMlp): GeMM1 -> GeLU -> GeMM2 -> all-reduce in one persistent launch per rank.

The GPU box has one B200, so a TP group is simulated on it: every rank is its own chain
(own weights shard, semaphores, scratch, done counter) launched on its own stream with
1/world of the SMs, and the "peer memory" is the other chains' buffers on the same device.
The cross-rank protocol (system-scope posts and acquires, ownership, in-place sums into
every rank's buffer, done counters, deferred semaphore reset) runs exactly as it would over
NVLink; only the transport differs.

Checks: the result on every rank is bit-exact against the fp32 sum of the ranks'
stand-alone partial outputs rounded once (what the stage computes), within tolerance of
the oracle's unsharded MLP, and every semaphore / done counter is back at zero.
"""

import numpy as np
import pytest
import torch

import paper_2305_13450_b200 as ts
from paper_2305_13450_b200 import tp
from oracle import tilesync_oracle as O

pytestmark = pytest.mark.gpu


def make(m, k, n1, n2, seed=0, dtype=torch.float16):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(m, k, generator=g).to(dtype)
    w1 = (torch.randn(n1, k, generator=g) / k ** 0.5).to(dtype)
    w2 = (torch.randn(n2, n1, generator=g) / n1 ** 0.5).to(dtype)
    return x, w1, w2


def run_group(x, w1, w2, world, mode="fused", **kw):
    dev = torch.device("cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ctas = (sms // world) // 2 * 2  # every rank's persistent grid fits at once
    members, parts = [], []
    for r in range(world):
        a, b = tp.shard_mlp(w1, w2, r, world)
        xr, ar, br = x.to(dev), a.to(dev), b.to(dev)
        members.append(tp.FusedTPMlp(xr, ar, br, mode=mode, num_ctas=ctas, **kw))
        ref = ts.MlpChain(xr, ar, br, mode=mode, **kw)  # the same chain without the stage
        parts.append(ref().clone())
    tp.connect_group(members)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()
    for _ in range(3):  # relaunches: the done counters and semaphores must reset
        for m in members:
            m.y.zero_()  # overwritten by GeMM2 every launch
        torch.cuda.synchronize()
        for m, s in zip(members, streams):
            m(s)
        torch.cuda.synchronize()
    return members, parts


def check_counters(m, launches):
    """Chain semaphores are back at zero; the all-reduce group's semaphores and done
    counter are monotone: after e launches every semaphore holds e x (its posts per
    launch) and the done counter e x tiles x cta_group (epoch scheme, ts_peer_desc)."""
    cs = m.chain.cs
    assert cs.epoch == launches
    ard = cs.allreduce_dep()
    g = ard.producer.grid
    assert int(cs.allreduce_done.item()) == launches * g.x * g.y * cs.cta_group
    for d in cs.deps:
        vals = d.sem.cpu().tolist()
        if d is ard:
            assert all(v == launches * g.z for v in vals), vals
        else:
            assert all(v == 0 for v in vals)


@pytest.mark.parametrize("world,mode,kw", [
    (1, "fused", dict(tile_n=256, cta_group=2)),
    (2, "fused", dict(tile_n=256, cta_group=2)),
    (2, "fused", dict(tile_n=128, cta_group=1, policy=ts.TileSync())),
    (2, "stream", dict(tile_n=256, cta_group=2)),
    (4, "fused", dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512)),
    (2, "fused", dict(tile_n=256, cta_group=2, cons_splits=2)),
])
def test_fused_allreduce_matches_sum_of_partials(world, mode, kw):
    x, w1, w2 = make(512, 1024, 2048, 1024, seed=world)
    members, parts = run_group(x, w1, w2, world, mode, **kw)
    expect = sum(p.float() for p in parts).to(parts[0].dtype)
    for m in members:
        assert not m.chain.cs.watchdog_fired()
        assert torch.equal(m.y, expect)
        check_counters(m, launches=3)
    # the TP result against the oracle's unsharded MLP (partials rounded per rank)
    _, ref = O.mlp_chain(x.float().numpy(), w1.float().numpy(), w2.float().numpy(), "fp16")
    err = np.abs(members[0].y.float().cpu().numpy() - ref)
    assert (err <= 2e-2 * world + 1e-2 * np.abs(ref)).all(), err.max()



def test_fused_allreduce_bf16_ragged_rows():
    """bf16, a row count that is not a multiple of the tile (partial last row tile), 3 ranks
    (a world that does not divide the tile count)."""
    x, w1, w2 = make(300, 512, 1536, 768, seed=9, dtype=torch.bfloat16)
    members, parts = run_group(x, w1, w2, 3, "fused", tile_n=256, cta_group=2)
    expect = sum(p.float() for p in parts).to(torch.bfloat16)
    for m in members:
        assert not m.chain.cs.watchdog_fired()
        assert torch.equal(m.y, expect)
        check_counters(m, launches=3)
