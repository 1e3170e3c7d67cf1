"""Halo-staged convolution stages (TS_FLAG_CONV_HALO): each tile's input rows + 3x3 halo
are loaded once (a 4-D TMA box with zero padding by out-of-bounds fill) and the nine taps
read row-shifted descriptor views of them; the layer's weight taps stay resident.

Numerics against the CPU oracle's direct convolution (pinned to torch conv2d in f64), the
synchronization against the oracle's final semaphores / dependency-safe trace for the
re-tiled grid, in both tile modes (width-padded rows; row segments for wide images)."""

import numpy as np
import pytest
import torch

import paper_2305_13450_b200 as ts
from oracle import tilesync_oracle as O
from test_gpu_chain import _scenario_dicts, check_close

pytestmark = pytest.mark.gpu

# (32, 56) and (80, 28): items of two 128-position sub-tiles (enough images for two items
# per SM); (2, 224) and (5, 129): wide images, two rows of a segment per item (129: an odd
# height, the last item holds one row); the rest one sub-tile
CASES = [(1, 56), (2, 56), (8, 56), (3, 28), (4, 14), (5, 7), (1, 224), (2, 130), (32, 56),
         (80, 28), (2, 224), (5, 129)]


def make(b, hw, c=64, seed=0):
    g = torch.Generator().manual_seed(seed + hw + b)
    x = torch.randn(b, hw, hw, c, generator=g).half()
    w1 = (torch.randn(c, 3, 3, c, generator=g) / (9 * c) ** 0.5).half()
    w2 = (torch.randn(c, 3, 3, c, generator=g) / (9 * c) ** 0.5).half()
    return x, w1, w2


@pytest.mark.parametrize("b,hw", CASES)
@pytest.mark.parametrize("mode", ["fused", "stream"])
def test_conv_halo_pair(b, hw, mode):
    x, w1, w2 = make(b, hw)
    ch = ts.ConvChain(x.cuda(), w1.cuda(), w2.cuda(), tile_n=64, cta_group=1, mode=mode,
                      halo=True, keep_sems=True)
    if mode == "fused":
        ch.cs.enable_trace()
    y = ch()
    torch.cuda.synchronize()
    assert not ch.cs.watchdog_fired()
    h_ref, y_ref = O.conv_chain(x.float().numpy(), w1.float().numpy(), w2.float().numpy(), "fp16")
    check_close(ch.h, h_ref, torch.float16)
    check_close(y, y_ref, torch.float16)
    if mode == "fused":
        stages, deps = _scenario_dicts(ch.cs)
        assert {k: tuple(v) for k, v in O.final_semaphores(stages, deps).items()} == \
            ch.cs.final_semaphores()
        evs = ch.cs.trace_events()
        ev = [{"t": e.time, "stage": e.stage, "tb": e.tb, "kind": e.kind, "tile": list(e.tile),
               "k": e.k, "dep": e.dep, "sem": e.sem, "expected": e.expected} for e in evs]
        assert O.validate_trace(ev, stages, deps, fine=True) == []
    # relaunch: semaphores back to zero, result bit-identical
    ch.cs.keep_sems = False
    ch.cs._desc = None
    ch.cs.reset_semaphores()
    y1 = ch().clone()
    ch()
    torch.cuda.synchronize()
    assert torch.equal(y1, ch.y) and torch.equal(y1, y)
    assert all(int(v) == 0 for d in ch.cs.deps for v in d.sem.cpu())


def test_conv_halo_grid_and_rejects():
    x, w1, w2 = make(2, 56)
    ch = ts.ConvChain(x.cuda(), w1.cuda(), w2.cuda(), tile_n=64, cta_group=1, halo=True)
    # rows of 58 width-padded positions, two per 128-row tile -> 28 tiles per image
    assert ch.prod.grid.x == 2 * 28 and ch.cons.grid.x == 2 * 28
    xb = torch.randn(1, 14, 14, 128, device="cuda").half()
    wb = torch.randn(128, 3, 3, 128, device="cuda").half()
    with pytest.raises(ts.ConfigError):
        ts.ConvChain(xb, wb, wb, tile_n=64, cta_group=1, halo=True)()
