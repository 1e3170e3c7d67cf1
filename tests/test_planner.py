"""Planner candidate generation (host logic, no GPU): every candidate is a configuration
the chain builders accept for the shapes it is generated for."""

import pytest

from paper_2305_13450_b200 import planner
from paper_2305_13450_b200.policies import RowSync, TileSync


@pytest.mark.parametrize("m", [1, 64, 256, 512, 1024, 2048])
@pytest.mark.parametrize("mode", ["fused", "stream"])
def test_mlp_candidates_are_well_formed(m, mode):
    cands = planner.candidates(m, mode)
    assert cands, "no candidates"
    for kw in cands:
        assert kw["mode"] == mode
        assert isinstance(kw["policy"], (RowSync, TileSync))
        if mode == "stream":
            assert isinstance(kw["policy"], RowSync)  # the stream baseline has no waits
        if kw.get("swap_ab"):
            assert m <= 256 and kw["tile_n"] >= min(m, 256) and kw["cta_group"] == 1
        else:
            assert kw["tile_n"] in (128, 256)
            if kw.get("prod_tile_n") or kw.get("cons_tile_n"):
                assert (kw["cta_group"], kw["tile_n"]) == (2, 256)
        d = planner.describe(kw)
        assert d["mode"] == mode and "tile" in d


@pytest.mark.parametrize("c", [64, 128, 256, 512])
@pytest.mark.parametrize("m", [49, 3136, 100352])
def test_conv_candidates_fit_the_layer(c, m):
    for kw in planner.conv_candidates(c, "fused", m):
        assert kw["tile_n"] <= c
        z = kw["prod_splits"]
        assert (9 * c // 64) % z == 0
        if z > 1:
            tiles = -(-m // (128 * kw["cta_group"])) * (c // kw["tile_n"])
            assert tiles * z <= 2 * 148


def test_wave_table_matches_survey_appendix_b():
    # B=1024 with 128x256 tiles: 5 stream waves vs 4 fused
    t = planner.wave_table(1024, 6144, 12288, 128, 256)
    assert t["tiles"] == (192, 384)
    assert t["stream_waves"] == 5 and t["fine_waves"] == 4


@pytest.mark.parametrize("h,w,n,want", [
    (56, 56, 1, 28),     # two 58-wide padded rows per 128-position tile
    (56, 56, 16, 28),    # 16 x 14 = 224 two-sub-tile items < 2 x 148: stay at 128
    (56, 56, 32, 14),    # four rows (232 of 256 positions) per two-sub-tile item
    (28, 28, 80, 4),     # eight 30-wide rows per item
    (28, 28, 8, 7),
    (14, 14, 300, 1),    # the whole 16-wide padded image in one item
    (7, 7, 1000, 1),     # 63 positions: one sub-tile is enough
    (224, 224, 64, 224),  # wide rows: 128-position segments of two rows
    (224, 224, 1, 448),   # one row per item: 224 two-row items would be < 2 per SM
])
def test_halo_tiles_per_image(h, w, n, want):
    """Mirror of the halo-conv re-tiling in ts_abi.cu build_params (host logic)."""
    from paper_2305_13450_b200.cusync import halo_tiles_per_image
    assert halo_tiles_per_image(h, w, n, 148) == want
