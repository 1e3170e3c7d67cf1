"""The drop-in policy layer (paper_2305_13450_b200.policies -> libtilesync_b200.so host
functions, the same code the kernels run) against the reference's golden vectors.

Host-only calls: no kernel is launched, so these run on the CPU-only build box."""

import itertools
import json

import pytest

import paper_2305_13450_b200 as ts
from conftest import GOLDEN

TABLES = json.loads((GOLDEN / "policy_tables.json").read_text())


def policy(p):
    kind, param = p
    return {"tile": lambda: ts.TileSync(), "row": lambda: ts.RowSync(),
            "strided": lambda: ts.StridedSync(param),
            "conv2d": lambda: ts.Conv2DTileSync(param)}[kind]()


@pytest.mark.parametrize("case", TABLES["tables"], ids=lambda c: f"{c['policy']}-{c['grid']}")
def test_policy_table(case):
    pol, grid = policy(case["policy"]), ts.Dim3(*case["grid"])
    if case["sem_count"] == "ConfigError":
        with pytest.raises(ts.ConfigError):
            ts.sem_count(pol, grid)
        with pytest.raises(ts.ConfigError):
            ts.check_policy(pol, grid)
        return
    assert ts.sem_count(pol, grid) == case["sem_count"]
    for x, y, z, idx in case["post_target"]:
        assert ts.post_target(pol, ts.TileCoord(x, y, z), grid) == idx
    for x, y, k, w in case["consumer_wait"]:
        got = ts.consumer_wait(pol, ts.TileCoord(x, y, 0), k, grid, grid.z)
        assert (None if got is None else [got.sem_index, got.expected]) == w
    for n, steps in case["wait_steps"].items():
        assert list(ts.wait_steps(pol, int(n))) == steps


@pytest.mark.parametrize("case", TABLES["orders"], ids=lambda c: f"{c['order']}-{c['grid']}")
def test_order_table(case):
    kind, s = case["order"]
    order = ts.RowMajor() if kind == "row_major" else ts.StridedRowMajor(s)
    grid = ts.Dim3(*case["grid"])
    if case["tiles"] == "ConfigError":
        with pytest.raises(ts.ConfigError):
            ts.order_tile(order, grid, 0)
        return
    got = [[t.x, t.y, t.z] for t in (ts.order_tile(order, grid, n) for n in range(grid.total()))]
    assert got == case["tiles"]


def test_error_types_follow_reference():
    # policies.py:133-134 / 188-189: out-of-grid -> ValueError; unknown -> TypeError
    with pytest.raises(ValueError):
        ts.post_target(ts.TileSync(), ts.TileCoord(3, 0, 0), ts.Dim3(3, 2, 1))
    with pytest.raises(ValueError):
        ts.order_tile(ts.RowMajor(), ts.Dim3(3, 2, 1), 6)
    with pytest.raises(TypeError):
        ts.sem_count(object(), ts.Dim3(1, 1, 1))
    with pytest.raises(TypeError):
        ts.order_tile(object(), ts.Dim3(1, 1, 1), 0)
    with pytest.raises(ts.ConfigError):
        ts.sem_count(ts.StridedSync(0), ts.Dim3(1, 6, 1))
    with pytest.raises(ts.ConfigError):
        ts.sem_count(ts.Conv2DTileSync(0), ts.Dim3(1, 6, 1))
    assert issubclass(ts.ConfigError, ValueError)


def test_conservation_law():
    """Every wait's expected value equals the posts that can reach its semaphore
    (test_policies.py:95-125) — checked on the device arithmetic."""
    for gx, gy, gz in itertools.product((1, 2, 3), (1, 2, 4, 6), (1, 2)):
        grid = ts.Dim3(gx, gy, gz)
        for pol in (ts.TileSync(), ts.RowSync(), ts.StridedSync(2), ts.Conv2DTileSync(3)):
            try:
                n = ts.sem_count(pol, grid)
            except ts.ConfigError:
                continue
            posts = [0] * n
            for x, y, z in itertools.product(range(gx), range(gy), range(gz)):
                posts[ts.post_target(pol, ts.TileCoord(x, y, z), grid)] += 1
            k_steps = gy * (3 if isinstance(pol, ts.Conv2DTileSync) else 1)
            for x, y, k in itertools.product(range(gx), range(gy), range(k_steps)):
                w = ts.consumer_wait(pol, ts.TileCoord(x, y), k, grid, gz)
                if w is not None:
                    assert w.expected == posts[w.sem_index]


def test_is_sync_matches_wait_steps():
    for pol in (ts.TileSync(), ts.RowSync(), ts.StridedSync(3), ts.Conv2DTileSync(9)):
        steps = set(ts.wait_steps(pol, 30))
        assert {k for k in range(30) if ts.is_sync(pol, k)} == steps


def test_banded_column_major_is_a_bijection():
    for gx, gy in itertools.product((1, 2, 3, 5, 8), (1, 2, 7, 48)):
        for band in (1, 2, 3, 4, 8):
            grid = ts.Dim3(gx, gy, 1)
            tiles = [ts.order_tile(ts.BandedColumnMajor(band), grid, n)
                     for n in range(grid.total())]
            assert len({(t.x, t.y) for t in tiles}) == grid.total()
            # rows are drawn band by band
            assert [t.x // band for t in tiles] == sorted(t.x // band for t in tiles)
    grid = ts.Dim3(4, 5, 1)
    assert [ts.order_tile(ts.BandedColumnMajor(1), grid, n) for n in range(20)] == \
        [ts.order_tile(ts.RowMajor(), grid, n) for n in range(20)]


def test_wave_arithmetic_b200():
    """128x256 tiles, GPT-3 MLP at B=1024 on 148 SMs."""
    g = ts.GpuConfig(148)
    assert ts.waves(192, g, 1).ceil == 2 and ts.waves(384, g, 1).ceil == 3
    assert ts.waves(192 + 384, g, 1).ceil == 4
    assert ts.utilization(148, g, 1) == 100
    assert ts.linearize(ts.Dim3(3, 2, 2), ts.TileCoord(2, 1, 1)) == 2 + 3 * (1 + 2 * 1)
