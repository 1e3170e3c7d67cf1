"""The C ABI boundary: the library loads, exports every symbol include/tilesync.h
declares, its struct layouts match the ctypes mirror, and host-side validation of a
chain descriptor raises the reference's exception types — all without a GPU."""

import ctypes
import re
import subprocess
import textwrap

import pytest

from conftest import ROOT
from paper_2305_13450_b200 import _lib
from paper_2305_13450_b200.errors import ConfigError

HEADER = ROOT / "include" / "tilesync.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ts_\w+)\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    assert set(names) == set(_lib.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                        capture_output=True, text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}$", nm, re.M), name


def test_abi_version():
    assert _lib.load().ts_abi_version() == 6


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "tilesync.h"
        int main(void) {
          printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(ts_stage_desc), sizeof(ts_dep_desc),
                 sizeof(ts_chain_desc), sizeof(ts_trace_rec),
                 offsetof(ts_chain_desc, scratch), offsetof(ts_trace_rec, clk),
                 sizeof(ts_peer_desc), offsetof(ts_chain_desc, peers));
          return 0;
        }"""))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_lib.StageDesc), ctypes.sizeof(_lib.DepDesc),
            ctypes.sizeof(_lib.ChainDesc), ctypes.sizeof(_lib.TraceRec),
            _lib.ChainDesc.scratch.offset, _lib.TraceRec.clk.offset,
            ctypes.sizeof(_lib.PeerDesc), _lib.ChainDesc.peers.offset]
    assert got == want


def _desc(m=256, n1=1024, k=1024, n2=1024, policy=_lib.TS_POLICY_ROW, param=0,
          tile_n=256, cta_group=1):
    d = _lib.ChainDesc()
    d.n_stages = 2
    fake = 1 << 20  # aligned non-null pointers; nothing is dereferenced on the host
    for i, (mm, nn, kk) in enumerate(((m, n1, k), (m, n2, n1))):
        s = d.stages[i]
        s.a, s.b, s.c = fake, fake, fake
        s.m, s.n, s.k = mm, nn, kk
        s.lda, s.ldb, s.ldc = kk, kk, nn
        s.dtype = _lib.TS_DTYPE_F16
        s.epilogue = _lib.TS_EPI_GELU if i == 0 else _lib.TS_EPI_NONE
    d.n_deps = 1
    dep = d.deps[0]
    dep.producer, dep.consumer, dep.operand = 0, 1, 0
    dep.policy, dep.param, dep.sem = policy, param, fake
    d.mode = _lib.TS_MODE_FUSED
    d.tile_n = tile_n
    d.cta_group = cta_group
    return d


def grid_of(d, s):
    gx, gy = ctypes.c_int(), ctypes.c_int()
    _lib.check(_lib.load().ts_chain_grid(ctypes.byref(d), s, ctypes.byref(gx), ctypes.byref(gy)))
    return gx.value, gy.value


def test_chain_grid_matches_tiling():
    assert grid_of(_desc(cta_group=1), 0) == (2, 4)
    assert grid_of(_desc(cta_group=2), 1) == (1, 4)
    assert grid_of(_desc(m=300, tile_n=128, cta_group=1), 1) == (3, 8)


def test_descriptor_validation_maps_to_reference_errors():
    # consumer K must be the producer's output width
    d = _desc()
    d.stages[1].k = 512
    with pytest.raises(ConfigError):
        grid_of(d, 0)
    # cycle / order (engine.py:142-145)
    d = _desc()
    d.deps[0].producer, d.deps[0].consumer = 1, 0
    with pytest.raises(ConfigError):
        grid_of(d, 0)
    # strided stride must divide the producer's columns (policies.py:102-112)
    with pytest.raises(ConfigError):
        grid_of(_desc(policy=_lib.TS_POLICY_STRIDED, param=3), 0)
    # unknown policy -> TypeError
    with pytest.raises(TypeError):
        grid_of(_desc(policy=9), 0)
    # N not a multiple of the tile width
    with pytest.raises(ConfigError):
        grid_of(_desc(n2=1000), 0)
    # tile_n outside {64, 128, 256}
    with pytest.raises(ValueError):
        grid_of(_desc(tile_n=96), 0)
    # TileSync needs one producer column tile per consumer k-step (engine.py:157-160)
    assert grid_of(_desc(policy=_lib.TS_POLICY_TILE), 1) == (2, 4)


def _allreduce_desc(world=2, rank=0, policy=_lib.TS_POLICY_TILE):
    """MLP chain + all-reduce stage over GeMM2's output (nothing is dereferenced)."""
    d = _desc(cta_group=2)
    d.n_stages = 3
    y = 2 << 20
    d.stages[1].c = y
    ar = d.stages[2]
    ar.a = ar.b = ar.c = y
    ar.m, ar.n, ar.k, ar.lda, ar.ldb, ar.ldc = 256, 1024, 1024, 1024, 1024, 1024
    ar.dtype = _lib.TS_DTYPE_F16
    ar.kind = _lib.TS_STAGE_ALLREDUCE
    d.n_deps = 2
    dep = d.deps[1]
    dep.producer, dep.consumer, dep.operand, dep.policy, dep.param = 1, 2, 0, policy, 0
    dep.sem = 3 << 20
    pd = _lib.PeerDesc()
    pd.world, pd.rank, pd.epoch = world, rank, 1
    for q in range(world):
        pd.bufs[q] = y if q == rank else (4 + q) << 20
        pd.sems[q] = dep.sem if q == rank else (12 + q) << 20
        pd.done[q] = (20 + q) << 20
    d.peers = ctypes.pointer(pd)
    d._keep = pd
    return d


def test_allreduce_stage_validation():
    """TS_STAGE_ALLREDUCE (fused TP all-reduce): tiles = the producer's; descriptor errors
    map onto the reference's exception types."""
    assert grid_of(_allreduce_desc(), 2) == grid_of(_allreduce_desc(), 1)
    d = _allreduce_desc()
    d.peers = None
    with pytest.raises(ValueError):
        grid_of(d, 2)
    with pytest.raises(ConfigError):  # the all-reduce waits tile by tile
        grid_of(_allreduce_desc(policy=_lib.TS_POLICY_ROW), 2)
    with pytest.raises(ValueError):  # rank outside the group
        grid_of(_allreduce_desc(world=2, rank=2), 2)
    d = _allreduce_desc()
    d._keep.bufs[0] = 9 << 20  # peers.bufs[rank] must be the stage's own buffer
    with pytest.raises(ValueError):
        grid_of(d, 2)
    d = _allreduce_desc()
    d.stages[2].c = d.stages[2].a = 7 << 20  # sums its producer's output in place
    d._keep.bufs[0] = 7 << 20
    with pytest.raises(ConfigError):
        grid_of(d, 2)
    d = _allreduce_desc()
    d._keep.epoch = 0  # launch generations start at 1 (monotone semaphores)
    with pytest.raises(ValueError):
        grid_of(d, 2)
    d = _allreduce_desc()  # no stage may follow the all-reduce (it borrows the smem ring)
    d.n_stages = 4
    d.stages[3] = d.stages[1]
    with pytest.raises(ConfigError):
        grid_of(d, 2)


def test_row_interleave_validation():
    """TS_FLAG_ROW_INTERLEAVE needs a fused two-GeMM Row/TileSync chain with RowMajor
    orders and equal row tiles; stream mode ignores it."""
    d = _desc(cta_group=2)
    d.flags = _lib.TS_FLAG_ROW_INTERLEAVE
    assert grid_of(d, 1) == (1, 4)
    d = _desc(cta_group=1, policy=_lib.TS_POLICY_STRIDED, param=2)
    d.flags = _lib.TS_FLAG_ROW_INTERLEAVE
    with pytest.raises(ConfigError):
        grid_of(d, 1)
    d = _desc(cta_group=1)
    d.flags = _lib.TS_FLAG_ROW_INTERLEAVE
    d.stages[1].order, d.stages[1].order_stride = _lib.TS_ORDER_BANDED_COLUMN_MAJOR, 2
    with pytest.raises(ConfigError):
        grid_of(d, 1)
    d.mode = _lib.TS_MODE_STREAM
    assert grid_of(d, 1) == (2, 4)
