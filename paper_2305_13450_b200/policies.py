"""Synchronization policies and tile orders — the hot-path API.

Drop-in for /root/reference/pkg/src/tilesync_sim/policies.py: the same frozen
dataclasses and the same five functions with the same signatures, results and
exceptions. The arithmetic is *not* re-implemented in Python: every function calls
the C ABI (``ts_sem_count`` ...), which runs the very ``__host__ __device__``
functions (csrc/ts_policy.cuh) the B200 kernels execute in their producer warp and
epilogue. Whatever the Python layer answers is what the device does.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Union

from . import _lib
from .gpu import Dim3, TileCoord


@dataclass(frozen=True)
class TileSync:
    """One semaphore per producer tile; the consumer waits before every k-step
    (policies.py:24-26)."""


@dataclass(frozen=True)
class RowSync:
    """One semaphore per producer row; the consumer waits once, at k-step 0
    (policies.py:29-31)."""


@dataclass(frozen=True)
class StridedSync:
    """Producer tiles whose columns are `stride` apart share a semaphore
    (policies.py:34-38)."""

    stride: int


@dataclass(frozen=True)
class Conv2DTileSync:
    """Tile sync through an implicit-GeMM KxK convolution: only every kk-th consumer
    k-step starts a new producer tile (policies.py:41-50)."""

    kk: int


SyncPolicy = Union[TileSync, RowSync, StridedSync, Conv2DTileSync]


@dataclass(frozen=True)
class RowMajor:
    """Tiles drawn in lexicographic (x, y, z) order (policies.py:56-58)."""


@dataclass(frozen=True)
class StridedRowMajor:
    """Row-major over columns regrouped so columns `stride` apart are drawn together
    (policies.py:61-70; the paper's StrideSync::prodOrder)."""

    stride: int


@dataclass(frozen=True)
class BandedColumnMajor:
    """Extension order (not in the reference simulator; the paper lists further orders,
    PAPER.md:427): bands of `band` tile rows in order, column by column inside a band,
    so the row tiles that share a weight column block run together and the block
    streams from HBM once per band. ``BandedColumnMajor(1)`` is RowMajor."""

    band: int


TileOrder = Union[RowMajor, StridedRowMajor, BandedColumnMajor]


@dataclass(frozen=True)
class WaitSpec:
    """Block until ``sem[sem_index] >= expected`` (policies.py:76-81)."""

    sem_index: int
    expected: int


class SemaphoreArray:
    """Host model of a device semaphore array: monotone counters from zero
    (policies.py:84-99). The device array is an ``int32`` tensor; see ``cusync``."""

    def __init__(self, count: int):
        self.values = [0] * count

    def post(self, index: int) -> int:
        self.values[index] += 1
        return self.values[index]

    def satisfied(self, spec: WaitSpec) -> bool:
        return self.values[spec.sem_index] >= spec.expected

    def __len__(self) -> int:
        return len(self.values)


def policy_code(policy: SyncPolicy) -> tuple[int, int]:
    """(ts_policy_kind, param) of a policy object, as the C ABI takes it."""
    if isinstance(policy, TileSync):
        return _lib.TS_POLICY_TILE, 0
    if isinstance(policy, RowSync):
        return _lib.TS_POLICY_ROW, 0
    if isinstance(policy, StridedSync):
        return _lib.TS_POLICY_STRIDED, policy.stride
    if isinstance(policy, Conv2DTileSync):
        return _lib.TS_POLICY_CONV2D, policy.kk
    raise TypeError(f"unknown policy {policy!r}")


def order_code(order: TileOrder) -> tuple[int, int]:
    """(ts_order_kind, stride) of a tile order."""
    if isinstance(order, RowMajor):
        return _lib.TS_ORDER_ROW_MAJOR, 1
    if isinstance(order, StridedRowMajor):
        return _lib.TS_ORDER_STRIDED_ROW_MAJOR, order.stride
    if isinstance(order, BandedColumnMajor):
        return _lib.TS_ORDER_BANDED_COLUMN_MAJOR, order.band
    raise TypeError(f"unknown order {order!r}")


def _out() -> ctypes.c_int:
    return ctypes.c_int(0)


def check_policy(policy: SyncPolicy, producer_grid: Dim3) -> None:
    """Raise ConfigError when the policy's divisibility constraints fail
    (policies.py:102-112)."""
    sem_count(policy, producer_grid)


def sem_count(policy: SyncPolicy, producer_grid: Dim3) -> int:
    """Semaphores a dependency under `policy` allocates (policies.py:115-125)."""
    kind, param = policy_code(policy)
    out = _out()
    _lib.call("ts_sem_count", kind, param, producer_grid.x, producer_grid.y,
              producer_grid.z, ctypes.byref(out))
    return out.value


def post_target(policy: SyncPolicy, tile: TileCoord, producer_grid: Dim3) -> int:
    """Semaphore a finished producer tile increments; all z-slices share it
    (policies.py:128-142)."""
    if not tile.within(producer_grid):
        raise ValueError(f"tile {tile} outside producer grid {producer_grid}")
    kind, param = policy_code(policy)
    out = _out()
    _lib.call("ts_post_target", kind, param, tile.x, tile.y, tile.z, producer_grid.x,
              producer_grid.y, producer_grid.z, ctypes.byref(out))
    return out.value


def consumer_wait(policy: SyncPolicy, consumer_tile: TileCoord, k_step: int,
                  producer_grid: Dim3, producer_z: int) -> WaitSpec | None:
    """The wait a consumer tile issues before `k_step`, or None (policies.py:145-166)."""
    kind, param = policy_code(policy)
    sem, exp = _out(), _out()
    _lib.call("ts_consumer_wait", kind, param, consumer_tile.x, consumer_tile.y,
              consumer_tile.z, k_step, producer_grid.x, producer_grid.y, producer_grid.z,
              producer_z, ctypes.byref(sem), ctypes.byref(exp))
    if sem.value < 0:
        return None
    return WaitSpec(sem.value, exp.value)


def wait_steps(policy: SyncPolicy, k_steps: int) -> tuple[int, ...]:
    """k-steps at which `policy` waits (policies.py:169-178) — the paper's isSync."""
    kind, param = policy_code(policy)
    cap = max(1, k_steps)
    buf = (ctypes.c_int * cap)()
    n = _out()
    _lib.call("ts_wait_steps", kind, param, k_steps, buf, cap, ctypes.byref(n))
    return tuple(buf[i] for i in range(n.value))


def is_sync(policy: SyncPolicy, k_step: int) -> bool:
    """True when `policy` waits before `k_step` — the paper's isSync hook."""
    return k_step in wait_steps(policy, k_step + 1)


def order_tile(order: TileOrder, grid: Dim3, counter: int) -> TileCoord:
    """Tile of the `counter`-th draw from a stage's global counter (policies.py:181-205)."""
    if not 0 <= counter < grid.total():
        raise ValueError(f"counter {counter} outside grid {grid}")
    kind, stride = order_code(order)
    x, y, z = _out(), _out(), _out()
    _lib.call("ts_order_tile", kind, stride, grid.x, grid.y, grid.z, counter,
              ctypes.byref(x), ctypes.byref(y), ctypes.byref(z))
    return TileCoord(x.value, y.value, z.value)
