"""ctypes binding of libtilesync_b200.so (include/tilesync.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2305_13450_b200``). There is no fallback: if the shared object is missing
every entry point raises, so a CPU path can never stand in for the device one.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError

LIB_PATH = Path(os.environ.get("TS_LIB_PATH",
                               Path(__file__).resolve().parent / "libtilesync_b200.so"))

TS_OK, TS_ERR_CONFIG, TS_ERR_VALUE, TS_ERR_TYPE, TS_ERR_CUDA, TS_ERR_DEADLOCK = range(6)

TS_POLICY_TILE, TS_POLICY_ROW, TS_POLICY_STRIDED, TS_POLICY_CONV2D = range(4)
TS_ORDER_ROW_MAJOR, TS_ORDER_STRIDED_ROW_MAJOR, TS_ORDER_BANDED_COLUMN_MAJOR = range(3)
TS_DTYPE_F16, TS_DTYPE_BF16 = range(2)
TS_EPI_NONE, TS_EPI_GELU, TS_EPI_SWIGLU, TS_EPI_RELU = range(4)
TS_MODE_STREAM, TS_MODE_FUSED, TS_MODE_CORESIDENT = range(3)
TS_STAGE_GEMM, TS_STAGE_ATTN_DOT, TS_STAGE_CONV2D, TS_STAGE_ALLREDUCE = range(4)
TS_FLAG_KEEP_SEMS, TS_FLAG_NO_REORDER, TS_FLAG_NO_WATCHDOG, TS_FLAG_ROW_INTERLEAVE = 1, 2, 4, 8
TS_FLAG_BALANCED = 16
TS_FLAG_CONV_HALO = 32

TS_MAX_STAGES = 4
TS_MAX_DEPS = 4
TS_SCRATCH_INTS = 32
TS_MAX_PEERS = 8

# Every symbol include/tilesync.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ts_abi_version", "ts_last_error", "ts_sem_count", "ts_post_target",
    "ts_consumer_wait", "ts_wait_steps", "ts_order_tile", "ts_avoid_wait_kernel",
    "ts_chain_launch", "ts_chain_grid", "ts_wait_kernel_launch",
    "ts_device_sm_count", "ts_stream_signal", "ts_stream_wait", "ts_chain_units",
    "ts_chain_launch_coresident",
)


class StageDesc(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p), ("b", ctypes.c_void_p), ("c", ctypes.c_void_p),
        ("m", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int),
        ("lda", ctypes.c_int), ("ldb", ctypes.c_int), ("ldc", ctypes.c_int),
        ("dtype", ctypes.c_int), ("epilogue", ctypes.c_int),
        ("order", ctypes.c_int), ("order_stride", ctypes.c_int),
        ("splits", ctypes.c_int), ("workspace", ctypes.c_void_p),
        ("counters", ctypes.c_void_p), ("kind", ctypes.c_int),
        ("conv_n", ctypes.c_int), ("conv_h", ctypes.c_int), ("conv_w", ctypes.c_int),
        ("tile_n", ctypes.c_int), ("in_sem", ctypes.c_void_p), ("in_expected", ctypes.c_int),
        ("out_sem", ctypes.c_void_p), ("tail_tiles", ctypes.c_int), ("tail_splits", ctypes.c_int),
    ]


class DepDesc(ctypes.Structure):
    _fields_ = [
        ("producer", ctypes.c_int), ("consumer", ctypes.c_int),
        ("operand", ctypes.c_int), ("policy", ctypes.c_int), ("param", ctypes.c_int),
        ("sem", ctypes.c_void_p),
    ]


class PeerDesc(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int), ("rank", ctypes.c_int),
        ("bufs", ctypes.c_void_p * TS_MAX_PEERS), ("sems", ctypes.c_void_p * TS_MAX_PEERS),
        ("done", ctypes.c_void_p * TS_MAX_PEERS), ("epoch", ctypes.c_int),
    ]


class ChainDesc(ctypes.Structure):
    _fields_ = [
        ("n_stages", ctypes.c_int), ("stages", StageDesc * TS_MAX_STAGES),
        ("n_deps", ctypes.c_int), ("deps", DepDesc * TS_MAX_DEPS),
        ("mode", ctypes.c_int), ("tile_n", ctypes.c_int), ("cta_group", ctypes.c_int),
        ("swap_ab", ctypes.c_int), ("flags", ctypes.c_int),
        ("num_ctas", ctypes.c_int), ("scratch", ctypes.c_void_p),
        ("trace", ctypes.c_void_p), ("trace_cap", ctypes.c_int),
        ("peers", ctypes.POINTER(PeerDesc)), ("cluster_pairs", ctypes.c_int),
    ]


class TraceRec(ctypes.Structure):
    _fields_ = [
        ("t_ns", ctypes.c_uint64), ("kind", ctypes.c_int32), ("stage", ctypes.c_int32),
        ("tb", ctypes.c_int32), ("k", ctypes.c_int32), ("dep", ctypes.c_int32),
        ("sem", ctypes.c_int32), ("value", ctypes.c_int32),
        ("x", ctypes.c_int16), ("y", ctypes.c_int16), ("z", ctypes.c_int16),
        ("smid", ctypes.c_int16), ("clk", ctypes.c_int32),
    ]


TRACE_REC_BYTES = ctypes.sizeof(TraceRec)

_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the shared library once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(os.fspath(LIB_PATH))
    ip = ctypes.POINTER(ctypes.c_int)
    i = ctypes.c_int
    sigs = {
        "ts_abi_version": ([], i),
        "ts_last_error": ([], ctypes.c_char_p),
        "ts_sem_count": ([i, i, i, i, i, ip], i),
        "ts_post_target": ([i, i, i, i, i, i, i, i, ip], i),
        "ts_consumer_wait": ([i, i, i, i, i, i, i, i, i, i, ip, ip], i),
        "ts_wait_steps": ([i, i, i, ip, i, ip], i),
        "ts_order_tile": ([i, i, i, i, i, i, ip, ip, ip], i),
        "ts_avoid_wait_kernel": ([i, i, i, i, i, ip], i),
        "ts_chain_launch": ([ctypes.POINTER(ChainDesc), ctypes.c_void_p], i),
        "ts_chain_grid": ([ctypes.POINTER(ChainDesc), i, ip, ip], i),
        "ts_wait_kernel_launch": ([ctypes.c_void_p, i, ctypes.c_void_p], i),
        "ts_device_sm_count": ([ip], i),
        "ts_chain_units": ([i, i, i, i, i, ip], i),
        "ts_stream_signal": ([ctypes.c_void_p, i, ctypes.c_void_p], i),
        "ts_stream_wait": ([ctypes.c_void_p, i, ctypes.c_void_p], i),
        "ts_chain_launch_coresident": ([ctypes.POINTER(ChainDesc),
                                        ctypes.POINTER(ctypes.c_void_p), i, i, i, ip], i),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.ts_abi_version() != 6:
        raise RuntimeError("libtilesync_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int) -> None:
    """Map a ts_status onto the reference's exception types (errors.py:4-9)."""
    if status == TS_OK:
        return
    msg = load().ts_last_error().decode()
    if status == TS_ERR_CONFIG:
        raise ConfigError(msg)
    if status == TS_ERR_VALUE:
        raise ValueError(msg)
    if status == TS_ERR_TYPE:
        raise TypeError(msg)
    raise RuntimeError(f"tilesync status {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
