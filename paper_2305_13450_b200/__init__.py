"""B200-native tile-level synchronization between dependent kernels (arXiv 2305.13450).

The public names of the reference package ``tilesync_sim`` that sit on the hot path
(/root/reference/pkg/src/tilesync_sim/__init__.py:32-49) are re-exported here with the
same signatures; the policy arithmetic runs in libtilesync_b200.so, the same code the
sm_100a kernels execute. ``CuSync``/``CuStage`` are the paper's host API driving the
persistent tcgen05 chain kernel.
"""

from .chains import AttentionChain, ConvChain, MlpChain, SwigluChain, interleave_gate_up, mlp
from .cusync import CuDep, CuStage, CuSync
from .engine import (CostModel, Dependency, Event, Metrics, Mode, Scenario, SimOptions,
                     SimTrace, Stage, StageMetrics, avoid_wait_kernel, gated_producers,
                     kstep_duration, validate_scenario)
from .errors import ConfigError, MalformedTraceError
from .gpu import (B200_SMS, Dim3, GpuConfig, TileCoord, WaveCount, linearize, tbs_per_wave,
                  utilization, waves)
from .policies import (BandedColumnMajor, Conv2DTileSync, RowMajor, RowSync, SemaphoreArray,
                       StridedRowMajor, StridedSync, SyncPolicy, TileOrder, TileSync, WaitSpec,
                       check_policy, consumer_wait, is_sync, order_tile, post_target,
                       sem_count, wait_steps)

__version__ = "0.1.0"

__all__ = [
    "CostModel", "Dependency", "Event", "Metrics", "Mode", "Scenario", "SimOptions",
    "SimTrace", "Stage", "StageMetrics", "avoid_wait_kernel", "gated_producers",
    "kstep_duration", "validate_scenario",
    "ConfigError", "MalformedTraceError",
    "B200_SMS", "Dim3", "GpuConfig", "TileCoord", "WaveCount", "linearize", "tbs_per_wave",
    "utilization", "waves",
    "BandedColumnMajor", "Conv2DTileSync", "RowMajor", "RowSync", "SemaphoreArray",
    "StridedRowMajor",
    "StridedSync", "SyncPolicy", "TileOrder", "TileSync", "WaitSpec", "check_policy",
    "consumer_wait", "is_sync", "order_tile", "post_target", "sem_count", "wait_steps",
    "CuSync", "CuStage", "CuDep", "AttentionChain", "ConvChain", "MlpChain", "SwigluChain", "interleave_gate_up", "mlp",
]
