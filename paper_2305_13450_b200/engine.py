"""Stage / dependency / scenario types and the protocol rules around them.

Drop-in for the host-side half of /root/reference/pkg/src/tilesync_sim/engine.py:
``Stage``, ``Dependency``, ``Scenario`` (engine.py:71-131) with the same structural
checks (``validate_scenario``, engine.py:134-170), the wait-kernel gate
(``avoid_wait_kernel`` / ``gated_producers``, engine.py:173-204), the "+R" k-step
formula (``kstep_duration``, engine.py:207-217) and the JSONL trace schema
(``Event`` / ``SimTrace``, engine.py:220-265).

What the reference's discrete-event loop (``_Engine``, engine.py:352-611) models in
abstract time, the B200 build *executes*: the persistent chain kernel
(csrc/ts_chain_kernel.cuh) claims tiles from one counter (``_grant``), spins on the
policy's semaphore before each dependent k-step while holding its SM (``_advance``),
and posts at tile completion (``_finish``). Its device trace comes back as ``Event``
records in this schema (see ``cusync.CuSync.trace``).
"""

from __future__ import annotations

import enum
import json
from dataclasses import dataclass, replace
from fractions import Fraction

from . import _lib
from .errors import ConfigError
from .gpu import Dim3, GpuConfig
from .policies import (Conv2DTileSync, RowMajor, RowSync, StridedRowMajor, SyncPolicy,
                       TileOrder, TileSync, check_policy)


class Mode(str, enum.Enum):
    STREAM = "stream"   # one kernel after another on one stream (coarse sync)
    FINE = "fine"       # tile-level semaphores, kernels overlap


@dataclass(frozen=True)
class CostModel:
    """Relative per-k-step costs (engine.py:45-56). Only the planner's wave model uses
    them; device timings are measured, never modelled."""

    load: float = 1
    compute: float = 1
    sync_overhead: float = 0
    epilogue: float = 0

    def __post_init__(self) -> None:
        if min(self.load, self.compute, self.sync_overhead, self.epilogue) < 0:
            raise ConfigError("cost parameters must be >= 0")


@dataclass(frozen=True)
class SimOptions:
    """Protocol switches (engine.py:59-68): the wait-kernel gate ("+W") and the
    dependent-load reorder ("+R")."""

    wait_kernel: str = "auto"  # on | off | auto
    reorder_loads: bool = False
    adversarial_order: bool = False

    def __post_init__(self) -> None:
        if self.wait_kernel not in ("on", "off", "auto"):
            raise ConfigError(f"wait_kernel must be on/off/auto, got {self.wait_kernel!r}")


@dataclass(frozen=True)
class Stage:
    """One tiled kernel: grid, occupancy, reduction depth in producer-tile units, order."""

    id: str
    grid: Dim3
    occupancy: int = 1
    k_steps: int = 1
    order: TileOrder = RowMajor()
    operands: tuple[str, ...] = ("a", "b")
    stream_priority: int | None = None
    cost: CostModel | None = None

    def __post_init__(self) -> None:
        if self.occupancy < 1:
            raise ConfigError(f"stage {self.id}: occupancy must be >= 1")
        if self.k_steps < 1:
            raise ConfigError(f"stage {self.id}: k_steps must be >= 1")
        if len(set(self.operands)) != len(self.operands):
            raise ConfigError(f"stage {self.id}: duplicate operand names")
        if isinstance(self.order, StridedRowMajor) and self.grid.y % self.order.stride:
            raise ConfigError(f"stage {self.id}: order stride {self.order.stride} does not "
                              f"divide grid columns {self.grid.y}")


@dataclass(frozen=True)
class Dependency:
    """The consumer's `operand` tiles come from `producer`, synchronized by `policy`."""

    producer: str
    consumer: str
    operand: str = "a"
    policy: SyncPolicy = RowSync()

    @property
    def id(self) -> str:
        return f"{self.producer}->{self.consumer}/{self.operand}"


@dataclass(frozen=True)
class Scenario:
    gpu: GpuConfig
    stages: tuple[Stage, ...]
    deps: tuple[Dependency, ...] = ()
    mode: Mode = Mode.FINE
    options: SimOptions = SimOptions()
    cost: CostModel = CostModel()

    def __post_init__(self) -> None:
        validate_scenario(self)

    def with_mode(self, mode: Mode) -> "Scenario":
        return replace(self, mode=mode)

    def stage_by_id(self, stage_id: str) -> Stage:
        for s in self.stages:
            if s.id == stage_id:
                return s
        raise KeyError(stage_id)


def validate_scenario(sc: Scenario) -> None:
    """Structural rules of engine.py:134-170, raised as ConfigError."""
    pos: dict[str, int] = {}
    for i, s in enumerate(sc.stages):
        if s.id in pos:
            raise ConfigError("duplicate stage ids")
        pos[s.id] = i
    for dep in sc.deps:
        if dep.producer not in pos or dep.consumer not in pos:
            raise ConfigError(f"dependency {dep.id} names unknown stage")
        if pos[dep.producer] >= pos[dep.consumer]:
            raise ConfigError(f"dependency {dep.id}: producer must be invoked before "
                              f"consumer (cycles are not allowed)")
        prod, cons = sc.stages[pos[dep.producer]], sc.stages[pos[dep.consumer]]
        if dep.operand not in cons.operands:
            raise ConfigError(f"dependency {dep.id}: {dep.operand!r} is not an operand of "
                              f"stage {cons.id}")
        check_policy(dep.policy, prod.grid)
        if cons.grid.x > prod.grid.x:
            raise ConfigError(f"dependency {dep.id}: consumer rows {cons.grid.x} exceed "
                              f"producer rows {prod.grid.x}")
        if isinstance(dep.policy, TileSync) and cons.k_steps > prod.grid.y:
            raise ConfigError(f"dependency {dep.id}: tile sync needs one producer column "
                              f"per consumer k-step ({cons.k_steps} > {prod.grid.y})")
        if isinstance(dep.policy, Conv2DTileSync):
            kk = dep.policy.kk
            if cons.k_steps % kk:
                raise ConfigError(f"dependency {dep.id}: kk {kk} does not divide consumer "
                                  f"k_steps {cons.k_steps}")
            if cons.k_steps > kk * prod.grid.y:
                raise ConfigError(f"dependency {dep.id}: consumer k_steps {cons.k_steps} "
                                  f"exceed kk * producer columns {kk * prod.grid.y}")


def avoid_wait_kernel(producer: Stage, consumer: Stage, gpu: GpuConfig) -> bool:
    """"+W": both grids fit one combined wave, so the
    wait kernel is unnecessary. Evaluated by the same C function the launcher uses."""
    import ctypes
    out = ctypes.c_int(0)
    _lib.call("ts_avoid_wait_kernel", producer.grid.total(), producer.occupancy,
              consumer.grid.total(), consumer.occupancy, gpu.num_sms, ctypes.byref(out))
    return bool(out.value)


def gated_producers(scenario: Scenario, stage: Stage) -> tuple[str, ...]:
    """Producers that must have started before `stage` may schedule (engine.py:183-204)."""
    if scenario.mode is not Mode.FINE or scenario.options.wait_kernel == "off":
        return ()
    out: list[str] = []
    for dep in scenario.deps:
        if dep.consumer != stage.id or dep.producer in out:
            continue
        prod = scenario.stage_by_id(dep.producer)
        if scenario.options.wait_kernel == "auto" and avoid_wait_kernel(prod, stage,
                                                                        scenario.gpu):
            continue
        out.append(dep.producer)
    return tuple(out)


def kstep_duration(wait: float, dep_load: float, other_loads: float, compute: float,
                   reorder: bool = False) -> float:
    """One k-step's length (engine.py:207-217). With "+R" the independent loads are
    issued before the semaphore spin and overlap it — what the TMA warp does when
    TS_FLAG_NO_REORDER is clear."""
    if reorder:
        return max(wait, other_loads) + dep_load + compute
    return wait + dep_load + other_loads + compute


@dataclass(frozen=True)
class Event:
    """One trace record (engine.py:220-248). Device traces use ns for `time`."""

    time: float
    stage: str
    tb: int
    kind: str  # scheduled | wait_begin | wait_end | post | finished
    tile: tuple[int, int, int]
    k: int | None = None
    dep: str | None = None
    sem: int | None = None
    expected: int | None = None
    value: int | None = None

    def to_json(self) -> str:
        rec: dict = {"t": self.time, "stage": self.stage, "tb": self.tb, "kind": self.kind,
                     "tile": list(self.tile)}
        for name in ("k", "sem", "expected", "value", "dep"):
            v = getattr(self, name)
            if v is not None:
                rec[name] = v
        return json.dumps(rec, sort_keys=True)

    @classmethod
    def from_json(cls, line: str) -> "Event":
        r = json.loads(line)
        return cls(time=r["t"], stage=r["stage"], tb=r["tb"], kind=r["kind"],
                   tile=tuple(r["tile"]), k=r.get("k"), dep=r.get("dep"), sem=r.get("sem"),
                   expected=r.get("expected"), value=r.get("value"))


@dataclass
class SimTrace:
    mode: Mode
    events: list[Event]
    final_semaphores: dict[str, tuple[int, ...]]

    def dump_jsonl(self, path) -> None:
        with open(path, "w") as fh:
            for ev in self.events:
                fh.write(ev.to_json() + "\n")

    @staticmethod
    def load_events(path) -> list[Event]:
        with open(path) as fh:
            return [Event.from_json(line) for line in fh if line.strip()]


@dataclass(frozen=True)
class StageMetrics:
    stage: str
    tbs: int
    waves_frac: Fraction
    waves_ceil: int
    utilization_pct: Fraction
    finish_time: float | None
    total_wait: float


@dataclass(frozen=True)
class Metrics:
    mode: Mode
    per_stage: tuple[StageMetrics, ...]
    combined_waves_frac: Fraction
    combined_waves_ceil_sum: int
    generations: int
    generation_sizes: tuple[int, ...]
    makespan: float
    total_wait: float
    deadlock: bool

    @property
    def combined_waves(self) -> Fraction | int:
        if self.mode is Mode.STREAM:
            return self.combined_waves_ceil_sum
        return self.combined_waves_frac
