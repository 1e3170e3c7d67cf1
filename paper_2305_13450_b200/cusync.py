"""The paper's host API on B200: ``CuSync`` / ``CuStage``.

    cs = CuSync(tile_n=256)
    prod = cs.stage(x, w1, h, epilogue="gelu")            # h  = GeLU(x @ w1^T)
    cons = cs.stage(h, w2, y)                             # y  = h @ w2^T
    cs.dependency(RowSync(), prod, cons, operand="a")     # cs.dependency<RowSync>(...)
    cs.launch()                                           # one persistent launch

A stage is a GeMM ``C = epi(A @ B^T)`` with ``A [m, k]`` and ``B [n, k]`` K-major
(weights in nn.Linear layout), fp16 or bf16, fp32 accumulate. Every tensor is owned by
PyTorch; the C ABI borrows the pointers for one stream-ordered launch on the current
torch stream. Semaphores are ``int32`` tensors, zero on entry; the kernel restores the
zero invariant on exit (unless ``keep_sems``), so a CuSync can be launched repeatedly
and captured in a CUDA graph.

Modes
  * ``"fused"``  — one persistent launch over all stages' tiles; consumers wait on
    semaphores (the paper's fine-grained synchronization, with the persistent claim
    order replacing the wait kernel: deadlock-free by construction).
  * ``"stream"`` — the same kernel, one launch per stage on one stream, no semaphores:
    the stream-synchronized baseline the paper compares against.
  * ``"coresident"`` — the paper's own form: one launch per stage,
    each on its own stream (producers at higher priority), semaphores live; a consumer
    stage's stream first runs the one-thread wait kernel on its producers' started flags
    (``wait_kernel`` = "on" / "off" / "auto", the reference's SimOptions.wait_kernel and
    gated_producers, engine.py:173-204; ``CuStage.wait_kernel()`` forces it on).
    ``adversarial=True`` enqueues consumers before producers (SimOptions.adversarial_order):
    with the gate off a consumer grid that fills the GPU deadlocks, and the semaphore
    watchdog aborts the launch (``watchdog_fired()``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib
from .engine import Dependency, Event, Mode, Scenario, SimOptions, SimTrace, Stage
from .errors import ConfigError
from .gpu import Dim3, GpuConfig
from .policies import (Conv2DTileSync, RowMajor, SyncPolicy, TileOrder, order_code,
                       policy_code, sem_count)

BM = 128
BK = 64
_EPI = {"none": _lib.TS_EPI_NONE, "gelu": _lib.TS_EPI_GELU, "swiglu": _lib.TS_EPI_SWIGLU,
        "relu": _lib.TS_EPI_RELU}
_DT = {torch.float16: _lib.TS_DTYPE_F16, torch.bfloat16: _lib.TS_DTYPE_BF16}
_KINDS = ("scheduled", "wait_begin", "wait_end", "post", "finished")
# Replay order for events sharing a timestamp: posts before the waits they justify
# (oracle.py:133-144), and a block's own events in program order.
_RANK = {"post": 0, "finished": 1, "scheduled": 2, "wait_begin": 3, "wait_end": 4}


@dataclass
class CuStage:
    """One GeMM stage (the paper's CuStage)."""

    cs: "CuSync"
    index: int
    id: str
    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor
    epilogue: str
    order: TileOrder
    splits: int = 1
    ws: torch.Tensor | None = None
    cnt: torch.Tensor | None = None
    kind: str = "gemm"  # "gemm", "dot" (attention's fused softmax-dot), "conv" or
    # "allreduce" (tensor-parallel sum of its producer's output over peer memory)
    conv: tuple | None = None  # (N, H, W) of a 3x3 "same" convolution stage
    in_sem: torch.Tensor | None = None   # external row gate on operand A (ts_stream_signal)
    out_sem: torch.Tensor | None = None  # per-row "tiles stored" counters (ts_stream_wait)
    tile_n: int = 0     # 0 = the chain's tile_n; 512 = double-width CTA-pair tile
    tail: tuple = (0, 1)  # (tiles, slices): last-wave balancing of a final stage

    @property
    def m(self) -> int:
        return self.a.shape[0]

    @property
    def n(self) -> int:
        """Output columns (accumulator columns for SwiGLU)."""
        return self.c.shape[1] if self.kind in ("dot", "allreduce") else self.b.shape[0]

    @property
    def k(self) -> int:
        """Reduction length (9 x Cin for a convolution: KRSC weight row length)."""
        return self.b.shape[1] if self.kind == "conv" else self.a.shape[1]

    @property
    def width(self) -> int:
        """Accumulator columns of one tile."""
        if self.cs.swap_ab:
            return 128
        return self.tile_n or self.cs.tile_n

    @property
    def out_tile_cols(self) -> int:
        """Output columns one tile writes (a consumer k-step in reference units)."""
        return self.width // 2 if self.epilogue == "swiglu" else self.width

    @property
    def grid(self) -> Dim3:
        """Tile grid as the reference's Stage.grid sees it: (activation-row tiles,
        output-column tiles, split-K slices). A halo-staged convolution tiles each image's
        positions separately (``halo_tiles_per_image``)."""
        if self.kind == "conv" and self.cs.conv_halo:
            n, h, w = self.conv
            return Dim3(n * halo_tiles_per_image(h, w, n, _device_sms()),
                        max(1, self.n // self.width), self.splits)
        return Dim3(-(-self.m // self.cs.tile_m), max(1, self.n // self.width), self.splits)

    def flops(self) -> int:
        return 0 if self.kind in ("dot", "allreduce") else 2 * self.m * self.n * self.k

    def wait_kernel(self) -> "CuStage":
        """``stage.wait_kernel()``: in co-resident mode, hold this
        stage's launch back until its producers have started (the chain's gate becomes
        "on")."""
        self.cs.wait_kernel = "on"
        return self


_SMS: int | None = None


def _device_sms() -> int:
    """SM count of the current device, as the library sees it (ts_device_sm_count)."""
    global _SMS
    if _SMS is None:
        out = ctypes.c_int(0)
        _lib.check(_lib.load().ts_device_sm_count(ctypes.byref(out)))
        _SMS = out.value
    return _SMS


_HALO_WINDOW_BYTES = 9 * 24576 - 9 * 8192  # ts_abi.cu: the BN = 64 ring minus resident weights


def halo_tiles_per_image(h: int, w: int, n: int = 1, sms: int = 148) -> int:
    """Tiles (items) of one H x W image under TS_FLAG_CONV_HALO (ts_abi.cu build_params):
    the whole width-padded rows (row stride W + 2) that fit 256 positions — two 128-row
    sub-tiles — when their window fits two buffers and n images give two items per SM
    (`sms`: the device's SM count), else 128 positions, while W + 2 <= 128; else
    128-position segments of one row, or of two rows under the same conditions."""
    srow = w + 2
    if srow <= 128:
        rpt = min(128 // srow, h)
        # two 128-position sub-tiles per item when their window fits two buffers and the
        # n images still give two items per SM
        rpt2 = min(256 // srow, h)
        win2 = -(-((rpt2 + 2) * srow * 128) // 1024) * 1024
        if rpt2 * srow > 128 and _HALO_WINDOW_BYTES // win2 >= 2 and n * -(-h // rpt2) >= 2 * sms:
            rpt = rpt2
        return -(-h // rpt)
    segs = -(-w // 128)
    # two image rows of a segment per item when two 4-row windows fit
    win2 = -(-(4 * 130 * 128) // 1024) * 1024
    rows = 2 if h >= 2 and _HALO_WINDOW_BYTES // win2 >= 2 and n * -(-h // 2) * segs >= 2 * sms else 1
    return -(-h // rows) * segs


@dataclass
class CuDep:
    producer: CuStage
    consumer: CuStage
    operand: str
    policy: SyncPolicy
    sem: torch.Tensor

    @property
    def id(self) -> str:
        return f"{self.producer.id}->{self.consumer.id}/{self.operand}"


@dataclass
class CuSync:
    """A chain of dependent GeMM stages launched through libtilesync_b200.so."""

    tile_n: int = 256
    cta_group: int = 2
    mode: str = "fused"
    reorder: bool = True
    watchdog: bool = True
    keep_sems: bool = False
    num_ctas: int = 0
    extra_flags: int = 0
    swap_ab: bool = False
    row_interleave: bool = False  # claim tiles row by row across two GeMM stages
    # 2: clusters of two CTA pairs sharing the activation rows by TMA multicast; a tile
    # (256 x 512, every GeMM stage tile_n=512) runs as two 256 x 256 pair tiles with
    # double-buffered accumulators (ts_chain_desc.cluster_pairs)
    cluster_pairs: int = 1
    # co-resident mode only: the scheduling gate and the launch order (SimOptions)
    wait_kernel: str = "auto"
    adversarial: bool = False
    coresident_grid: tuple | None = None  # CTAs (pairs) per stage launch; None = per tile
    # static stream-K schedule (TS_FLAG_BALANCED): every CTA pair runs an equal K-block
    # range of each GeMM stage, tiles split across pairs are reduced by their head segment
    balanced: bool = False
    # halo-staged convolution stages (TS_FLAG_CONV_HALO: Cin = Cout = 64, cta_group 1,
    # tile_n 64): each tile's input rows + halo loaded once, tap views by descriptor offset
    conv_halo: bool = False
    device: torch.device | None = None
    stages: list[CuStage] = field(default_factory=list)
    deps: list[CuDep] = field(default_factory=list)

    def __post_init__(self) -> None:
        if self.mode not in ("fused", "stream", "coresident"):
            raise ConfigError(f"mode must be 'fused', 'stream' or 'coresident', got {self.mode!r}")
        if self.wait_kernel not in ("on", "off", "auto"):
            raise ConfigError(f"wait_kernel must be on/off/auto, got {self.wait_kernel!r}")
        if self.swap_ab:
            if self.tile_n not in (32, 64, 128, 256):
                raise ConfigError(f"swapped tile_n must be 32, 64, 128 or 256, got {self.tile_n}")
            self.cta_group = 1
        elif self.tile_n not in (64, 128, 256):
            raise ConfigError(f"tile_n must be 64, 128 or 256, got {self.tile_n}")
        if self.cta_group not in (1, 2) or (self.cta_group == 2 and self.tile_n == 64):
            raise ConfigError("cta_group must be 1 or 2 (2 needs tile_n >= 128)")
        if self.cluster_pairs not in (1, 2) or (self.cluster_pairs == 2 and (
                self.cta_group != 2 or self.tile_n != 256 or self.swap_ab)):
            raise ConfigError("cluster_pairs=2 needs cta_group=2, tile_n=256 (normal layout)")
        self._desc: _lib.ChainDesc | None = None
        self._peers: _lib.PeerDesc | None = None
        self._ar_done: torch.Tensor | None = None
        self._scratch: torch.Tensor | None = None
        self._trace: torch.Tensor | None = None
        self._trace_cap = 0
        self._streams: list | None = None

    @property
    def tile_m(self) -> int:
        """Activation rows of one tile: 128 per CTA, 256 for a CTA pair, tile_n when
        swapped."""
        return self.tile_n if self.swap_ab else BM * self.cta_group

    def _check_open(self, kind: str = "gemm") -> None:
        """Stages may not follow an all-reduce stage: it stages peer vectors in the
        operand ring, which is idle only when no GeMM item comes after it. Two-pair
        clusters run GeMM stages only."""
        if kind != "gemm" and self.cluster_pairs == 2:
            raise ConfigError(f"cluster_pairs=2 runs GeMM stages only (not {kind})")
        if len(self.stages) >= _lib.TS_MAX_STAGES:
            raise ConfigError(f"at most {_lib.TS_MAX_STAGES} stages per chain")
        if any(st.kind == "allreduce" for st in self.stages):
            raise ConfigError("the all-reduce stage must be the chain's last stage")

    @property
    def ctas_per_tile(self) -> int:
        """CTAs that compute one tile: 1, 2 (a CTA pair) or 4 (two pairs)."""
        return self.cta_group * self.cluster_pairs

    def _check_tile_n(self, tile_n: int) -> None:
        """Per-stage tile width: 0 (the chain's), or 384 / 512 (two MMAs of 192 / 256
        columns per K-block) on cta_group=2, tile_n=256 chains."""
        if tile_n not in (0, self.tile_n) and not (
                tile_n in (384, 512) and self.tile_n == 256 and self.cta_group == 2
                and not self.swap_ab):
            raise ConfigError(f"stage tile_n {tile_n} unsupported (0, {self.tile_n}, or "
                              "384 / 512 with cta_group=2, tile_n=256)")

    # -- construction ---------------------------------------------
    def stage(self, a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, epilogue: str = "none",
              order: TileOrder = RowMajor(), id: str | None = None,
              splits: int = 1, tile_n: int = 0, tail: tuple = (0, 1)) -> CuStage:
        """Add a GeMM stage. ``splits`` > 1 splits K into that many slices (the
        reference's z extent): each slice posts once, consumers wait for all of them.
        ``tile_n=512`` gives this stage double-width CTA-pair tiles (256 x 512 outputs;
        chains with ``cta_group=2, tile_n=256`` only)."""
        self._check_tile_n(tile_n)
        self._check_open()
        if self.cluster_pairs == 2 and tile_n != 512:
            raise ConfigError("cluster_pairs=2 runs tile_n=512 (256 x 512) GeMM stages")
        if epilogue not in _EPI:
            raise ConfigError(f"unknown epilogue {epilogue!r}")
        for t, name in ((a, "a"), (b, "b"), (c, "c")):
            if t.dim() != 2 or t.stride(1) != 1:
                raise ValueError(f"{name} must be a row-major 2-D tensor")
            if t.dtype not in _DT:
                raise TypeError(f"{name}: dtype {t.dtype} unsupported (fp16/bf16)")
            if not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor")
        if a.shape[1] != b.shape[1]:
            raise ValueError(f"inner dimensions differ: a {tuple(a.shape)} b {tuple(b.shape)}")
        n_out = b.shape[0] // 2 if epilogue == "swiglu" else b.shape[0]
        if c.shape[0] != a.shape[0] or c.shape[1] != n_out:
            raise ValueError(f"c must be [{a.shape[0]}, {n_out}], got {tuple(c.shape)}")
        if splits < 1:
            raise ConfigError("splits must be >= 1")
        st = CuStage(self, len(self.stages), id or f"gemm{len(self.stages) + 1}", a, b, c,
                     epilogue, order, splits, tile_n=tile_n, tail=tuple(tail))
        if tail[0] > 0:
            # last-wave balancing (extension): the last tail[0] tiles in claim order run as
            # tail[1] split-K slices; only for a stage nothing waits on (checked at build)
            tiles = st.grid.x * st.grid.y
            st.ws = torch.empty(tiles * tail[1] * self.tile_m * st.width, dtype=torch.float32,
                                device=a.device)
            st.cnt = torch.zeros(2 * tiles * self.ctas_per_tile, dtype=torch.int32,
                                 device=a.device)
        if splits > 1:
            # fp32 partials [tile][slice][tile_m rows][width] and per-(tile, CTA) arrival
            # and partial-ready counters
            tiles = st.grid.x * st.grid.y
            st.ws = torch.empty(tiles * splits * self.tile_m * st.width, dtype=torch.float32,
                                device=a.device)
            st.cnt = torch.zeros(2 * tiles * self.ctas_per_tile, dtype=torch.int32,
                                 device=a.device)
        self.stages.append(st)
        self.device = a.device
        self._desc = None
        return st

    def stage_dot(self, qkv: torch.Tensor, out: torch.Tensor, order: TileOrder = RowMajor(),
                  id: str | None = None) -> CuStage:
        """Attention's fused dot kernel: ``out`` [m, n] =
        Dropout(Softmax(XQ . XV)) . XK per 128-column head, with ``qkv`` [m, 3n] holding
        [Q heads | K heads | V heads]. Column-tile local, as its StridedSync dependency
        defines it; dropout p = 0 (inference)."""
        self._check_open("dot")
        for t, name in ((qkv, "qkv"), (out, "out")):
            if t.dim() != 2 or t.stride(1) != 1 or t.dtype not in _DT or not t.is_cuda:
                raise ValueError(f"{name} must be a row-major fp16/bf16 CUDA matrix")
        if qkv.shape[0] != out.shape[0] or qkv.shape[1] != 3 * out.shape[1]:
            raise ValueError(f"qkv must be [m, 3n] for out [m, n], got {tuple(qkv.shape)}")
        st = CuStage(self, len(self.stages), id or f"dot{len(self.stages) + 1}", qkv, qkv, out,
                     "none", order, kind="dot")
        self.stages.append(st)
        self.device = qkv.device
        self._desc = None
        return st

    def stage_conv(self, x: torch.Tensor, w: torch.Tensor, out: torch.Tensor,
                   epilogue: str = "none", order: TileOrder = RowMajor(), id: str | None = None,
                   tile_n: int = 0, splits: int = 1) -> CuStage:
        """A 3x3, stride-1, padding-1 Conv2D as an implicit GeMM (the paper's ResNet conv
        pairs): ``x`` NHWC [N, H, W, Cin], ``w`` KRSC [Cout, 3, 3, Cin],
        ``out`` NHWC [N, H, W, Cout]. Output rows are the N*H*W pixels, columns the output
        channels; the A operand is gathered by an im2col TMA map (zero padding at the
        image border). Feed it from another stage with ``Conv2DTileSync(9)``."""
        self._check_open("conv")
        if epilogue not in ("none", "relu", "gelu"):
            raise ConfigError(f"unsupported conv epilogue {epilogue!r}")
        if x.dim() != 4 or out.dim() != 4 or w.dim() != 4 or tuple(w.shape[1:3]) != (3, 3):
            raise ValueError("conv needs x [N,H,W,Cin], w [Cout,3,3,Cin], out [N,H,W,Cout]")
        for t, name in ((x, "x"), (w, "w"), (out, "out")):
            if not t.is_contiguous() or t.dtype not in _DT or not t.is_cuda:
                raise ValueError(f"{name} must be a contiguous fp16/bf16 CUDA tensor")
        n, h, wd, cin = x.shape
        if w.shape[3] != cin or tuple(out.shape) != (n, h, wd, w.shape[0]):
            raise ValueError(f"shape mismatch: x {tuple(x.shape)} w {tuple(w.shape)} "
                             f"out {tuple(out.shape)}")
        self._check_tile_n(tile_n)
        if splits < 1 or (9 * cin // BK) % splits:
            raise ConfigError(f"splits={splits} must divide the {9 * cin // BK} K-blocks")
        st = CuStage(self, len(self.stages), id or f"conv{len(self.stages) + 1}",
                     x.view(n * h * wd, cin), w.reshape(w.shape[0], 9 * cin),
                     out.view(n * h * wd, w.shape[0]), epilogue, order, splits=splits,
                     kind="conv", conv=(n, h, wd), tile_n=tile_n)
        if splits > 1:
            tiles = st.grid.x * st.grid.y
            st.ws = torch.empty(tiles * splits * self.tile_m * st.width, dtype=torch.float32,
                                device=x.device)
            st.cnt = torch.zeros(2 * tiles * self.cta_group, dtype=torch.int32, device=x.device)
        self.stages.append(st)
        self.device = x.device
        self._desc = None
        return st

    def stage_allreduce(self, producer: CuStage, id: str | None = None) -> CuStage:
        """Tensor-parallel all-reduce of ``producer``'s output, fused into the chain
        (extension; SURVEY.md §8f "next"): the producer's output buffer is summed in place
        across the group given by ``set_peers``. This rank owns the producer tiles t with
        t % world == rank; an owned tile waits for its post on every rank (system-scope
        acquire), is summed over the ranks' buffers in fp32 and stored back into all of
        them — the reduction of a row tile starts as soon as every rank has produced it,
        instead of after the whole GeMM. Adds the producer -> all-reduce TileSync
        dependency."""
        from .policies import TileSync
        if len(self.stages) >= _lib.TS_MAX_STAGES:
            raise ConfigError(f"at most {_lib.TS_MAX_STAGES} stages per chain")
        if producer.kind != "gemm" or producer.epilogue == "swiglu" or self.swap_ab:
            raise ConfigError("the all-reduce stage sums a normal-layout GeMM stage's output")
        if any(st.kind == "allreduce" for st in self.stages):
            raise ConfigError("a chain has at most one all-reduce stage")
        self._check_open("allreduce")
        c = producer.c
        st = CuStage(self, len(self.stages), id or "allreduce", c, c, c, "none", RowMajor(),
                     kind="allreduce", tile_n=producer.tile_n)
        self.stages.append(st)
        self.dependency(TileSync(), producer, st)
        self._ar_done = torch.zeros(1, dtype=torch.int32, device=c.device)
        self._desc = None
        return st

    @property
    def allreduce_done(self) -> torch.Tensor:
        """This rank's all-reduce arrival counter (epoch x tiles x cta_group after the
        epoch-th launch)."""
        return self._ar_done

    @property
    def epoch(self) -> int:
        """Launches of the all-reduce group so far (0 before the first)."""
        return 0 if self._peers is None else int(self._peers.epoch)

    def allreduce_dep(self) -> "CuDep":
        return next(d for d in self.deps if d.consumer.kind == "allreduce")

    def set_peers(self, rank: int, bufs, sems, dones) -> None:
        """The tensor-parallel group of the all-reduce stage: for every rank q, its
        buffer (the all-reduce stage's c), its producer -> all-reduce semaphores and its
        done counter, as device pointers valid in this process (ints or tensors: P2P /
        IPC-mapped / symmetric memory; on one GPU, plain tensors simulate the group)."""
        world = len(bufs)
        if not (1 <= world <= _lib.TS_MAX_PEERS) or len(sems) != world or len(dones) != world:
            raise ConfigError(f"peer lists must have 1..{_lib.TS_MAX_PEERS} equal entries")
        if not 0 <= rank < world:
            raise ConfigError(f"rank {rank} outside world {world}")
        ptr = (lambda v: v.data_ptr() if isinstance(v, torch.Tensor) else int(v))
        pd = _lib.PeerDesc()
        pd.world, pd.rank = world, rank
        for q in range(world):
            pd.bufs[q], pd.sems[q], pd.done[q] = ptr(bufs[q]), ptr(sems[q]), ptr(dones[q])
        # launch generation: the group's all-reduce semaphores and done counters are
        # monotone (zero now); every rank advances the epoch once per launch in lockstep
        pd.epoch = 0
        self._peers = pd
        self._desc = None

    def dependency(self, policy: SyncPolicy, producer: CuStage, consumer: CuStage,
                   operand: str = "a") -> CuDep:
        """cs.dependency<Policy>(prod, cons, operand) — allocates the semaphore array."""
        if len(self.deps) >= _lib.TS_MAX_DEPS:
            raise ConfigError(f"at most {_lib.TS_MAX_DEPS} dependencies per chain")
        n = sem_count(policy, producer.grid)
        sem = torch.zeros(n, dtype=torch.int32, device=producer.a.device)
        d = CuDep(producer, consumer, operand, policy, sem)
        self.deps.append(d)
        self._desc = None
        return d

    # -- reference view (for the oracle and the planner) ------------------------------
    def scenario(self, num_sms: int = 148) -> Scenario:
        """The reference Scenario this chain executes, with B200 grids."""
        in_dep = {d.consumer.index: d for d in self.deps}
        stages = []
        for st in self.stages:
            if st.kind == "allreduce":
                continue  # the collective is outside the reference model
            d = in_dep.get(st.index)
            if st.kind == "dot":
                k_steps = 1  # attention_scenario's dot stage (workloads.py:124-153)
            elif d is None:
                k_steps = max(1, st.k // st.out_tile_cols)
            else:
                k_steps = st.k // d.producer.out_tile_cols
                if isinstance(d.policy, Conv2DTileSync) and st.kind != "conv":
                    k_steps *= d.policy.kk  # a GeMM consumer splits producer tiles kk-fold
            operands = ("qkv",) if st.kind == "dot" else ("a", "b")
            stages.append(Stage(id=st.id, grid=st.grid, occupancy=1, k_steps=k_steps,
                                order=st.order, operands=operands))
        deps = tuple(Dependency(d.producer.id, d.consumer.id, d.operand, d.policy)
                     for d in self.deps if d.consumer.kind != "allreduce")
        mode = Mode.STREAM if self.mode == "stream" else Mode.FINE
        opts = SimOptions(wait_kernel=self.wait_kernel, adversarial_order=self.adversarial)
        return Scenario(gpu=GpuConfig(num_sms), stages=tuple(stages), deps=deps, mode=mode,
                        options=opts)

    # -- launch ------------------------------------------------------------------------
    def _build(self) -> _lib.ChainDesc:
        if not self.stages:
            raise ConfigError("chain has no stages")
        d = _lib.ChainDesc()
        d.n_stages = len(self.stages)
        for i, st in enumerate(self.stages):
            sd = d.stages[i]
            sd.a, sd.b, sd.c = st.a.data_ptr(), st.b.data_ptr(), st.c.data_ptr()
            sd.m, sd.n, sd.k = st.m, st.n, st.k
            sd.lda, sd.ldb, sd.ldc = st.a.stride(0), st.b.stride(0), st.c.stride(0)
            sd.dtype = _DT[st.a.dtype]
            sd.epilogue = _EPI[st.epilogue]
            sd.order, sd.order_stride = order_code(st.order)
            sd.splits = st.splits
            sd.kind = {"dot": _lib.TS_STAGE_ATTN_DOT, "conv": _lib.TS_STAGE_CONV2D,
                       "allreduce": _lib.TS_STAGE_ALLREDUCE}.get(st.kind, _lib.TS_STAGE_GEMM)
            if st.conv is not None:
                sd.conv_n, sd.conv_h, sd.conv_w = st.conv
            sd.in_sem = st.in_sem.data_ptr() if st.in_sem is not None else None
            sd.out_sem = st.out_sem.data_ptr() if st.out_sem is not None else None
            sd.tile_n = st.tile_n
            sd.tail_tiles, sd.tail_splits = st.tail
            sd.workspace = st.ws.data_ptr() if st.ws is not None else None
            sd.counters = st.cnt.data_ptr() if st.cnt is not None else None
        d.n_deps = len(self.deps)
        for i, dep in enumerate(self.deps):
            dd = d.deps[i]
            dd.producer, dd.consumer = dep.producer.index, dep.consumer.index
            if dep.operand != ("qkv" if dep.consumer.kind == "dot" else "a"):
                raise ConfigError("GeMM stages consume their producer through operand 'a', "
                                  "the dot stage through 'qkv'")
            dd.operand = 0
            dd.policy, dd.param = policy_code(dep.policy)
            dd.sem = dep.sem.data_ptr()
        d.mode = {"fused": _lib.TS_MODE_FUSED, "stream": _lib.TS_MODE_STREAM,
                  "coresident": _lib.TS_MODE_CORESIDENT}[self.mode]
        d.tile_n = self.tile_n
        d.cta_group = self.cta_group
        d.swap_ab = 1 if self.swap_ab else 0
        d.flags = ((0 if self.reorder else _lib.TS_FLAG_NO_REORDER)
                   | (0 if self.watchdog else _lib.TS_FLAG_NO_WATCHDOG)
                   | (_lib.TS_FLAG_KEEP_SEMS if self.keep_sems else 0)
                   | (_lib.TS_FLAG_ROW_INTERLEAVE if self.row_interleave else 0)
                   | self.extra_flags)
        d.num_ctas = self.num_ctas
        d.cluster_pairs = self.cluster_pairs
        if self.balanced:
            d.flags |= _lib.TS_FLAG_BALANCED
            self._balanced_buffers(d)
        if self.conv_halo:
            d.flags |= _lib.TS_FLAG_CONV_HALO
        if self._scratch is None:
            self._scratch = torch.zeros(_lib.TS_SCRATCH_INTS, dtype=torch.int32,
                                        device=self.device)
        d.scratch = self._scratch.data_ptr()
        d.trace = None
        d.trace_cap = 0
        if any(st.kind == "allreduce" for st in self.stages):
            if getattr(self, "_peers", None) is None:
                raise ConfigError("the all-reduce stage needs set_peers(...) before launch")
            d.peers = ctypes.pointer(self._peers)
        return d

    def balanced_units(self) -> int:
        """Work units (CTA pairs) of a balanced launch: one per SM pair, capped at the
        co-resident cluster count (ts_chain_units), or num_ctas / 2."""
        out = ctypes.c_int()
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().ts_chain_units(self.tile_n, self.cta_group, 1, 0,
                                                  _DT[self.stages[0].a.dtype],
                                                  ctypes.byref(out)))
        units = out.value
        if self.num_ctas:
            units = min(units, self.num_ctas // self.cta_group)
        return units

    def _balanced_buffers(self, d) -> None:
        """Per stage: fp32 partial planes [units][2 CTAs][128 rows][tile width] (one per
        unit: only a unit's first segment of a stage can start inside a tile) and one
        ready counter per tile half (zero; the head segment restores it)."""
        if self.mode != "fused" or self.cta_group != 2 or self.tile_n != 256 or self.swap_ab \
                or self.cluster_pairs != 1:
            raise ConfigError("balanced=True needs mode='fused', cta_group=2, tile_n=256, "
                              "cluster_pairs=1")
        units = self.balanced_units()
        for i, st in enumerate(self.stages):
            if st.kind != "gemm" or st.splits != 1 or st.tail[0] or st.epilogue == "swiglu":
                raise ConfigError(f"stage {st.id}: the balanced schedule takes unsplit GeMM "
                                  "stages (no tail, no SwiGLU)")
            need = units * 2 * BM * st.width
            if st.ws is None or st.ws.numel() < need:
                st.ws = torch.empty(need, dtype=torch.float32, device=st.a.device)
                st.cnt = torch.zeros(2 * st.grid.x * st.grid.y, dtype=torch.int32,
                                     device=st.a.device)
            d.stages[i].workspace = st.ws.data_ptr()
            d.stages[i].counters = st.cnt.data_ptr()

    def enable_trace(self, capacity: int | None = None) -> None:
        """Record the reference's per-block events on the device (engine.py:220-248)."""
        if capacity is None:
            capacity = 0
            for st in self.stages:
                capacity += st.grid.total() * (5 + 2 * 2 * max(1, st.k // BK))
        self._trace_cap = capacity
        self._trace = torch.zeros(capacity * _lib.TRACE_REC_BYTES, dtype=torch.uint8,
                                  device=self.device)
        self._desc = None

    def launch(self, stream: torch.cuda.Stream | None = None) -> None:
        """Enqueue the chain on `stream` (default: the current torch stream)."""
        if self._desc is None:
            self._desc = self._build()
            if self._trace is not None:
                self._desc.trace = self._trace.data_ptr()
                self._desc.trace_cap = self._trace_cap
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self._peers is not None:
            self._peers.epoch += 1  # ts_chain_launch copies the peer descriptor
        # the library launches on (and sizes the grid for) the caller's current device
        with torch.cuda.device(self.device):
            if self._trace is not None:
                self._scratch[2].zero_()
            if self.mode == "coresident":
                self._launch_coresident(s)
                return
            _lib.check(_lib.load().ts_chain_launch(ctypes.byref(self._desc),
                                                   ctypes.c_void_p(s.cuda_stream)))

    def _launch_coresident(self, s: torch.cuda.Stream) -> None:
        """One launch per stage on its own stream (stage 0 at the highest priority), the
        stage streams ordered after `s` and `s` after all of them, so consecutive chains
        never overlap (the semaphores and started flags are reset by the consumers)."""
        n = len(self.stages)
        if self._streams is None:
            lo, hi = torch.cuda.Stream.priority_range()
            self._streams = [torch.cuda.Stream(device=self.device,
                                               priority=max(hi, lo - (n - 1 - i)))
                             for i in range(n)]
        for st in self._streams:
            st.wait_stream(s)
        ptrs = (ctypes.c_void_p * n)(*[st.cuda_stream for st in self._streams])
        grid = None
        if self.coresident_grid is not None:
            grid = (ctypes.c_int * n)(*self.coresident_grid)
        gate = {"off": 0, "on": 1, "auto": 2}[self.wait_kernel]
        _lib.check(_lib.load().ts_chain_launch_coresident(
            ctypes.byref(self._desc), ptrs, n, gate, 1 if self.adversarial else 0, grid))
        for st in self._streams:
            s.wait_stream(st)

    __call__ = launch

    def set_in_expected(self, stage: CuStage, value: int) -> None:
        """Gate value for `stage`'s external row semaphores on the next launch."""
        if self._desc is None:
            self._desc = self._build()
            if self._trace is not None:
                self._desc.trace = self._trace.data_ptr()
                self._desc.trace_cap = self._trace_cap
        self._desc.stages[stage.index].in_expected = value

    # -- results -------------------------------------------------------------------------
    def watchdog_fired(self) -> bool:
        """True if a semaphore wait timed out (the device analogue of detect_deadlock,
        engine.py:614-637). Synchronizes."""
        return bool(self._scratch is not None and int(self._scratch[3].item()) != 0)

    def final_semaphores(self) -> dict[str, tuple[int, ...]]:
        """Semaphore values after a ``keep_sems=True`` launch (SimTrace.final_semaphores)."""
        return {d.id: tuple(int(v) for v in d.sem.cpu().tolist()) for d in self.deps}

    def reset_semaphores(self) -> None:
        for d in self.deps:
            d.sem.zero_()

    def trace_records(self) -> list:
        """Raw device trace records (ts_trace_rec), in recording order."""
        if self._trace is None:
            raise RuntimeError("tracing is not enabled (call enable_trace() first)")
        count = int(self._scratch[2].item())
        if count > self._trace_cap:
            raise RuntimeError("trace buffer overflowed")
        raw = self._trace[: count * _lib.TRACE_REC_BYTES].cpu().numpy().tobytes()
        return list((_lib.TraceRec * count).from_buffer_copy(raw)) if count else []

    def trace_events(self) -> list[Event]:
        """The device trace as reference Events, times in ns from the first event."""
        recs = self.trace_records()
        t0 = min((r.t_ns for r in recs), default=0)
        dep_ids = [d.id for d in self.deps]
        evs = []
        for i, r in enumerate(recs):
            if r.kind >= len(_KINDS):
                continue  # MMA-side extension records (see trace_records)
            kind = _KINDS[r.kind]
            ev = Event(time=int(r.t_ns - t0), stage=self.stages[r.stage].id, tb=r.tb, kind=kind,
                       tile=(r.x, r.y, r.z),
                       k=r.k if r.k >= 0 else None,
                       dep=dep_ids[r.dep] if r.dep >= 0 else None,
                       sem=r.sem if r.sem >= 0 else None,
                       expected=r.value if kind in ("wait_begin", "wait_end") else None,
                       value=r.value if kind == "post" else None)
            evs.append((ev.time, _RANK[kind], i, ev))
        evs.sort(key=lambda e: e[:3])
        return [e[3] for e in evs]

    def sim_trace(self) -> SimTrace:
        mode = Mode.STREAM if self.mode == "stream" else Mode.FINE
        return SimTrace(mode=mode, events=self.trace_events(),
                        final_semaphores=self.final_semaphores())

    def flops(self) -> int:
        return sum(st.flops() for st in self.stages)
