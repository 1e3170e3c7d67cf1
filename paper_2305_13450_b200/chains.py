"""The paper's dependent-kernel chains as ready-made CuSync builders.

* GPT-3 MLP: ``XW1 = GeLU(X @ W1)``, ``XW12 = XW1 @ W2`` — two
  dependent GeMMs, RowSync or TileSync.
* LLaMA-style SwiGLU MLP (BASELINE.json configs[3]): ``H = SiLU(X Wg) * (X Wu)``,
  ``Y = H Wd`` with gate/up columns interleaved per tile so one tile's accumulator holds
  matching gate and up columns (``interleave_gate_up``).

Weights are stored K-major, i.e. ``W1`` as ``[N, K]`` (nn.Linear layout): the chain
computes ``A @ W^T``.
"""

from __future__ import annotations

import ctypes

import torch

from .cusync import CuSync
from .policies import RowMajor, RowSync, SyncPolicy, TileOrder


class MlpChain:
    """GeMM -> GeLU -> GeMM with a reusable CuSync (semaphores, scratch, descriptor)."""

    def __init__(self, x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor,
                 policy: SyncPolicy = RowSync(), mode: str = "fused", tile_n: int = 256,
                 reorder: bool = True, keep_sems: bool = False, num_ctas: int = 0,
                 extra_flags: int = 0, cta_group: int = 2, prod_order: TileOrder = RowMajor(),
                 cons_order: TileOrder = RowMajor(), swap_ab: bool = False,
                 prod_splits: int = 1, cons_splits: int = 1, prod_tile_n: int = 0,
                 cons_tile_n: int = 0, row_interleave: bool = False,
                 cons_tail: tuple = (0, 1), cluster_pairs: int = 1, balanced: bool = False):
        """``row_interleave`` claims GeMM1 row r, GeMM2 row r, GeMM1 row r+1, ... (fused
        RowSync/TileSync, RowMajor orders): for inputs that arrive row by row
        (``run_host``), a row's GeMM2 tiles are not queued behind later rows' GeMM1 tiles
        that still wait for their copy. ``balanced`` runs both GeMMs on the static
        stream-K schedule (TS_FLAG_BALANCED; CTA-pair 256-wide tiles)."""
        m = x.shape[0]
        self.x, self.w1, self.w2 = x, w1, w2
        self.h = torch.empty(m, w1.shape[0], dtype=x.dtype, device=x.device)
        self.y = torch.empty(m, w2.shape[0], dtype=x.dtype, device=x.device)
        self.cs = CuSync(tile_n=tile_n, mode=mode, reorder=reorder, keep_sems=keep_sems,
                         num_ctas=num_ctas, extra_flags=extra_flags, cta_group=cta_group,
                         swap_ab=swap_ab, row_interleave=row_interleave,
                         cluster_pairs=cluster_pairs, balanced=balanced)
        self.prod = self.cs.stage(x, w1, self.h, epilogue="gelu", order=prod_order, id="gemm1",
                                  splits=prod_splits, tile_n=prod_tile_n)
        self.cons = self.cs.stage(self.h, w2, self.y, order=cons_order, id="gemm2",
                                  splits=cons_splits, tile_n=cons_tile_n, tail=cons_tail)
        self.dep = self.cs.dependency(policy, self.prod, self.cons, operand="a")

    def __call__(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        self.cs.launch(stream)
        return self.y

    def run_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """End to end from pinned host memory: X row tiles are copied in on one stream,
        each chunk signalling a row semaphore (ts_stream_signal) that GeMM1's tiles of that
        row wait on; Y row tiles are copied out on another stream as soon as every GeMM2
        tile of the row has stored (ts_stream_wait on the row's counter). The paper's
        tile-level producer -> consumer signalling, with the copy engines as producer
        and consumer, so both PCIe directions overlap the chain."""
        from . import _lib
        lib = _lib.load()
        rows = self.cs.tile_m  # one semaphore per activation-row tile
        m = self.x.shape[0]
        chunks = -(-m // rows)
        if getattr(self, "_in_sem", None) is None:
            dev = self.x.device
            self._in_sem = torch.zeros(chunks, dtype=torch.int32, device=dev)
            self._out_sem = torch.zeros(chunks, dtype=torch.int32, device=dev)
            self.prod.in_sem, self.cons.out_sem = self._in_sem, self._out_sem
            self.cs._desc = None
            self._epoch = 0
            self._s_in, self._s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self._epoch += 1
        per_row = self.cons.grid.y * self.cons.splits  # out_sem increments per row per launch
        cur = torch.cuda.current_stream(self.x.device)
        self._s_in.wait_stream(cur)   # the previous launch no longer reads X ...
        self._s_out.wait_stream(cur)  # ... nor writes Y
        with torch.cuda.stream(self._s_in):
            for c in range(chunks):
                r = slice(c * rows, min(m, (c + 1) * rows))
                self.x[r].copy_(x_host[r], non_blocking=True)
                _lib.check(lib.ts_stream_signal(ctypes.c_void_p(self._in_sem[c:].data_ptr()),
                                                self._epoch,
                                                ctypes.c_void_p(self._s_in.cuda_stream)))
        self.cs.set_in_expected(self.prod, self._epoch)
        self.cs.launch(cur)
        with torch.cuda.stream(self._s_out):
            for c in range(chunks):
                r = slice(c * rows, min(m, (c + 1) * rows))
                _lib.check(lib.ts_stream_wait(ctypes.c_void_p(self._out_sem[c:].data_ptr()),
                                              self._epoch * per_row,
                                              ctypes.c_void_p(self._s_out.cuda_stream)))
                y_host[r].copy_(self.y[r], non_blocking=True)
        cur.wait_stream(self._s_in)
        cur.wait_stream(self._s_out)
        return y_host


def mlp(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, policy: SyncPolicy = RowSync(),
        mode: str = "fused", tile_n: int = 256) -> torch.Tensor:
    """One-shot GPT-3 MLP: ``GeLU(x @ w1^T) @ w2^T`` on the B200 chain kernel."""
    return MlpChain(x, w1, w2, policy, mode, tile_n)()


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, tile_n: int) -> torch.Tensor:
    """Pack [F, K] gate and up weights into [2F, K] so every tile_n-row block holds
    tile_n/2 gate rows followed by the matching tile_n/2 up rows."""
    f, k = w_gate.shape
    half = tile_n // 2
    if f % half:
        raise ValueError(f"F={f} must be a multiple of tile_n/2={half}")
    g = w_gate.reshape(f // half, half, k)
    u = w_up.reshape(f // half, half, k)
    return torch.cat([g, u], dim=1).reshape(2 * f, k).contiguous()


class SwigluChain:
    """GeMM(gate|up) -> SwiGLU -> GeMM(down)."""

    def __init__(self, x: torch.Tensor, w_gate_up: torch.Tensor, w_down: torch.Tensor,
                 policy: SyncPolicy = RowSync(), mode: str = "fused", tile_n: int = 256,
                 reorder: bool = True, keep_sems: bool = False, num_ctas: int = 0,
                 cta_group: int = 2, prod_tile_n: int = 0, cons_tile_n: int = 0,
                 cluster_pairs: int = 1, prod_splits: int = 1, cons_splits: int = 1,
                 extra_flags: int = 0):
        """``prod_tile_n`` = 512 packs gate/up per 512-row block
        (``interleave_gate_up(wg, wu, 512)``); with ``cluster_pairs=2`` each pair holds
        256 accumulator columns, so gate/up are packed per 256 rows
        (``interleave_gate_up(wg, wu, 256)``) and both stages use tile_n=512."""
        m = x.shape[0]
        f = w_gate_up.shape[0] // 2
        self.h = torch.empty(m, f, dtype=x.dtype, device=x.device)
        self.y = torch.empty(m, w_down.shape[0], dtype=x.dtype, device=x.device)
        self.cs = CuSync(tile_n=tile_n, mode=mode, reorder=reorder, keep_sems=keep_sems,
                         num_ctas=num_ctas, cta_group=cta_group, cluster_pairs=cluster_pairs,
                         extra_flags=extra_flags)
        # (split-K under SwiGLU: the tensor-core reduction, extra_flags |= 1 << 27)
        self.prod = self.cs.stage(x, w_gate_up, self.h, epilogue="swiglu", id="gate_up",
                                  tile_n=prod_tile_n, splits=prod_splits)
        self.cons = self.cs.stage(self.h, w_down, self.y, id="down", tile_n=cons_tile_n,
                                  splits=cons_splits)
        self.dep = self.cs.dependency(policy, self.prod, self.cons, operand="a")

    def __call__(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        self.cs.launch(stream)
        return self.y


class AttentionChain:
    """GPT-3 self-attention block of the paper, TP-sharded:
    XQKV = X @ Wqkv^T -> XDot = Dropout(Softmax(XQ . XV)) . XK -> Y = XDot @ W2^T.

    Wqkv rows are [Q heads | K heads | V heads] with 128-wide heads (12 heads per rank
    at TP=8). The QKV GeMM draws its tiles in StridedRowMajor(heads) order so the three
    tiles of one head finish together (the paper's prodOrder); the dot
    waits on StridedSync(heads) (one semaphore per row and head, expected 3); the output
    GeMM consumes the dot's head tiles under `second_policy` (TileSync in the paper).
    """

    def __init__(self, x: torch.Tensor, w_qkv: torch.Tensor, w2: torch.Tensor,
                 second_policy: SyncPolicy | None = None, mode: str = "fused",
                 cta_group: int = 2, keep_sems: bool = False, num_ctas: int = 0,
                 extra_flags: int = 0, tile_n: int = 256, qkv_splits: int = 1,
                 out_splits: int = 1, out_tile_n: int = 0):
        """``qkv_splits`` / ``out_splits`` > 1 split the GeMMs' K into reference z-slices
        (each posts once; StridedSync/TileSync expect x z) — the QKV GeMM of a short
        sequence has too few output tiles to fill 148 SMs otherwise."""
        from .policies import StridedRowMajor, StridedSync, TileSync
        m = x.shape[0]
        n3 = w_qkv.shape[0]
        if n3 % (3 * tile_n):
            raise ValueError(f"Wqkv rows must be 3 x (a multiple of tile_n={tile_n})")
        self.heads = n3 // (3 * 128)
        # column tiles per Q/K/V third = the StridedSync stride H / (8 Ty)
        stride = n3 // (3 * tile_n)
        self.qkv = torch.empty(m, n3, dtype=x.dtype, device=x.device)
        self.dot = torch.empty(m, n3 // 3, dtype=x.dtype, device=x.device)
        self.y = torch.empty(m, w2.shape[0], dtype=x.dtype, device=x.device)
        self.cs = CuSync(tile_n=tile_n, mode=mode, cta_group=cta_group, keep_sems=keep_sems,
                         num_ctas=num_ctas, extra_flags=extra_flags)
        self.s_qkv = self.cs.stage(x, w_qkv, self.qkv, order=StridedRowMajor(stride), id="qkv",
                                   splits=qkv_splits)
        self.s_dot = self.cs.stage_dot(self.qkv, self.dot, id="dot")
        self.s_out = self.cs.stage(self.dot, w2, self.y, id="out", splits=out_splits,
                                   tile_n=out_tile_n)
        self.cs.dependency(StridedSync(stride), self.s_qkv, self.s_dot, operand="qkv")
        self.cs.dependency(second_policy or TileSync(), self.s_dot, self.s_out, operand="a")

    def __call__(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        self.cs.launch(stream)
        return self.y


class ConvChain:
    """A ResNet conv pair: ``H = ReLU(conv3x3(X, W1))``,
    ``Y = conv3x3(H, W2)``, NHWC activations and KRSC weights (BatchNorm folded into the
    weights at inference), synchronized with Conv2DTileSync(9): the
    second convolution's k-step (input-channel tile, tap) waits for the producer tile that
    wrote that channel tile of its rows (plus, untraced, the neighbouring row tiles its
    3x3 window reaches)."""

    def __init__(self, x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor,
                 policy: SyncPolicy | None = None, mode: str = "fused", tile_n: int = 128,
                 cta_group: int = 1, keep_sems: bool = False, num_ctas: int = 0,
                 extra_flags: int = 0, prod_order: TileOrder = RowMajor(),
                 cons_order: TileOrder = RowMajor(), act: str = "relu", prod_splits: int = 1,
                 cons_splits: int = 1, halo: bool = False):
        """``halo=True`` (64-channel layers, tile_n=64, cta_group=1): each tile's input
        rows + halo are staged once and the nine taps read shifted views of them
        (TS_FLAG_CONV_HALO)."""
        from .policies import Conv2DTileSync
        n, h, w, _ = x.shape
        self.x, self.w1, self.w2 = x, w1, w2
        self.h = torch.empty(n, h, w, w1.shape[0], dtype=x.dtype, device=x.device)
        self.y = torch.empty(n, h, w, w2.shape[0], dtype=x.dtype, device=x.device)
        self.cs = CuSync(tile_n=tile_n, mode=mode, keep_sems=keep_sems, num_ctas=num_ctas,
                         cta_group=cta_group, extra_flags=extra_flags, conv_halo=halo)
        self.prod = self.cs.stage_conv(x, w1, self.h, epilogue=act, order=prod_order, id="conv1",
                                       splits=prod_splits)
        self.cons = self.cs.stage_conv(self.h, w2, self.y, order=cons_order, id="conv2",
                                       splits=cons_splits)
        self.dep = self.cs.dependency(policy or Conv2DTileSync(9), self.prod, self.cons,
                                      operand="a")

    def __call__(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        self.cs.launch(stream)
        return self.y
