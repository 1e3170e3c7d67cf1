"""Megatron tensor parallelism for the dependent-GeMM chains.

The paper's shapes are the TP=8 shard of GPT-3 145B: W1 is split by
columns (each rank owns FFN/world rows of the [FFN, H] weight and computes its slice of
GeLU(X W1)), W2 by rows (each rank owns the matching FFN/world columns of [H, FFN]).
Each rank runs its own fused chain with its own semaphores — there is no cross-rank
synchronization inside the chain — and the single exchange is an all-reduce(sum) of the
partial outputs Y[B, H] (NCCL over NVLink/NVSwitch on B200).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .chains import AttentionChain, MlpChain, SwigluChain, interleave_gate_up
from .policies import RowSync, SyncPolicy, TileSync

HEAD_DIM = 128  # GPT-3 head width


def shard_rows(w: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Rows [rank*n/world, (rank+1)*n/world) of a [n, k] weight (column-parallel)."""
    n = w.shape[0]
    if n % world:
        raise ValueError(f"{n} rows do not split over {world} ranks")
    per = n // world
    return w[rank * per:(rank + 1) * per].contiguous()


def shard_cols(w: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Columns [rank*k/world, (rank+1)*k/world) of a [n, k] weight (row-parallel)."""
    k = w.shape[1]
    if k % world:
        raise ValueError(f"{k} columns do not split over {world} ranks")
    per = k // world
    return w[:, rank * per:(rank + 1) * per].contiguous()


def shard_mlp(w1: torch.Tensor, w2: torch.Tensor, rank: int, world: int):
    """(W1 shard [FFN/world, H], W2 shard [H, FFN/world]) for Megatron TP."""
    return shard_rows(w1, rank, world), shard_cols(w2, rank, world)


def shard_attention(w_qkv: torch.Tensor, w2: torch.Tensor, rank: int, world: int,
                    head_dim: int = HEAD_DIM):
    """Megatron attention shard: this rank's heads of Q, K and V (column-parallel QKV)
    and the matching input columns of the output projection (row-parallel).

    ``w_qkv`` is [3 * heads * head_dim, H] laid out [Q h0..h(n-1) | K ... | V ...] as the
    chain reads it (the StridedSync stride is the per-rank head count,
    reference workloads.py:112-114); the shard keeps that layout over the rank's heads
    [rank * heads/world, (rank+1) * heads/world). ``w2`` is [H, heads * head_dim]."""
    n3, hdim = w_qkv.shape
    if n3 % (3 * head_dim):
        raise ValueError(f"QKV rows {n3} are not 3 x heads x {head_dim}")
    heads = n3 // (3 * head_dim)
    if heads % world:
        raise ValueError(f"{heads} heads do not split over {world} ranks")
    if w2.shape[1] != heads * head_dim:
        raise ValueError(f"output projection has {w2.shape[1]} input columns, "
                         f"expected {heads * head_dim}")
    per = heads // world
    lo, hi = rank * per * head_dim, (rank + 1) * per * head_dim
    qkv = w_qkv.reshape(3, heads * head_dim, hdim)[:, lo:hi].reshape(3 * (hi - lo), hdim)
    return qkv.contiguous(), w2[:, lo:hi].contiguous()


def shard_swiglu(w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor, rank: int,
                 world: int, tile_n: int | None = 256):
    """Megatron SwiGLU shard: this rank's rows of the gate and up projections
    (column-parallel), packed gate/up-interleaved per ``tile_n`` rows so one producer tile's
    accumulator holds matching gate and up columns (``interleave_gate_up``; ``tile_n=None``
    returns the two shards unpacked), and the matching input columns of the down
    projection (row-parallel). Returns (gate_up [2F/world, H] or (gate, up),
    down [H, F/world])."""
    g, u = shard_rows(w_gate, rank, world), shard_rows(w_up, rank, world)
    d = shard_cols(w_down, rank, world)
    if tile_n is None:
        return (g, u), d
    return interleave_gate_up(g, u, tile_n), d


class _TPBase:
    """Local chain -> all-reduce(sum) of the row-parallel output over the group."""

    group = None
    local: Callable[[], torch.Tensor]

    def __call__(self) -> torch.Tensor:
        y = self.local()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y


class TPAttention(_TPBase):
    """One rank of a tensor-parallel GPT-3 attention block: the rank's
    heads through QKV GeMM -> softmax-dot -> output GeMM as one fused chain
    (``AttentionChain``: StridedSync(heads per rank) then ``second_policy``), then the
    single all-reduce(sum) of Y[S, H]. Takes the rank's shards (``shard_attention``);
    `local` is injectable for CPU (gloo) tests."""

    def __init__(self, x: torch.Tensor, w_qkv_shard: torch.Tensor, w2_shard: torch.Tensor,
                 group=None, second_policy: SyncPolicy = TileSync(),
                 local: Callable[[], torch.Tensor] | None = None, **chain_kw):
        self.group = group
        if local is None:
            self.chain = AttentionChain(x, w_qkv_shard, w2_shard, second_policy=second_policy,
                                        **chain_kw)
            local = self.chain
        self.local = local


class TPSwiglu(_TPBase):
    """One rank of a tensor-parallel LLaMA SwiGLU MLP (BASELINE.json configs[3]): the
    rank's interleaved gate/up shard -> SiLU(g) * u -> down shard as one fused chain
    (``SwigluChain``), then all-reduce(sum) of Y[B, H]. Shards from ``shard_swiglu``."""

    def __init__(self, x: torch.Tensor, w_gate_up_shard: torch.Tensor,
                 w_down_shard: torch.Tensor, group=None, policy: SyncPolicy = RowSync(),
                 local: Callable[[], torch.Tensor] | None = None, **chain_kw):
        self.group = group
        if local is None:
            self.chain = SwigluChain(x, w_gate_up_shard, w_down_shard, policy=policy, **chain_kw)
            local = self.chain
        self.local = local


class TPMlp(_TPBase):
    """One rank of a tensor-parallel MLP: local fused chain, then all-reduce(sum).

    `local` computes this rank's partial output from its weight shards; it defaults to
    the device chain (MlpChain) and is injectable so the sharding and reduction logic can
    be exercised on CPU (gloo) against the oracle.
    """

    def __init__(self, x: torch.Tensor, w1_shard: torch.Tensor, w2_shard: torch.Tensor,
                 group=None, policy: SyncPolicy = RowSync(),
                 local: Callable[[], torch.Tensor] | None = None, **chain_kw):
        self.group = group
        if local is None:
            self.chain = MlpChain(x, w1_shard, w2_shard, policy=policy, **chain_kw)
            local = self.chain
        self.local = local


class FusedTPMlp:
    """One rank of a tensor-parallel MLP with the all-reduce fused into the chain
    (SURVEY.md §8f): GeMM1 -> GeLU -> GeMM2 -> all-reduce in one persistent launch. The
    all-reduce stage sums GeMM2's output tiles across the group over peer memory as soon
    as every rank has posted them (``CuSync.stage_allreduce``), so the reduction of early
    tiles overlaps the GeMMs of later ones instead of waiting for the whole chain and an
    NCCL call. Tile ownership is round-robin (tile t belongs to rank t % world).

    Peers are connected with ``connect_group`` (one process addressing every member's
    memory: a single GPU simulating the group, or one process driving P2P-enabled GPUs),
    or — one process per GPU — with ``FusedTPMlp.from_group``, which allocates the
    exchanged buffers in torch symmetric memory and rendezvouses them over the process
    group (``handles`` lists what each rank publishes).
    """

    def __init__(self, x: torch.Tensor, w1_shard: torch.Tensor, w2_shard: torch.Tensor,
                 policy: SyncPolicy = RowSync(), **chain_kw):
        self.chain = MlpChain(x, w1_shard, w2_shard, policy=policy, **chain_kw)
        self.ar = self.chain.cs.stage_allreduce(self.chain.cons)

    @property
    def y(self) -> torch.Tensor:
        return self.chain.y

    def handles(self) -> tuple[int, int, int]:
        """(buffer, semaphores, done counter) device pointers this rank publishes."""
        cs = self.chain.cs
        return (self.chain.y.data_ptr(), cs.allreduce_dep().sem.data_ptr(),
                cs.allreduce_done.data_ptr())

    def __call__(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        return self.chain(stream)

    @classmethod
    def from_group(cls, x: torch.Tensor, w1_shard: torch.Tensor, w2_shard: torch.Tensor,
                   group=None, policy: SyncPolicy = RowSync(), **chain_kw) -> "FusedTPMlp":
        """One rank of a multi-process tensor-parallel group (one process per GPU, the
        group initialised with torch.distributed): the all-reduced output Y, the
        GeMM2 -> all-reduce semaphores and the done counter are allocated in torch's
        symmetric memory and exchanged with ``rendezvous`` (CUDA IPC / cuMem handles over
        the group's store), so every rank's kernel addresses its peers' buffers directly
        over NVLink — the pointer exchange ``connect_group`` does within one process.
        Collective: every rank of `group` must call it with the same shapes."""
        import torch.distributed._symmetric_memory as symm
        self = cls(x, w1_shard, w2_shard, policy=policy, **chain_kw)
        cs = self.chain.cs
        dev = x.device
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        y = symm.empty(*self.chain.y.shape, dtype=x.dtype, device=dev)
        dep = cs.allreduce_dep()
        sem = symm.empty(dep.sem.numel(), dtype=torch.int32, device=dev)
        done = symm.empty(1, dtype=torch.int32, device=dev)
        sem.zero_()
        done.zero_()
        # the consumer GeMM writes Y and the all-reduce stage sums it in place
        self.chain.y = y
        self.chain.cons.c = y
        for st in cs.stages:
            if st.kind == "allreduce":
                st.a = st.b = st.c = y
        dep.sem = sem
        cs._ar_done = done
        handles = [symm.rendezvous(t, group if group is not None else dist.group.WORLD)
                   for t in (y, sem, done)]
        torch.cuda.synchronize(dev)
        # a tensor may sit at an offset inside its symmetric allocation: same offset on
        # every rank (collective allocation of equal shapes)
        bufs, sems, dones = ([int(p) + t.data_ptr() - int(h.buffer_ptrs[rank])
                              for p in h.buffer_ptrs]
                             for h, t in zip(handles, (y, sem, done)))
        cs.set_peers(rank, bufs, sems, dones)
        self._symm = handles  # keep the mappings alive
        if world > 1:
            dist.barrier(group)
        return self


def connect_group(members: list[FusedTPMlp]) -> None:
    """Give every member of a single-process group the others' buffers, semaphores and
    done counters (rank = list position)."""
    hs = [m.handles() for m in members]
    bufs, sems, dones = ([h[i] for h in hs] for i in range(3))
    for r, m in enumerate(members):
        m.chain.cs.set_peers(r, bufs, sems, dones)


def owned_tiles(tiles: int, rank: int, world: int) -> list[int]:
    """Producer tiles whose all-reduce rank `rank` performs (the kernel's ownership rule:
    item i of the all-reduce stage is tile i * world + rank)."""
    return list(range(rank, tiles, world))
