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

from .chains import MlpChain
from .policies import RowSync, SyncPolicy


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


class TPMlp:
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

    def __call__(self) -> torch.Tensor:
        y = self.local()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y
