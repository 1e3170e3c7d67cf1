"""Tensor-parallel sharding + all-reduce on CPU with gloo, world_size 2 (the N>1 path of
bench.py without a GPU). Each rank computes its shard with the oracle's numeric chain;
the all-reduced result must equal the unsharded chain."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tilesync_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_13450_b200.tp import TPMlp, shard_mlp
    g = torch.Generator().manual_seed(0)
    x = torch.randn(8, 64, generator=g)
    w1 = torch.randn(96, 64, generator=g) / 8
    w2 = torch.randn(64, 96, generator=g) / 10
    w1s, w2s = shard_mlp(w1, w2, rank, world)
    assert w1s.shape == (96 // world, 64) and w2s.shape == (64, 96 // world)

    def local():
        _, y = O.mlp_chain(x.numpy(), w1s.numpy(), w2s.numpy(), dtype="fp32")
        return torch.from_numpy(np.ascontiguousarray(y))

    y = TPMlp(x, w1s, w2s, local=local)()
    if rank == 0:
        _, ref = O.mlp_chain(x.numpy(), w1.numpy(), w2.numpy(), dtype="fp32")
        out.put(float(np.abs(y.numpy() - ref).max()))
    dist.barrier()
    dist.destroy_process_group()


def test_tp_mlp_allreduce_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-4


def test_shard_shapes_and_errors():
    from paper_2305_13450_b200.tp import shard_cols, shard_rows
    w = torch.arange(24.0).reshape(6, 4)
    assert torch.equal(shard_rows(w, 1, 3), w[2:4])
    assert torch.equal(shard_cols(w, 1, 2), w[:, 2:4])
    try:
        shard_rows(w, 0, 4)
    except ValueError:
        pass
    else:
        raise AssertionError("expected ValueError")


def test_allreduce_ownership_rule():
    """The fused all-reduce stage's ownership (item i of rank r = tile i * world + r):
    every producer tile is reduced by exactly one rank."""
    from paper_2305_13450_b200 import tp
    for tiles in (1, 7, 48, 96):
        for world in (1, 2, 3, 8):
            owned = [t for r in range(world) for t in tp.owned_tiles(tiles, r, world)]
            assert sorted(owned) == list(range(tiles))
