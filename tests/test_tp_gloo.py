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


def _run_world2(target):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return err


def _attention_worker(rank, world, port, out):
    """Megatron attention: QKV split by heads (each rank keeps [Q_r | K_r | V_r]), the
    out-projection row-parallel, one all-reduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_13450_b200.tp import TPAttention, shard_attention
    g = torch.Generator().manual_seed(1)
    heads, hd = 4, 64
    x = torch.randn(16, hd, generator=g)
    wqkv = torch.randn(3 * heads * 128, hd, generator=g) / 8
    w2 = torch.randn(hd, heads * 128, generator=g) / 23
    wq_s, w2_s = shard_attention(wqkv, w2, rank, world)
    assert wq_s.shape == (3 * heads * 128 // world, hd) and w2_s.shape == (hd, heads * 128 // world)

    def local():
        _, _, y = O.attention_chain(x.numpy(), wq_s.numpy(), w2_s.numpy(), dtype="fp32")
        return torch.from_numpy(np.ascontiguousarray(y))

    y = TPAttention(x, wq_s, w2_s, local=local)()
    if rank == 0:
        _, _, ref = O.attention_chain(x.numpy(), wqkv.numpy(), w2.numpy(), dtype="fp32")
        out.put(float(np.abs(y.numpy() - ref).max()))
    dist.barrier()
    dist.destroy_process_group()


def _swiglu_worker(rank, world, port, out):
    """Megatron SwiGLU: gate/up column-parallel (interleaved per tile on each rank), down
    row-parallel, one all-reduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_13450_b200.chains import interleave_gate_up
    from paper_2305_13450_b200.tp import TPSwiglu, shard_swiglu
    g = torch.Generator().manual_seed(2)
    hd, f, tile = 64, 512, 256
    x = torch.randn(8, hd, generator=g)
    wg = torch.randn(f, hd, generator=g) / 8
    wu = torch.randn(f, hd, generator=g) / 8
    wd = torch.randn(hd, f, generator=g) / 22
    wgu_s, wd_s = shard_swiglu(wg, wu, wd, rank, world, tile_n=tile)
    (g_s, u_s), wd_s2 = shard_swiglu(wg, wu, wd, rank, world, tile_n=None)
    assert torch.equal(wgu_s, interleave_gate_up(g_s, u_s, tile)) and torch.equal(wd_s, wd_s2)

    def local():
        _, y = O.swiglu_chain(x.numpy(), g_s.numpy(), u_s.numpy(), wd_s.numpy(), dtype="fp32")
        return torch.from_numpy(np.ascontiguousarray(y))

    y = TPSwiglu(x, wgu_s, wd_s, local=local)()
    if rank == 0:
        _, ref = O.swiglu_chain(x.numpy(), wg.numpy(), wu.numpy(), wd.numpy(), dtype="fp32")
        out.put(float(np.abs(y.numpy() - ref).max()))
    dist.barrier()
    dist.destroy_process_group()


def test_tp_attention_allreduce_matches_unsharded():
    assert _run_world2(_attention_worker) < 1e-4


def test_tp_swiglu_allreduce_matches_unsharded():
    assert _run_world2(_swiglu_worker) < 1e-4


def test_shard_attention_layout():
    """Rank r's QKV shard is [Q heads of r | K heads of r | V heads of r]."""
    from paper_2305_13450_b200.tp import shard_attention
    heads, hd = 8, 4
    w = torch.arange(3 * heads * 128, dtype=torch.float32)[:, None].expand(-1, hd).contiguous()
    w2 = torch.arange(heads * 128, dtype=torch.float32)[None, :].expand(hd, -1).contiguous()
    for world in (1, 2, 4, 8):
        per = heads // world
        for r in range(world):
            q, o = shard_attention(w, w2, r, world)
            rows = q[:, 0].long().tolist()
            want = [t * heads * 128 + r * per * 128 + i for t in range(3) for i in range(per * 128)]
            assert rows == want
            assert o[0].long().tolist() == list(range(r * per * 128, (r + 1) * per * 128))
    import pytest
    with pytest.raises(ValueError):
        shard_attention(w, w2, 0, 3)
