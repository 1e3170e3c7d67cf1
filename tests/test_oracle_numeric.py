"""The oracle's numeric chain and its CPU protocol executor (test infrastructure).

The reference has no numeric code, so the numeric restatement of
PAPER.md:143-165 is cross-checked here against an independent float64 evaluation, and
the CPU executor of the protocol against the plain chain and the closed-form final
semaphores."""

import math

import numpy as np
import pytest

from oracle import tilesync_oracle as O


def f64_mlp(x, w1, w2, dtype):
    h = x.astype(np.float64) @ w1.astype(np.float64).T
    h = 0.5 * h * (1 + np.tanh(math.sqrt(2 / math.pi) * (h + 0.044715 * h ** 3)))
    h = O.round_to(h.astype(np.float32), dtype).astype(np.float64)
    return h, h @ w2.astype(np.float64).T


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_mlp_chain_matches_float64(dtype):
    rng = np.random.default_rng(0)
    x = O.round_to(rng.standard_normal((40, 96), dtype=np.float32), dtype)
    w1 = O.round_to(rng.standard_normal((64, 96), dtype=np.float32) / 10, dtype)
    w2 = O.round_to(rng.standard_normal((32, 64), dtype=np.float32) / 8, dtype)
    h, y = O.mlp_chain(x, w1, w2, dtype)
    h64, y64 = f64_mlp(x, w1, w2, dtype)
    # h is rounded to the storage dtype: allow one ulp flips from fp32 vs fp64 rounding
    ulp = 2 ** -10 if dtype == "fp16" else 2 ** -7
    assert np.all(np.abs(h - h64) <= ulp * np.maximum(np.abs(h64), 1e-3) + 1e-6)
    assert np.allclose(y, y64, rtol=1e-3, atol=1e-3)


def test_round_to_bf16_is_round_nearest_even():
    v = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e38], dtype=np.float32)
    r = O.round_to(v, "bf16")
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.015625 and r[3] == -2.5


@pytest.mark.parametrize("policy", [(O.ROW, 0), (O.TILE, 0), (O.CONV2D, 1)])
def test_cpu_protocol_executor(policy):
    rng = np.random.default_rng(1)
    m, k, n1, n2 = 300, 128, 256, 192
    x = O.round_to(rng.standard_normal((m, k), dtype=np.float32), "fp16")
    w1 = O.round_to(rng.standard_normal((n1, k), dtype=np.float32) / 11, "fp16")
    w2 = O.round_to(rng.standard_normal((n2, n1), dtype=np.float32) / 16, "fp16")
    h, y, sems = O.run_chain_cpu(x, w1, w2, tile_m=128, tile_n=64, policy=policy, threads=4)
    h_ref, y_ref = O.mlp_chain(x, w1, w2, "fp16")
    assert np.array_equal(h, h_ref)
    assert np.allclose(y, y_ref, rtol=1e-4, atol=1e-4)
    g1 = (3, 4, 1)
    stages = [{"id": "p", "grid": g1, "k_steps": 4, "order": (O.ROW_MAJOR, 1)},
              {"id": "c", "grid": (3, 3, 1), "k_steps": 4, "order": (O.ROW_MAJOR, 1)}]
    deps = [{"producer": "p", "consumer": "c", "operand": "a", "policy": policy}]
    assert sems == O.final_semaphores(stages, deps)["p->c/a"]


def test_conv3x3_matches_torch_float64():
    """The implicit-GeMM conv restatement against torch's direct conv2d in float64."""
    import torch
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 7, 9, 16)).astype(np.float32)
    w = rng.standard_normal((24, 3, 3, 16)).astype(np.float32)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double().permute(0, 3, 1, 2),
                                     torch.from_numpy(w).double().permute(0, 3, 1, 2),
                                     padding=1).permute(0, 2, 3, 1).numpy()
    got = O.conv3x3_nhwc(x, w)
    assert np.abs(got - ref).max() < 1e-3 * np.abs(ref).max()


def test_conv_chain_relu_and_rounding():
    rng = np.random.default_rng(4)
    x = O.round_to(rng.standard_normal((1, 5, 6, 8)).astype(np.float32), "fp16")
    w1 = O.round_to(rng.standard_normal((8, 3, 3, 8)).astype(np.float32) / 8, "fp16")
    w2 = O.round_to(rng.standard_normal((4, 3, 3, 8)).astype(np.float32) / 8, "fp16")
    h, y = O.conv_chain(x, w1, w2, "fp16")
    assert (h >= 0).all() and np.array_equal(h, O.round_to(h, "fp16"))
    assert np.allclose(y, O.conv3x3_nhwc(h, w2))
