"""CPU oracle for the tile-synchronization hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference
arm may import this module, and only as the checker. The product
(``paper_2305_13450_b200``) never imports it; the device path fails loudly when its CUDA
library is missing.

What it restates (plain Python / numpy), each function citing the reference it follows
under /root/reference/pkg/src/tilesync_sim/:

* the policy layer — ``sem_count``, ``post_target``, ``consumer_wait``, ``wait_steps``,
  ``order_tile`` (policies.py:115-205);
* the brute-force dependency DAG and the trace validator (oracle.py:45-191);
* the closed-form final semaphore values (conservation, oracle.py:62-67 /
  test_engine.py:170-194);
* the numeric chains of the paper: MLP ``GeLU(X W1) W2`` and the
  SwiGLU variant, in fp32 over the same fp16/bf16-rounded inputs;
* a CPU executor of the paper's protocol (``run_chain_cpu``): producer and consumer tiles
  on a thread pool, consumers blocking on semaphores until the producer tiles they read
  have posted — the CPU path ``bench.py --impl reference`` times.

Parity status: the policy/DAG/trace functions are pinned against golden vectors produced
by the reference itself (tests/golden/make_golden.py, committed fixtures). The numerics
are *not* pinned by the reference — it has no GeMM/GeLU code — so the
numeric chain is a restatement of PAPER.md:143-165 checked against an independent
float64 evaluation in tests; see DESIGN.md "Parity".
"""

from __future__ import annotations

import hashlib
import json
import math
import threading
from collections import defaultdict
from concurrent.futures import ThreadPoolExecutor

import numpy as np

TILE, ROW, STRIDED, CONV2D = "tile", "row", "strided", "conv2d"
ROW_MAJOR, STRIDED_ROW_MAJOR = "row_major", "strided_row_major"


class OracleConfigError(ValueError):
    """Mirrors ConfigError (errors.py:4-5) without importing the product."""


# ---- policy layer (policies.py:102-205) ------------------------------------------------

def check_policy(policy, pgrid):
    """policies.py:102-112."""
    kind, param = policy
    if kind == STRIDED:
        if param < 1:
            raise OracleConfigError("stride must be >= 1")
        if pgrid[1] % param:
            raise OracleConfigError("stride does not divide producer columns")
    elif kind == CONV2D and param < 1:
        raise OracleConfigError("kk must be >= 1")


def sem_count(policy, pgrid):
    """policies.py:115-125: Tile/Conv x*y, Row x, Strided x*stride (z never counts)."""
    check_policy(policy, pgrid)
    kind, param = policy
    gx, gy = pgrid[0], pgrid[1]
    return {TILE: gx * gy, CONV2D: gx * gy, ROW: gx, STRIDED: gx * (param or 1)}[kind]


def post_target(policy, tile, pgrid):
    """policies.py:128-142 (bounds check 133-134)."""
    x, y, z = tile
    if not (0 <= x < pgrid[0] and 0 <= y < pgrid[1] and 0 <= z < pgrid[2]):
        raise ValueError("tile outside producer grid")
    kind, param = policy
    if kind in (TILE, CONV2D):
        return x * pgrid[1] + y
    if kind == ROW:
        return x
    return x * param + y % param


def consumer_wait(policy, tile, k, pgrid, pz):
    """policies.py:145-166 -> (sem, expected) or None."""
    kind, param = policy
    row, col = tile[0], tile[1]
    if kind == TILE:
        return (row * pgrid[1] + k, pz)
    if kind == ROW:
        return (row, pgrid[1] * pz) if k == 0 else None
    if kind == STRIDED:
        return (row * param + col % param, (pgrid[1] // param) * pz) if k == 0 else None
    if k % param == 0:
        return (row * pgrid[1] + k // param, pz)
    return None


def wait_steps(policy, k_steps):
    """policies.py:169-178."""
    kind, param = policy
    if kind == TILE:
        return tuple(range(k_steps))
    if kind in (ROW, STRIDED):
        return (0,)
    return tuple(range(0, k_steps, param))


def order_tile(order, grid, n):
    """policies.py:181-205: lexicographic (x, y, z), z fastest; StridedRowMajor regroups
    the column walk so columns `stride` apart come consecutively."""
    kind, stride = order
    gx, gy, gz = grid
    if not 0 <= n < gx * gy * gz:
        raise ValueError("counter outside grid")
    z, rest = n % gz, n // gz
    pos, x = rest % gy, rest // gy
    if kind == ROW_MAJOR:
        return (x, pos, z)
    if gy % stride:
        raise OracleConfigError("stride does not divide grid columns")
    group_len = gy // stride
    return (x, pos // group_len + (pos % group_len) * stride, z)


# ---- scenarios as plain dicts ------------------------------------------------------------
# stage: {"id", "grid": (x, y, z), "k_steps", "order": (kind, stride)}
# dep:   {"producer", "consumer", "operand", "policy": (kind, param)}

def final_semaphores(stages, deps):
    """Closed form of SimTrace.final_semaphores for a run without deadlock: every
    producer tile (each z-slice) posts once to post_target (engine.py:527-560)."""
    by_id = {s["id"]: s for s in stages}
    out = {}
    for d in deps:
        g = tuple(by_id[d["producer"]]["grid"])
        vals = [0] * sem_count(d["policy"], g)
        for x in range(g[0]):
            for y in range(g[1]):
                for z in range(g[2]):
                    vals[post_target(d["policy"], (x, y, z), g)] += 1
        out[dep_id(d)] = tuple(vals)
    return out


def dep_id(d):
    """Dependency.id (engine.py:107-109)."""
    return f"{d['producer']}->{d['consumer']}/{d['operand']}"


def build_dep_dag(stages, deps):
    """oracle.py:45-76: expand each wait into the full preimage of its semaphore and
    assert conservation (expected == posts that can reach the semaphore)."""
    by_id = {s["id"]: s for s in stages}
    requires = {}
    for d in deps:
        prod, cons = by_id[d["producer"]], by_id[d["consumer"]]
        pg = tuple(prod["grid"])
        pre = defaultdict(set)
        for x in range(pg[0]):
            for y in range(pg[1]):
                pre[post_target(d["policy"], (x, y, 0), pg)].add((x, y))
        for cx in range(cons["grid"][0]):
            for cy in range(cons["grid"][1]):
                for k in range(cons["k_steps"]):
                    w = consumer_wait(d["policy"], (cx, cy, 0), k, pg, pg[2])
                    if w is None:
                        continue
                    tiles = pre[w[0]]
                    if w[1] != len(tiles) * pg[2]:
                        raise AssertionError(f"conservation broken for {dep_id(d)} sem {w[0]}")
                    key = (cons["id"], cx, cy, k)
                    t, n = requires.get(key, (set(), 0))
                    t |= {(prod["id"], x, y) for x, y in tiles}
                    requires[key] = (t, n + 1)
    return {k: (frozenset(t), n) for k, (t, n) in requires.items()}


def dag_digest(dag):
    """Order-independent sha256 of a DAG (for compact golden fixtures)."""
    rows = sorted(
        [list(k), sorted(list(t) for t in v[0]), v[1]] for k, v in dag.items())
    return hashlib.sha256(json.dumps(rows).encode()).hexdigest()


def validate_trace(events, stages, deps, fine=True):
    """oracle.py:114-191 over events given as dicts with keys t, stage, tb, kind, tile,
    k, dep, sem, expected. Returns a list of (kind, stage, tile, k) violations."""
    dag = build_dep_dag(stages, deps)
    slices = {s["id"]: s["grid"][2] for s in stages}
    k_steps = {s["id"]: s["k_steps"] for s in stages}
    last = None
    counts = defaultdict(lambda: [0, 0])
    for e in events:  # _check_shape, oracle.py:92-111
        if e["stage"] not in slices:
            raise ValueError(f"unknown stage {e['stage']!r}")
        if last is not None and e["t"] < last:
            raise ValueError("trace times are not non-decreasing")
        last = e["t"]
        c = counts[(e["stage"], e["tb"])]
        if e["kind"] == "scheduled":
            c[0] += 1
        elif e["kind"] == "finished":
            c[1] += 1
    for key, (s, f) in counts.items():
        if s != 1 or f > 1:
            raise ValueError(f"block {key} has {s} scheduled and {f} finished events")
    out = []
    sems = defaultdict(int)
    for e in events:  # replay (b)
        if e["kind"] == "post":
            sems[(e["dep"], e["sem"])] += 1
        elif e["kind"] == "wait_end" and sems[(e["dep"], e["sem"])] < e["expected"]:
            out.append(("weak_semaphore", e["stage"], tuple(e["tile"]), e["k"]))
    fin_t = defaultdict(list)
    sched_t, wend_t, done, tiles = {}, {}, set(), {}
    for e in events:  # check (a)
        if e["kind"] == "finished":
            fin_t[(e["stage"], e["tile"][0], e["tile"][1])].append(e["t"])
            done.add((e["stage"], e["tb"]))
        elif e["kind"] == "scheduled":
            sched_t[(e["stage"], e["tb"])] = e["t"]
            tiles[(e["stage"], e["tb"])] = tuple(e["tile"])
        elif e["kind"] == "wait_end":
            wend_t[(e["stage"], e["tb"], e["k"])] = e["t"]
    for (stage, tb), tile in tiles.items():
        for k in range(k_steps[stage]):
            need = dag.get((stage, tile[0], tile[1], k))
            if not need:
                continue
            if fine:
                t_read = wend_t.get((stage, tb, k))
                if t_read is None:
                    if (stage, tb) in done:
                        out.append(("missing_wait", stage, tile, k))
                    continue
            else:
                t_read = sched_t[(stage, tb)]
            for ps, px, py in sorted(need[0]):
                on_time = [t for t in fin_t.get((ps, px, py), []) if t <= t_read]
                if len(on_time) < slices[ps]:
                    out.append(("missing_post", stage, tile, k))
    return out


# ---- numerics -----------------------------------------------------------

def gelu(x):
    """GeLU in GPT-3's tanh form ("gelu_new", the MLP activation of GPT-2/3):
    0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))) — the form the device epilogue
    implements (with the hardware tanh approximation; its error is far inside the
    fp16/bf16 tolerance of the parity tests)."""
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x * x * x)))


def silu(x):
    return x / (1.0 + np.exp(-x))


def round_to(x, dtype):
    """Round fp32 values to fp16 or bf16 (returned as fp32)."""
    x = np.asarray(x, dtype=np.float32)
    if dtype == "fp16":
        return x.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        u = x.view(np.uint32).astype(np.uint64)
        rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return rounded.astype(np.uint32).view(np.float32)
    return x


def mlp_chain(x, w1, w2, dtype="fp16"):
    """XW1 = GeLU(X W1^T) rounded to the storage dtype; XW12 = XW1 W2^T (fp32 result).
    Weights are [N, K] (K-major), as the device stores them."""
    h = round_to(gelu(x.astype(np.float32) @ w1.astype(np.float32).T), dtype)
    return h, h @ w2.astype(np.float32).T


def attention_dot(qkv, heads, dtype="fp16"):
    """The paper's fused dot, column-tile local as its StridedSync
    dependency defines it: per row and 128-wide head, softmax(q*v) * k (dropout p=0)."""
    m = qkv.shape[0]
    q = qkv[:, : heads * 128].reshape(m, heads, 128).astype(np.float32)
    k = qkv[:, heads * 128: 2 * heads * 128].reshape(m, heads, 128).astype(np.float32)
    v = qkv[:, 2 * heads * 128:].reshape(m, heads, 128).astype(np.float32)
    s = q * v
    s = s - s.max(axis=2, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=2, keepdims=True)
    return round_to((p * k).reshape(m, heads * 128), dtype)


def attention_chain(x, w_qkv, w2, dtype="fp16"):
    """XQKV = X Wqkv^T (rounded) -> XDot -> Y = XDot W2^T."""
    qkv = round_to(x.astype(np.float32) @ w_qkv.astype(np.float32).T, dtype)
    heads = w_qkv.shape[0] // (3 * 128)
    dot = attention_dot(qkv, heads, dtype)
    return qkv, dot, dot @ w2.astype(np.float32).T


def swiglu_chain(x, w_gate, w_up, w_down, dtype="bf16"):
    g = x.astype(np.float32) @ w_gate.astype(np.float32).T
    u = x.astype(np.float32) @ w_up.astype(np.float32).T
    h = round_to(silu(g) * u, dtype)
    return h, h @ w_down.astype(np.float32).T


def conv3x3_nhwc(x, w):
    """3x3, stride-1, padding-1 convolution as the implicit GeMM the device runs:
    x NHWC [N, H, W, C], w KRSC [Co, 3, 3, C] -> NHWC [N, H, W, Co] (fp32). The K order of
    the patch matrix is (tap r*3+s, channel), the KRSC weight row order."""
    n, h, wd, c = x.shape
    xp = np.zeros((n, h + 2, wd + 2, c), dtype=np.float32)
    xp[:, 1:h + 1, 1:wd + 1] = x
    cols = np.stack([xp[:, r:r + h, s_:s_ + wd] for r in range(3) for s_ in range(3)], axis=3)
    a = cols.reshape(n * h * wd, 9 * c)
    y = a @ w.reshape(w.shape[0], 9 * c).astype(np.float32).T
    return y.reshape(n, h, wd, w.shape[0])


def conv_chain(x, w1, w2, dtype="fp16"):
    """A ResNet conv pair: H = ReLU(conv(X, W1)) rounded to the storage
    dtype, Y = conv(H, W2) in fp32 (BatchNorm folded into the weights at inference)."""
    h = round_to(np.maximum(conv3x3_nhwc(x.astype(np.float32), w1), 0.0), dtype)
    return h, conv3x3_nhwc(h, w2)


# ---- CPU executor of the paper's protocol --------------------------------------------------

class _Sems:
    def __init__(self, n):
        self.v = [0] * n
        self.cv = threading.Condition()

    def post(self, i):
        with self.cv:
            self.v[i] += 1
            self.cv.notify_all()

    def wait(self, i, expected):
        with self.cv:
            self.cv.wait_for(lambda: self.v[i] >= expected)


def run_chain_cpu(x, w1, w2, tile_m=256, tile_n=256, policy=(ROW, 0), threads=None,
                  dtype="fp16"):
    """Execute GeMM -> GeLU -> GeMM tile by tile under `policy` on a thread pool.

    Tiles are claimed in RowMajor order from one counter (policies.py:181-205), producer
    tiles first; a consumer tile waits on consumer_wait(...) before each k-step
    (engine.py:469-514) and every producer tile posts post_target(...) when done
    (engine.py:527-560). Returns (h, y) and the final semaphore values.
    """
    m, k1 = x.shape
    n1, n2 = w1.shape[0], w2.shape[0]
    g1 = (-(-m // tile_m), n1 // tile_n, 1)
    g2 = (-(-m // tile_m), n2 // tile_n, 1)
    x32, w1t, w2t = x.astype(np.float32), w1.astype(np.float32).T, w2.astype(np.float32).T
    h = np.zeros((m, n1), np.float32)
    y = np.zeros((m, n2), np.float32)
    sems = _Sems(sem_count(policy, g1))
    k_steps = g1[1]
    items = [(0, n) for n in range(g1[0] * g1[1])] + [(1, n) for n in range(g2[0] * g2[1])]

    def run(item):
        s, n = item
        if s == 0:
            tx, ty, _ = order_tile((ROW_MAJOR, 1), g1, n)
            r, c = slice(tx * tile_m, (tx + 1) * tile_m), slice(ty * tile_n, (ty + 1) * tile_n)
            h[r, c] = round_to(gelu(x32[r] @ w1t[:, c]), dtype)
            sems.post(post_target(policy, (tx, ty, 0), g1))
            return
        tx, ty, _ = order_tile((ROW_MAJOR, 1), g2, n)
        r, c = slice(tx * tile_m, (tx + 1) * tile_m), slice(ty * tile_n, (ty + 1) * tile_n)
        acc = np.zeros((min(tile_m, m - tx * tile_m), tile_n), np.float32)
        for k in range(k_steps):
            w = consumer_wait(policy, (tx, ty, 0), k, g1, 1)
            if w is not None:
                sems.wait(*w)
            ks = slice(k * tile_n, (k + 1) * tile_n)
            acc += h[r, ks] @ w2t[ks, c]
        y[r, c] = acc

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(run, items))
    return h, y, tuple(sems.v)
