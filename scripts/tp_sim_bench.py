"""Simulated tensor-parallel group on one B200 (each rank = one chain on 1/world of the SMs,
own stream): GPT-3 MLP shard chains with the all-reduce fused in (FusedTPMlp) vs the same
chains followed by a separate device sum into every rank's buffer (what a non-fused
all-reduce does, without NCCL's transport). argv: B world"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_13450_b200 as ts  # noqa: E402
from paper_2305_13450_b200 import tp  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
H, FFN = 12288, 6144
torch.manual_seed(0)
x = torch.randn(b, H, device="cuda").half()
sms = torch.cuda.get_device_properties(0).multi_processor_count
ctas = (sms // world) // 2 * 2
kw = dict(tile_n=256, cta_group=2, prod_tile_n=512, cons_tile_n=512, num_ctas=ctas)
w1 = [(torch.randn(FFN // world, H, device="cuda") / H ** 0.5).half() for _ in range(world)]
w2 = [(torch.randn(H, FFN // world, device="cuda") / FFN ** 0.5).half() for _ in range(world)]
fused = [tp.FusedTPMlp(x, w1[r], w2[r], **kw) for r in range(world)]
tp.connect_group(fused)
plain = [ts.MlpChain(x, w1[r], w2[r], **kw) for r in range(world)]
streams = [torch.cuda.Stream() for _ in range(world)]


def run(chains, reduce):
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for c, s in zip(chains, streams):
        c(s)
    for s in streams:
        cur.wait_stream(s)
    if reduce:
        tot = sum(c.y.float() for c in chains).half()
        for c in chains:
            c.y.copy_(tot)


def time_it(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


tf = time_it(lambda: run(fused, False))
tn = time_it(lambda: run(plain, False))
tr = time_it(lambda: run(plain, True))
assert not any(f.chain.cs.watchdog_fired() for f in fused)
print(f"B={b} world={world} ({ctas} CTAs per rank): fused chain+all-reduce {tf:.1f} us, "
      f"chains alone {tn:.1f} us, chains + separate sum {tr:.1f} us")
