"""The fused all-reduce stage wired through torch symmetric memory (FusedTPMlp.from_group):
one process per GPU, the exchanged buffers rendezvoused over a process group. On the 1-GPU
box the group has one rank (the exchange, the epoch protocol and the kernel path run; the
sum is the identity); the same code runs per rank on an NVLink node."""

import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = textwrap.dedent('''
    import os, sys, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["REPO"])
    import paper_2305_13450_b200 as ts
    from paper_2305_13450_b200.tp import FusedTPMlp
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    g = torch.Generator().manual_seed(5)
    x = torch.randn(512, 2048, generator=g).half().cuda()
    w1 = (torch.randn(2048, 2048, generator=g) / 45).half().cuda()
    w2 = (torch.randn(2048, 2048, generator=g) / 45).half().cuda()
    ref = ts.MlpChain(x, w1, w2, policy=ts.RowSync())().clone()
    m = FusedTPMlp.from_group(x, w1, w2)
    for i in range(3):
        y = m()
        torch.cuda.synchronize()
        assert torch.equal(y, ref), (y.float() - ref.float()).abs().max()
    assert not m.chain.cs.watchdog_fired()
    assert int(m.chain.cs.allreduce_done.item()) == 3 * m.chain.cons.grid.x * m.chain.cons.grid.y * 2
    dist.destroy_process_group()
    print("symm ok")
''')


def test_from_group_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
               REPO=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "symm ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
