"""Times the reference simulator's simulate() (SURVEY.md §8(d) CPU baseline 1) on the
B200-grid scenario of the shipped B=1024 plan — build container only (/root/reference does
not exist on the GPU box), single-threaded (the simulator holds the GIL).

    python scripts/time_reference_simulate.py > profiles/r02qq_reference_simulate.txt
"""
import os
import platform
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import tilesync_sim as r  # noqa: E402  (the reference, read-only)


def scenario(pol, z1, gx=4, n1=12, n2=24, k1=24, k2=12):
    """GPT-3 MLP shard B=1024 on B200 grids: 256x512 CTA-pair tiles, 74 pairs."""
    return r.Scenario(
        gpu=r.GpuConfig(74),
        stages=(r.Stage("gemm1", r.Dim3(gx, n1, z1), k_steps=k1, order=r.RowMajor()),
                r.Stage("gemm2", r.Dim3(gx, n2, 1), k_steps=k2, order=r.RowMajor())),
        deps=(r.Dependency("gemm1", "gemm2", "a", pol),))


print(f"# reference simulate() on the B200-grid GPT-3 MLP B=1024 scenario (GeMM1 4x12xz, "
      f"GeMM2 4x24 tiles, GpuConfig(74) CTA pairs); host: {platform.processor() or platform.machine()}, "
      f"os.cpu_count() = {os.cpu_count()}, 1 core used (GIL); best / median of 5")
for name, pol in (("RowSync", r.RowSync()), ("TileSync", r.TileSync())):
    for z1 in (1, 2):
        sc = scenario(pol, z1)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            trace, metrics = r.simulate(sc)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:8s} GeMM1 z={z1}: best {min(ts):8.1f} ms, median {statistics.median(ts):8.1f} ms, "
              f"{len(trace.events)} events, deadlock {metrics.deadlock}")
