"""Test configuration: the `gpu` marker, repo on sys.path, and an in-tree build of
libtilesync_b200.so when it is missing (nvcc cross-compiles without a GPU)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    lib = ROOT / "paper_2305_13450_b200" / "libtilesync_b200.so"
    if not lib.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2305_13450_b200")], check=True)


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
