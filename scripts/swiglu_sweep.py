"""LLaMA-8B SwiGLU MLP sweep (fused vs stream vs cuBLAS), as in bench.py's sweep."""
import json
import sys

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402

if __name__ == "__main__":
    for r in planner.sweep_swiglu(device="cuda"):
        print(json.dumps(r), flush=True)
