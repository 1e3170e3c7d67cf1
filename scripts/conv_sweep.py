"""ResNet-38 conv-pair latency sweep (fused Conv2DTileSync vs stream-synced vs cuDNN)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2305_13450_b200 import planner  # noqa: E402

if __name__ == "__main__":
    batches = tuple(int(b) for b in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1, 8, 32, 128, 256)
    for r in planner.sweep_conv(batches=batches, device="cuda"):
        print(json.dumps(r), flush=True)
