import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""C5 sampling rollout timing only (bench.py's secondary C5 measurement): B=64, 4 cond -> 12 generated frames, 25
MaskGIT steps. Environment switches (e.g. JZ_LN_FUSION=0) select variants for same-box A/B runs."""
import torch

import bench
from paper_2510_27002_b200 import _lib as L

L.ensure_device()
r = bench.secondary_configs(torch.device("cuda"))["sample"]
print(f"sample {r['value']} frames/s, rollouts {r['rollouts_ms']} ms")
