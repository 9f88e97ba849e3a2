import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Run a few dynamics train steps at B=36 (target for ncu captures; no timing printed)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.optim import WsdSchedule
from paper_2510_27002_b200.rng import stream
from paper_2510_27002_b200.tensor import Tensor
from paper_2510_27002_b200.trainer import DynamicsTrainStep

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = 36
cfg = DynamicsConfig(patches_per_frame=256, max_frames=16)
m = DynamicsModel(cfg, seed=0)
tr = DynamicsTrainStep(m, WsdSchedule(3e-5, 1000, 10))
tok = torch.as_tensor(stream(1, "t").integers(0, 1024, size=(B, 16, 256))).cuda()
lat = Tensor(torch.randn(B, 15, 32, device="cuda") * 0.1)
for k in range(steps):
    l = tr.step(k, tok, lat)
torch.cuda.synchronize()
print("loss", float(l.data))
