import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Scratch: time one dynamics train step at B=36 (jasmine-base dims, patch 4)."""
import sys
import time

import numpy as np
import torch

from paper_2510_27002_b200 import rng as R
from paper_2510_27002_b200.dynamics import DynamicsConfig, DynamicsModel
from paper_2510_27002_b200.optim import adamw_init, adamw_step
from paper_2510_27002_b200.tensor import Tensor

B = int(sys.argv[1]) if len(sys.argv) > 1 else 36
cfg = DynamicsConfig(model_dim=512, heads=8, ffn_dim=2048, blocks=6, token_codes=1024, action_latent_dim=32,
                     patches_per_frame=256, max_frames=16)
m = DynamicsModel(cfg, seed=0)
tokens = torch.as_tensor(R.stream(1, "bench-tokens").integers(0, 1024, size=(B, 16, 256))).cuda()
lat = Tensor(torch.randn(B, 15, 32, device="cuda") * 0.1)
opt = adamw_init(m.params)


def step(k):
    loss, _ = m.loss(tokens, lat, R.stream(0, "dynamics", "step", k))
    loss.backward()
    adamw_step(m.params, {n: p.grad for n, p in m.params.items()}, opt, 3e-5, check="deferred")
    return loss


for k in range(3):
    l = step(k)
torch.cuda.synchronize()
print("warm loss", float(l.data))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
t0 = time.time()
e0.record()
for k in range(n):
    l = step(3 + k)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"B={B}: {ms:.2f} ms/step  {B * 16 / ms * 1e3:.0f} frames/s  (host {1e3 * (time.time() - t0) / n:.1f} ms/step) loss {float(l.data):.4f}")
if "prof" in sys.argv:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step(100)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40))
