import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Event-timed AdamW over the jasmine-base dynamics parameter count (26,432,032 fp32 params, flat)."""
import torch

from paper_2510_27002_b200 import _lib as L
from paper_2510_27002_b200 import kernels as Kn

L.ensure_device()
n = 26432032
p, g, m, v = (torch.randn(n, device="cuda") for _ in range(4))
v = v.abs()
fn = lambda: Kn.adamw(p, g, m, v, lr=1e-4, b1=0.9, b2=0.95, omb1=0.1, omb2=0.05, bc1=0.65, bc2=0.4, eps=1e-8, lrwd=1e-5)
for _ in range(3):
    fn()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    fn()
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) / 20 * 1e3
print(f"AdamW n={n}: {us:.1f} us  {28 * n / us / 1e3:.0f} GB/s (28 B/param)")
