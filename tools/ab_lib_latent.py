import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""512 -> 32 fp32 latent projection timing at R = 147456 (B=36) for the libjz.so in argv[1]."""
import torch

from paper_2510_27002_b200 import _lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(147456, 512, device="cuda", generator=g)
W = torch.randn(512, 32, device="cuda", generator=g)
b = torch.randn(32, device="cuda", generator=g)
y = torch.empty(147456, 32, device="cuda")
fn = lambda: Kn.linear_f32(x, W, b, out=y)
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fn()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"latent projection {us:.1f} us  {2.0 * 147456 * 512 * 32 / us / 1e6:.1f} TFLOP/s")
