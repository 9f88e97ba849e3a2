import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""VQ forward timing at the B=36 latent shape (147456 x 32 against 1024 codes) for the libjz.so in argv[1]."""
import torch

from paper_2510_27002_b200 import _lib as L
if len(sys.argv) > 1:
    L.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
from paper_2510_27002_b200 import kernels as Kn  # noqa: E402

L.ensure_device()
g = torch.Generator(device="cuda").manual_seed(0)
z = torch.randn(147456, 32, device="cuda", generator=g) * 0.3
cb = torch.randn(1024, 32, device="cuda", generator=g) * 0.3
fn = lambda: Kn.vq_fwd(z, cb)
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
print(f"vq_fwd {us:.1f} us  {2.0 * 147456 * 1024 * 32 / us / 1e6:.1f} TFLOP/s ({pathlib.Path(sys.argv[1]).name if len(sys.argv) > 1 else 'default'})")
