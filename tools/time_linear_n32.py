import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""fp32 latent projection 512 -> 32 (tokenizer/LAM to_latent) at the pretrain_lam stage shape."""
import torch

from paper_2510_27002_b200 import kernels as K, _lib as L

L.ensure_device()
R = 147456
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(R, 512, device="cuda", generator=g)
w = torch.randn(512, 32, device="cuda", generator=g) * 0.05
b = torch.randn(32, device="cuda", generator=g)
y = K.linear_f32(x, w, b)
ref = x.double() @ w.double() + b.double()
print("rel err vs f64", float((y.double() - ref).norm() / ref.norm()))
for _ in range(3):
    K.linear_f32(x, w, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    K.linear_f32(x, w, b)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"linear_f32 512->32, R={R}: {us:.1f} us ({R * 512 * 4 / us / 1e3:.0f} GB/s, {2 * R * 512 * 32 / us / 1e6:.1f} TFLOP/s)")
torch.save(y.cpu(), "/tmp/lin_y.pt")
# bit-identity against the one-thread-per-output kernel (chosen for a 4-byte-misaligned x)
xb = torch.empty(R * 512 + 1, device="cuda")
xm = xb[1:].view(R, 512)
xm.copy_(x)
yg = K.linear_f32(xm, w, b)
print("bit-identical to the sequential-k kernel:", bool(torch.equal(yg, y)))
