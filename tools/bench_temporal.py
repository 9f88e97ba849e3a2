import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))  # noqa: E402
"""Temporal attention fwd/bwd per-launch time at the C3 shape (B=36, T=16, S=257, H=8)."""
import torch

from paper_2510_27002_b200 import kernels as K, _lib as L

L.ensure_device()
B, T, S, H = 36, 16, 257, 8
D = H * 64
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (torch.randn(B * T * S, 3 * D, device="cuda", generator=g)).bfloat16()
out, lse = K.attn_temporal_fwd(qkv, B, T, S, H)
dout = torch.randn(B * T * S, D, device="cuda", generator=g).bfloat16()
dq = torch.empty_like(qkv)
cs = torch.empty(3 * D, device="cuda")


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


f = t(lambda: K.attn_temporal_fwd(qkv, B, T, S, H))
b = t(lambda: K.attn_temporal_bwd(qkv, out, dout, lse, B, T, S, H, dqkv=dq, colsum=cs))
rows = B * T * S
print(f"temporal fwd {f:.1f} us ({rows * (3 * D * 2 + D * 2 + H * 4) / f / 1e3:.0f} GB/s), "
      f"bwd {b:.1f} us ({rows * (3 * D * 2 + D * 2 + 3 * D * 2) / b / 1e3:.0f} GB/s)")
b2 = t(lambda: K.attn_temporal_bwd(qkv, out, dout, lse, B, T, S, H, dqkv=dq))
print(f"bwd without column sums {b2:.1f} us")
for Bx in (4, 12):
    q2 = qkv[: Bx * T * S]
    o2, l2 = K.attn_temporal_fwd(q2, Bx, T, S, H)
    tb = t(lambda: K.attn_temporal_bwd(q2, o2, dout[: Bx * T * S], l2, Bx, T, S, H))
    print(f"B={Bx}: bwd {tb:.1f} us ({Bx * T * S * (3 * D * 2 + D * 2 + 3 * D * 2) / tb / 1e3:.0f} GB/s)")
